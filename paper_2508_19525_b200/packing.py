"""Client-side slot layouts of BLB's packings (argument marshalling for the C ABI).

* spatial-first: ciphertext b holds column b*c + tau of X (L x D)
  at slots tau*L + i, c = N/(2L) columns per ciphertext;
* dense multi-head diagonal (App. C.2): block
  beta = d*heads + h holds Att_h[i, (i+d) mod d_h] for Att of shape (heads, L, d_h).
"""
from __future__ import annotations

import numpy as np


def spatial_slots(X: np.ndarray, n: int) -> np.ndarray:
    """[n_ct][n] float64 slot vectors of X (L x D)."""
    L, D = X.shape
    c = n // L
    n_ct = -(-D // c)
    Xp = np.zeros((L, n_ct * c))
    Xp[:, :D] = X
    # slot tau*L + i of ciphertext b <- X[i, b*c + tau]
    return np.ascontiguousarray(Xp.T.reshape(n_ct, c * L))


def spatial_unslots(Z: np.ndarray, L: int, D: int) -> np.ndarray:
    n_ct, n = Z.shape
    c = n // L
    return Z.reshape(n_ct * c, L).T[:, :D].copy()


def diagonal_slots(Att: np.ndarray, n: int) -> np.ndarray:
    H, L, dh = Att.shape
    c = n // L
    nblk = dh * H
    n_ct = -(-nblk // c)
    blocks = np.zeros((n_ct * c, L))
    i = np.arange(L)
    for d in range(dh):
        blocks[d * H:(d + 1) * H] = Att[:, i, (i + d) % dh]
    return np.ascontiguousarray(blocks.reshape(n_ct, c * L))


def mhp_slots(M: np.ndarray, n: int) -> np.ndarray:
    """Multi-head packing (L, H_p, g) of M (heads, L, D): block c*H_p + h of ciphertext j
    holds column j*g + c of head h; heads padded to H_p = next power of two, g = n/(L H_p)."""
    H, L, D = M.shape
    Hp = 1 << (H - 1).bit_length()
    g = n // (L * Hp)
    J = -(-D // g)
    Mp = np.zeros((J * g, Hp, L))       # [column][head][row]
    Mp[:D, :H, :] = np.transpose(M, (2, 0, 1))
    return np.ascontiguousarray(Mp.reshape(J, g * Hp * L))


def softmax_v_operands(S: np.ndarray, V: np.ndarray, n: int):
    """Slots of the two ct-ct operands of Softmax x V_h: S_h (L x L) and
    Vpad_h^T with V zero-padded from d_h to L columns."""
    H, L, dh = V.shape
    Vt = np.zeros((H, L, L))
    Vt[:, :dh, :] = np.transpose(V, (0, 2, 1))
    return mhp_slots(S, n), mhp_slots(Vt, n)
