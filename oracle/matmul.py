"""Oracle ct-pt MatMul protocols -- TEST INFRASTRUCTURE ONLY.

C11: spatial-first ct-pt MatMul with BSGS (BOLT's protocol, referenced at
     P:361, P:511, P:515 but not restated; reconstructed as the block-diagonal
     identity below, reading S14), with the multi-head-packing (MHP)
     column reorder of P:463-466.
C12: diagonal-input ct-pt MatMul for W_O (App. C.2).

Everything is written at the slot level with numpy (plaintext slot vectors)
and executed with the oracle's CKKS primitives in the order of App. C.1's
BSGS formula:
    Y_b' = sum_g Rot^{gBL}( sum_b sum_i Rot^{-gBL}(Pi_{b,b',gB+i}) (x) Rot^{iL}(X_b) ).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import Ct, Ctx, Keys, add, add_ext, encode, moddown_rescale, mul_pt, rescale, rotate, rotate_ext


# ---------------------------------------------------------------------------
# packing (P:359-361 spatial-first; P:463 MHP (L, H, D/H); P:511 diagonal)
# ---------------------------------------------------------------------------
def pack_spatial(X: np.ndarray, n: int) -> list[np.ndarray]:
    """Spatial-first: ciphertext b holds column bc+tau of X at slots tau*L + i."""
    L, D = X.shape
    c = n // L
    out = []
    for b in range(math.ceil(D / c)):
        z = np.zeros(n)
        for tau in range(c):
            col = b * c + tau
            if col < D:
                z[tau * L:(tau + 1) * L] = X[:, col]
        out.append(z)
    return out


def unpack_spatial(zs: list[np.ndarray], L: int, D: int) -> np.ndarray:
    n = zs[0].shape[0]
    c = n // L
    Y = np.zeros((L, D))
    for col in range(D):
        b, tau = divmod(col, c)
        Y[:, col] = zs[b][tau * L:(tau + 1) * L]
    return Y


def mhp_column_map(d: int, H: int, L: int, n: int) -> list[int]:
    """MHP reorder of output columns (reading S16): heads padded to
    H_p = next pow2 >= H; virtual column v = j*c + cc*H_p + h holds source
    column h*d_h + j*g + cc (g = c/H_p within-head columns per ciphertext),
    or -1 (zero) for padded heads."""
    c = n // L
    Hp = 1 << (H - 1).bit_length()
    dh = d // H
    g = c // Hp
    J = math.ceil(dh / g)
    out = []
    for j in range(J):
        for cc in range(g):
            for h in range(Hp):
                src = h * dh + j * g + cc
                out.append(src if (h < H and j * g + cc < dh) else -1)
    return out


def pack_diagonal_mh(Att: np.ndarray, n: int) -> list[np.ndarray]:
    """Dense multi-head diagonal packing of Att_h (H, L, d_h): block beta = d*H + h
    holds Att_h[i, (i+d) mod d_h] (reading C12)."""
    H, L, dh = Att.shape
    c = n // L
    nblk = dh * H
    out = []
    for b in range(math.ceil(nblk / c)):
        z = np.zeros(n)
        for tau in range(c):
            beta = b * c + tau
            if beta < nblk:
                d, h = divmod(beta, H)
                z[tau * L:(tau + 1) * L] = Att[h, np.arange(L), (np.arange(L) + d) % dh]
        out.append(z)
    return out


# ---------------------------------------------------------------------------
# plan (C11 / C12)
# ---------------------------------------------------------------------------
@dataclass
class Plan:
    L: int
    n: int
    n_in: int
    n_out: int
    B: int
    G: int
    # entries[(b', g)] = list of (b, i) with a non-zero P_{b,b',g,i}
    entries: dict = field(default_factory=dict)
    blocks_fn: object = None

    def pt_vector(self, bp: int, g: int, b: int, i: int) -> np.ndarray:
        """P_{b,b',g,i} = Rot^{-gBL}(Pi_{b,b',gB+i}) as a slot vector (C11)."""
        c = self.n // self.L
        tau = np.arange(c)
        t = g * self.B + i
        Pi = self.blocks_fn(b * c + (tau + t) % c, bp * c + tau).reshape(self.n)
        return np.roll(Pi, g * self.B * self.L)   # right rotation by gBL slots

    @property
    def baby_steps(self) -> dict:
        need = {}
        for (bp, g), lst in self.entries.items():
            for b, i in lst:
                if i > 0:
                    need.setdefault(b, set()).add(i)
        return {b: sorted(s) for b, s in need.items()}

    @property
    def giant_steps(self) -> dict:
        need = {}
        for (bp, g), lst in self.entries.items():
            if g > 0 and lst:
                need.setdefault(bp, set()).add(g)
        return {b: sorted(s) for b, s in need.items()}

    @property
    def n_plaintexts(self) -> int:
        return sum(len(v) for v in self.entries.values())

    @property
    def n_rotations(self) -> int:
        return sum(len(v) for v in self.baby_steps.values()) + sum(len(v) for v in self.giant_steps.values())

    def rotation_steps(self) -> list[int]:
        s = set()
        for b, lst in self.baby_steps.items():
            s.update(i * self.L for i in lst)
        for b, lst in self.giant_steps.items():
            s.update(g * self.B * self.L for g in lst)
        return sorted(s)


def _build(L, n, n_in, n_out, B, blocks_fn) -> Plan:
    """blocks_fn(r[c], col[c]) -> (c, L) array: row tau = the block of Pi for
    input block r[tau] (global index b*c + tau') feeding output column col[tau]
    (zero where out of range)."""
    c = n // L
    G = math.ceil(c / B)
    plan = Plan(L, n, n_in, n_out, B, G, blocks_fn=blocks_fn)
    tau = np.arange(c)
    for bp in range(n_out):
        for g in range(G):
            lst = []
            for b in range(n_in):
                for i in range(B):
                    t = g * B + i
                    if t >= c:
                        continue
                    blocks = blocks_fn(b * c + (tau + t) % c, bp * c + tau)
                    if not np.any(blocks != 0):
                        continue
                    lst.append((b, i))
            if lst:
                plan.entries[(bp, g)] = lst
    return plan


def plan_spatial(W: np.ndarray, L: int, n: int, B: int, col_map: list[int] | None = None) -> Plan:
    """C11.  W: D_in x D_out.  col_map (optional): virtual output column -> source
    column of W or -1 (zero), e.g. mhp_column_map for Q/K feeding matmul_cc."""
    D_in, D_src = W.shape
    if col_map is None:
        col_map = list(range(D_src))
    D_out = len(col_map)
    c = n // L

    cmap = np.asarray(list(col_map) + [-1], dtype=np.int64)

    def fn(r, col):
        src = cmap[np.minimum(col, D_out)]
        ok = (r < D_in) & (src >= 0)
        v = np.where(ok, W[np.minimum(r, D_in - 1), np.maximum(src, 0)], 0.0)
        return np.repeat(v[:, None], L, axis=1)

    return _build(L, n, math.ceil(D_in / c), math.ceil(D_out / c), B, fn)


def plan_diagonal(WO: np.ndarray, H: int, L: int, n: int, B: int) -> Plan:
    """C12.  WO: (H*d_h) x D_out; input = pack_diagonal_mh (block beta = d*H + h).
    Plaintext block for (beta -> col): w[i] = WO[h*d_h + (i+d) mod d_h, col]."""
    D, D_out = WO.shape
    dh = D // H
    c = n // L
    nblk = dh * H
    rows = np.arange(L)

    def fn(beta, col):
        d, h = np.divmod(np.minimum(beta, nblk - 1), H)
        ok = (beta < nblk) & (col < D_out)
        rowidx = h[:, None] * dh + (rows[None, :] + d[:, None]) % dh
        v = WO[rowidx, np.minimum(col, D_out - 1)[:, None]]
        return np.where(ok[:, None], v, 0.0)

    return _build(L, n, math.ceil(nblk / c), math.ceil(D_out / c), B, fn)


# ---------------------------------------------------------------------------
# execution
# ---------------------------------------------------------------------------
def matmul_cp(ctx: Ctx, keys: Keys, cts: list[Ct], plan: Plan, out_ids=None) -> list[Ct]:
    """Evaluate the plan on input ciphertexts (all at one level l).  Plaintexts
    are encoded at scale q_l (reading S6), so one rescale per output ciphertext
    after the giant-step sum returns the input scale exactly (C11)."""
    level = cts[0].level
    assert all(ct.level == level for ct in cts)
    pt_scale = float(ctx.q[level])
    R = {}
    for b, steps in plan.baby_steps.items():
        for i in steps:
            R[(b, i)] = rotate(ctx, cts[b], keys, i * plan.L)
    for b in range(len(cts)):
        R[(b, 0)] = cts[b]
    outs = []
    ids = range(plan.n_out) if out_ids is None else out_ids
    for bp in ids:
        Y = None
        for g in range(plan.G):
            lst = plan.entries.get((bp, g), [])
            # encodes are independent: run them on a thread pool (the C encoder releases the GIL)
            from concurrent.futures import ThreadPoolExecutor
            with ThreadPoolExecutor() as ex:
                pts = list(ex.map(lambda bi: encode(ctx, plan.pt_vector(bp, g, bi[0], bi[1]), pt_scale, level), lst))
            acc = None
            for (b, i), pt in zip(lst, pts):
                term = mul_pt(ctx, R[(b, i)], pt, pt_scale)
                acc = term if acc is None else add(ctx, acc, term)
            if acc is None:
                continue
            # giant step kept in Q_l u P (reading C11, lazy ModDown): Rot_ext(acc) =
            # (P sigma(c0) + u0, u1); g = 0 is the lift (P c0, P c1)
            term = rotate_ext(ctx, acc, keys, g * plan.B * plan.L)
            Y = term if Y is None else add_ext(ctx, Y, term)
        if Y is None:
            Y = Ct(np.zeros_like(cts[0].data), level, cts[0].scale * pt_scale)
            outs.append(rescale(ctx, Y))
            continue
        outs.append(moddown_rescale(ctx, Y))   # ModDown + rescale as one exact rounding (C17)
    return outs


def slot_level(zs: list[np.ndarray], plan: Plan) -> list[np.ndarray]:
    """The same schedule on plaintext slot vectors (no encryption): a pin that the
    plan computes X W exactly up to float rounding (App. A item 6)."""
    n, L = plan.n, plan.L
    outs = []
    for bp in range(plan.n_out):
        Y = np.zeros(n)
        for g in range(plan.G):
            acc = np.zeros(n)
            for b, i in plan.entries.get((bp, g), []):
                acc += plan.pt_vector(bp, g, b, i) * np.roll(zs[b], -i * L)
            Y += np.roll(acc, -g * plan.B * L)
        outs.append(Y)
    return outs
