"""Oracle fused-linear layer step -- TEST INFRASTRUCTURE ONLY.

The order in which one Transformer layer's fused linear operators run under
CKKS and are converted to MPC shares (SURVEY 8(d) configs 2 + 3; BLB's fused
blocks, fig:fusion_pattern P:699-704, Table 6), stated with the
oracle's own plans and primitives so that the product's layer driver
(paper_2508_19525_b200/layer.py) can be compared with it output by output:

  attention  X --QKV ct-pt (C11, MHP column reorder P:466)--> Q^(j), K^(j), V
             Q, K --ct-ct Q_h K_h^T (C13)--> diagonals --CKKS->MPC (Alg. 1)--> shares
             V --CKKS->MPC--> shares ("convert V_h to secret-share form")
  f1         S_h, Vpad_h^T --ct-ct (C15)--> dense-diagonal collapse
             --diagonal-input ct-pt W_O (C12, App. C.2)--> CKKS->MPC
  FFN        X2 --FFN1 ct-pt--> CKKS->MPC;  H1 --FFN2 ct-pt--> CKKS->MPC

Every MatMul starts from a fresh ciphertext at the top level l, except Q K^T
(QKV outputs, level l - 1) and W_O (the Softmax x V outputs, level l - 3).

Mask object ids (reading C19): the mask r of an output ciphertext
must be fresh for every conversion (Alg. 1 line 1 samples r uniformly, P:629;
Theorem 1's simulation, needs an independent r per conversion), so
the ChaCha20 object id of the mask of output o of block b in inference seq is
    id = seq * 2^24 + b * 2^16 + o      (o < 2^16; b: qkv 0, oproj 1, ffn1 2, ffn2 3, qk 4).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

import oracle as O
import oracle.matmul as mm
import oracle.matmul_cc as cc

BLOCK = {"qkv": 0, "oproj": 1, "ffn1": 2, "ffn2": 3, "qk": 4}


def mask_id(seq: int, block: str, o: int) -> int:
    """Reading C19: fresh mask object id per (inference, block, output)."""
    assert 0 <= o < (1 << 16) and 0 <= seq < (1 << 32)
    return (seq << 24) | (BLOCK[block] << 16) | o


@dataclass
class LayerSpec:
    L: int
    d: int
    H: int
    ffn: int
    bsgs: dict
    level: int           # top level l of the fresh input ciphertexts
    plans: dict = field(default_factory=dict)

    @property
    def Hp(self) -> int:
        return 1 << (self.H - 1).bit_length()


def build(ctx: O.Ctx, spec: LayerSpec, WQ, WK, WV, WO, W1, W2) -> LayerSpec:
    """Plans of the layer (C11 / C12 / C13 / C15) for weights W (float64)."""
    L, d, H, n = spec.L, spec.d, spec.H, ctx.n
    cm = mm.mhp_column_map(d, H, L, n)
    # virtual QKV output columns: MHP-reordered Q, then K, then V in natural order
    qkv_map = cm + [d + c if c >= 0 else -1 for c in cm] + list(range(2 * d, 3 * d))
    Wqkv = np.concatenate([WQ, WK, WV], axis=1)
    qk = cc.plan_qk(L, H, d // H, n, spec.bsgs.get("qk") or None)
    spec.plans = {
        "qkv": mm.plan_spatial(Wqkv, L, n, spec.bsgs["qkv"], col_map=qkv_map),
        "qk": qk,
        "sv": cc.plan_sv(L, H, n, spec.bsgs.get("qk") or None),
        "oproj": mm.plan_diagonal(cc.pad_heads_rows(WO, H, spec.Hp), spec.Hp, L, n, spec.bsgs["oproj"]),
        "ffn1": mm.plan_spatial(W1, L, n, spec.bsgs["ffn1"]),
        "ffn2": mm.plan_spatial(W2, L, n, spec.bsgs["ffn2"]),
    }
    spec.J = len(cm) // (n // L)       # MHP ciphertexts of Q (and of K) among the QKV outputs
    return spec


def rotation_steps(spec: LayerSpec) -> list[int]:
    s = set()
    for p in spec.plans.values():
        s.update(p.rotation_steps())
    return sorted(s)


def _masks(ctx, cts, mask_key, seq, block, outs):
    return [(mask_id(seq, block, o),) + tuple(O.mask(ctx, ct, mask_key, mask_id(seq, block, o)))
            for o, ct in zip(outs, cts)]


def layer_step(ctx: O.Ctx, keys: O.Keys, spec: LayerSpec, inputs: dict, mask_key: bytes, seq: int) -> dict:
    """inputs: {'qkv': [Ct] (X), 'sv_s': [Ct] (S_h MHP), 'sv_v': [Ct] (Vpad_h^T MHP), 'ffn1': [Ct] (X2),
    'ffn2': [Ct] (H1)} -> {block: [(mask id, masked [2][N] coef mod q0, server share [N])]}."""
    P, J = spec.plans, spec.J
    res = {}
    qkv = mm.matmul_cp(ctx, keys, inputs["qkv"], P["qkv"])
    qk = cc.qk_encrypted(ctx, keys, qkv[:J], qkv[J:2 * J], P["qk"])
    res["qk"] = _masks(ctx, qk, mask_key, seq, "qk", range(len(qk)))
    res["qkv"] = _masks(ctx, qkv[2 * J:], mask_key, seq, "qkv", range(2 * J, len(qkv)))
    sv = cc.qk_encrypted(ctx, keys, inputs["sv_s"], inputs["sv_v"], P["sv"])
    dense = cc.collapse_dense(sv, P["sv"], spec.d // spec.H, add_fn=lambda a, b: O.add(ctx, a, b))
    op = mm.matmul_cp(ctx, keys, dense, P["oproj"])
    res["oproj"] = _masks(ctx, op, mask_key, seq, "oproj", range(len(op)))
    for name in ("ffn1", "ffn2"):
        y = mm.matmul_cp(ctx, keys, inputs[name], P[name])
        res[name] = _masks(ctx, y, mask_key, seq, name, range(len(y)))
    return res
