"""Row f2: the fused-block HE chains between MPC steps (reading C21).

The linear operators of BLB's nonlinear-layer decompositions kept under CKKS by the
fine-grained fusion (fig:fusion_pattern P:699-704; App. B), as sequences of C-ABI
calls (every step runs in libblb.so kernels; this module only sequences them and encodes the
constant plaintexts):

  negexp     Softmax lines 2-4: (1 + (X - Xbar)/2^6)^(2^6), depth 7
  ln_head    LayerNorm lines 1-6: X_mu = X - mean_j X, sigma^2, depth 3
  ln_tail    LayerNorm lines 8-10: X_mu (x) (1/sigma) * gamma + beta, depth 2
  gelu_head  GeLU lines 1-4: F0, F1 from x^2, x^3, x^4, depth 3

Constants and per-column weights are encoded at the scale of the prime the following rescale
drops (reading S6), or at q_l * target / scale to land a sum's terms on one scale; ct x ct
products are relinearised and rescaled; levels are aligned by exact limb drops (C9).  The same
sequences, written independently with the oracle's primitives, are oracle/blocks.py.
"""
from __future__ import annotations

import numpy as np
import torch

import paper_2508_19525_b200 as blb


class Chains:
    def __init__(self, params: blb.Params, keys: blb.Keys):
        self.p, self.keys = params, keys
        self._const = {}

    def _encode(self, vec, scale: float, level: int) -> torch.Tensor:
        v = np.broadcast_to(np.asarray(vec, dtype=np.float64), (self.p.n,))
        key = (v.tobytes() if v.ndim and not np.all(v == v[0]) else float(v[0]), float(scale), int(level))
        pt = self._const.get(key)
        if pt is None:
            pt = self.p.encode(torch.tensor(np.ascontiguousarray(v))[None], scale, level)[0]
            self._const[key] = pt
        return pt

    def drop(self, ct: blb.Ciphertext, level: int) -> blb.Ciphertext:
        return ct if ct.level == level else blb.drop_level(self.p, ct, level)

    def add_const(self, ct, vec):
        return blb.add_pt(self.p, ct, self._encode(vec, ct.scale, ct.level))

    def mul_const(self, ct, vec, target: float | None = None):
        return self.mul_consts([ct], [vec], None if target is None else [target])[0]

    def mul_consts(self, cts: list, vecs: list, targets: list | None = None) -> list:
        """ewmul_cp + rescale of several ciphertexts at one level in one batch."""
        out = [None] * len(cts)
        by_level = {}
        for t, c in enumerate(cts):
            by_level.setdefault(c.level, []).append(t)
        for lvl, idx in by_level.items():
            q = float(self.p.moduli[lvl])
            sc = [q if targets is None else q * targets[t] / cts[t].scale for t in idx]
            pts = [self._encode(vecs[t], s, lvl) for t, s in zip(idx, sc)]
            for t, r in zip(idx, blb.mul_pt_rescale_batch(self.p, [cts[t] for t in idx], pts, sc)):
                out[t] = r
        return out

    def square(self, a):
        return self.squares([a])[0]

    def mul(self, a, b):
        return self.muls([a], [b])[0]

    # batched ct x ct products (one tensor / ModUp / key-switch / rescale batch per call)
    def squares(self, xs: list) -> list:
        return blb.mul_relin_batch(self.p, self.keys, xs, xs)

    def muls(self, as_: list, bs: list) -> list:
        lv = min(min(a.level for a in as_), min(b.level for b in bs))
        return blb.mul_relin_batch(self.p, self.keys, [self.drop(a, lv) for a in as_], [self.drop(b, lv) for b in bs])

    # ---- the chains (lists of independent ciphertexts run in lockstep) ----
    def negexp_n(self, xs: list, xbars: list, t: int = 6) -> list:
        ds = [blb.sub(self.p, x, xb) for x, xb in zip(xs, xbars)]
        ys = [self.add_const(y, 1.0) for y in self.mul_consts(ds, [2.0 ** -t] * len(ds))]
        for _ in range(t):
            ys = self.squares(ys)
        return ys

    def negexp(self, x, xbar, t: int = 6):
        return self.negexp_n([x], [xbar], t)[0]

    def row_sum(self, cts: list, L: int):
        s = cts[0]
        for c in cts[1:]:
            s = blb.add(self.p, s, c)
        return blb.rotate_sum(self.p, self.keys, s, L, self.p.n // L)

    def ln_head(self, xs: list, L: int, D: int):
        mu = self.mul_const(self.row_sum(xs, L), 1.0 / D)
        xmu = [blb.sub(self.p, self.drop(x, mu.level), mu) for x in xs]
        var = self.mul_const(self.row_sum(self.squares(xmu), L), 1.0 / D)
        return xmu, var

    def ln_tail(self, xmu: list, rs, gamma: list, beta: list) -> list:
        ys = self.mul_consts(self.muls(xmu, [rs] * len(xmu)), gamma)
        return [self.add_const(y, b) for y, b in zip(ys, beta)]

    def gelu_head_n(self, xs: list, coef) -> list:
        a, b, c, d, e = coef
        x2 = self.squares(xs)
        x3 = self.muls(x2, xs)
        x4 = self.squares(x2)
        n = len(xs)
        s4 = [y.scale for y in x4]
        ax4 = self.mul_consts(x4, [a] * n)
        bx3 = self.mul_consts(x3, [b] * n, s4)
        cx2 = self.mul_consts(x2, [c] * n, s4)
        xm = self.mul_consts(xs, [0.5 - d] * n, s4)
        xp = self.mul_consts(xs, [0.5 + d] * n, s4)
        out = []
        for t in range(n):
            lv = ax4[t].level
            base = blb.add(self.p, ax4[t], self.drop(cx2[t], lv))
            bx3_t, xm_t, xp_t = self.drop(bx3[t], lv), self.drop(xm[t], lv), self.drop(xp[t], lv)
            f0 = self.add_const(blb.add(self.p, blb.sub(self.p, base, bx3_t), xm_t), e)
            f1 = self.add_const(blb.add(self.p, blb.add(self.p, base, bx3_t), xp_t), e)
            out.append((f0, f1))
        return out

    def gelu_head(self, x, coef):
        return self.gelu_head_n([x], coef)[0]

    def rotation_steps(self, L: int) -> list[int]:
        steps, s = [], L
        while s < self.p.n:
            steps.append(s)
            s *= 2
        return steps
