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
        q = float(self.p.moduli[ct.level])
        s = q if target is None else q * target / ct.scale
        return blb.rescale(self.p, blb.mul_pt(self.p, ct, self._encode(vec, s, ct.level), s))

    def square(self, a):
        return blb.rescale(self.p, blb.mul_relin(self.p, self.keys, a, a))

    def mul(self, a, b):
        lv = min(a.level, b.level)
        return blb.rescale(self.p, blb.mul_relin(self.p, self.keys, self.drop(a, lv), self.drop(b, lv)))

    # ---- the chains ----
    def negexp(self, x, xbar, t: int = 6):
        y = self.mul_const(blb.sub(self.p, x, xbar), 2.0 ** -t)
        y = self.add_const(y, 1.0)
        for _ in range(t):
            y = self.square(y)
        return y

    def row_sum(self, cts: list, L: int):
        s = cts[0]
        for c in cts[1:]:
            s = blb.add(self.p, s, c)
        return blb.rotate_sum(self.p, self.keys, s, L, self.p.n // L)

    def ln_head(self, xs: list, L: int, D: int):
        mu = self.mul_const(self.row_sum(xs, L), 1.0 / D)
        xmu = [blb.sub(self.p, self.drop(x, mu.level), mu) for x in xs]
        var = self.mul_const(self.row_sum([self.square(v) for v in xmu], L), 1.0 / D)
        return xmu, var

    def ln_tail(self, xmu: list, rs, gamma: list, beta: list) -> list:
        out = []
        for v, g, b in zip(xmu, gamma, beta):
            y = self.mul_const(self.mul(v, rs), g)
            out.append(self.add_const(y, b))
        return out

    def gelu_head(self, x, coef):
        a, b, c, d, e = coef
        x2 = self.square(x)
        x3 = self.mul(x2, x)
        x4 = self.square(x2)
        s4 = x4.scale
        ax4 = self.mul_const(x4, a)
        lv = ax4.level
        bx3 = self.drop(self.mul_const(x3, b, s4), lv)
        cx2 = self.drop(self.mul_const(x2, c, s4), lv)
        xm = self.drop(self.mul_const(x, 0.5 - d, s4), lv)
        xp = self.drop(self.mul_const(x, 0.5 + d, s4), lv)
        base = blb.add(self.p, ax4, cx2)
        f0 = self.add_const(blb.add(self.p, blb.sub(self.p, base, bx3), xm), e)
        f1 = self.add_const(blb.add(self.p, blb.add(self.p, base, bx3), xp), e)
        return f0, f1

    def rotation_steps(self, L: int) -> list[int]:
        steps, s = [], L
        while s < self.p.n:
            steps.append(s)
            s *= 2
        return steps
