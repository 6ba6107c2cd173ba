"""Oracle fused-block HE chains of row f2 -- TEST INFRASTRUCTURE ONLY.

The linear (green) operators of BLB's nonlinear-layer decompositions that the fine-grained
fusion keeps under CKKS between two MPC steps (fig:fusion_pattern P:699-704, Table 6
P:716-720; operator decompositions App. B, Alg. "Secure LayerNorm / GeLU / Softmax",
P:1059-1186), stated with the oracle's CKKS primitives in the order the algorithms give
(reading C21):

  negexp     Softmax lines 2-4: d = X - Xbar (sadd_cc), t = d * 2^-6 (ewmul_cp),
             y = t + 1 (ewadd_cp), six squarings y <- y (x) y (ewmul_cc) = (1 + d/2^6)^(2^6).
  ln_head    LayerNorm lines 1-6: row sums over the D columns of the spatial-first
             ciphertexts (ewadd_cc across ciphertexts + rotate-and-sum over the c column blocks,
             P:365-376, fused form: every block holds the total, no mask / broadcast),
             mu = sum * (1/D), X_mu = X - mu, X_mu^2, the same row sum, sigma^2 = sum * (1/D).
  ln_tail    LayerNorm lines 8-10: X_mu (x) (1/sigma) (smul_cc with the client's
             spatial-first broadcast of 1/sigma), * gamma (ewmul_cp), + beta (ewadd_cp).
  gelu_head  GeLU lines 1-4: x^2, x^3 = x^2 x, x^4 = x^2 x^2 (ewmul_cc), the
             ewmul_cp's a x^4, b x^3, c x^2, (0.5 +- d) x, and F0 = a x^4 - b x^3 + c x^2 +
             (0.5 - d) x + e, F1 = a x^4 + b x^3 + c x^2 + (0.5 + d) x + e.

Every ct x pt product uses a constant / per-column plaintext encoded at the scale of the prime
the following rescale drops (reading S6), every ct x ct product is relinearised and rescaled;
levels are aligned by dropping limbs (C9); ewadd_cp encodes the constant at the ciphertext's own
scale and level.
"""
from __future__ import annotations

import numpy as np

import oracle as O

# BOLT's GeLU approximation coefficients are not printed in the paper ("The concrete parameters can
# be found in BOLT"); reading C21 fits a|x|^4 + b|x|^3 + c|x|^2 + d|x| + e to
# GeLU(x) - 0.5 x = 0.5 x erf(x / sqrt 2) on [0, 2.7] by least squares (blb_inputs.GELU_COEF, an input).


def drop(ct: O.Ct, level: int) -> O.Ct:
    """Exact level drop (C9): keep the limbs q_0..q_level."""
    assert level <= ct.level
    return O.Ct(ct.data[:, : level + 1].copy(), level, ct.scale)


def sub(ctx: O.Ctx, a: O.Ct, b: O.Ct) -> O.Ct:
    """a - b limb-wise mod q_i (same level)."""
    assert a.level == b.level
    out = np.empty_like(a.data)
    for i in range(a.level + 1):
        q = np.uint64(ctx.mods[i])
        out[:, i] = (a.data[:, i] + (q - b.data[:, i])) % q
    return O.Ct(out, a.level, a.scale)


def add_const(ctx: O.Ctx, ct: O.Ct, vec) -> O.Ct:
    """ewadd_cp: ct + Encode(vec) at the ciphertext's scale and level."""
    pt = O.encode(ctx, np.broadcast_to(np.asarray(vec, dtype=np.float64), (ctx.n,)).copy(), ct.scale, ct.level)
    z = np.zeros_like(pt)
    return O.add(ctx, ct, O.Ct(np.stack([pt, z]), ct.level, ct.scale))


def mul_const(ctx: O.Ctx, ct: O.Ct, vec, target: float | None = None) -> O.Ct:
    """ewmul_cp + rescale: the plaintext at scale q_level (S6), so the scale is kept exactly; with
    a target scale, at q_level * target / ct.scale so the result lands on that scale (the terms of
    one sum are brought to one scale this way)."""
    s = float(ctx.q[ct.level]) if target is None else float(ctx.q[ct.level]) * target / ct.scale
    pt = O.encode(ctx, np.broadcast_to(np.asarray(vec, dtype=np.float64), (ctx.n,)).copy(), s, ct.level)
    return O.rescale(ctx, O.mul_pt(ctx, ct, pt, s))


def square(ctx, keys, a):
    return O.rescale(ctx, O.mul_relin(ctx, a, a, keys))


def mul(ctx, keys, a, b):
    lv = min(a.level, b.level)
    return O.rescale(ctx, O.mul_relin(ctx, drop(a, lv), drop(b, lv), keys))


def negexp(ctx: O.Ctx, keys: O.Keys, x: O.Ct, xbar: O.Ct, t: int = 6) -> O.Ct:
    y = mul_const(ctx, sub(ctx, x, xbar), 2.0 ** -t)
    y = add_const(ctx, y, 1.0)
    for _ in range(t):
        y = square(ctx, keys, y)
    return y


def row_sum(ctx: O.Ctx, keys: O.Keys, cts: list, L: int) -> O.Ct:
    """sum over all columns: add the ciphertexts, then rotate-and-sum over the n/L blocks."""
    s = cts[0]
    for c in cts[1:]:
        s = O.add(ctx, s, c)
    return O.rotate_sum(ctx, s, keys, L, ctx.n // L)


def ln_head(ctx: O.Ctx, keys: O.Keys, xs: list, L: int, D: int):
    """-> (X_mu ciphertexts, sigma^2 ciphertext)."""
    mu = mul_const(ctx, row_sum(ctx, keys, xs, L), 1.0 / D)
    xmu = [sub(ctx, drop(x, mu.level), mu) for x in xs]
    sq = [square(ctx, keys, v) for v in xmu]
    var = mul_const(ctx, row_sum(ctx, keys, sq, L), 1.0 / D)
    return xmu, var


def ln_tail(ctx: O.Ctx, keys: O.Keys, xmu: list, rs: O.Ct, gamma: list, beta: list) -> list:
    """gamma / beta: per ciphertext, slot vectors of the per-column weights (spatial-first)."""
    out = []
    for v, g, b in zip(xmu, gamma, beta):
        y = mul(ctx, keys, v, rs)
        y = mul_const(ctx, y, g)
        out.append(add_const(ctx, y, b))
    return out


def gelu_head(ctx: O.Ctx, keys: O.Keys, x: O.Ct, coef) -> tuple:
    a, b, c, d, e = coef
    x2 = square(ctx, keys, x)
    x3 = mul(ctx, keys, x2, x)
    x4 = square(ctx, keys, x2)
    s4 = x4.scale
    ax4 = mul_const(ctx, x4, a)
    lv = ax4.level
    bx3 = drop(mul_const(ctx, x3, b, s4), lv)
    cx2 = drop(mul_const(ctx, x2, c, s4), lv)
    xm = drop(mul_const(ctx, x, 0.5 - d, s4), lv)
    xp = drop(mul_const(ctx, x, 0.5 + d, s4), lv)
    base = O.add(ctx, ax4, cx2)
    f0 = add_const(ctx, O.add(ctx, sub(ctx, base, bx3), xm), e)
    f1 = add_const(ctx, O.add(ctx, O.add(ctx, base, bx3), xp), e)
    return f0, f1
