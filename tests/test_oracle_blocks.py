"""Row f2 oracle pins: the fused-block HE chains (oracle/blocks.py, reading C21) decrypt to the
float64 evaluation of the operator sequences of App. B (LayerNorm lines 1-10 P:1067-1096, GeLU
lines 1-4 P:1107-1113, Softmax lines 2-4 P:1135-1140) within the paper's accuracy target
(MSE < 1e-11), with the multiplicative depths of the algorithms and log2(n/L)
rotations per row sum (Table 3: log2 D rotations, fused form)."""
import math

import numpy as np
import pytest

import blb_inputs as bi
import oracle as O
import oracle.blocks as OB
import oracle.matmul as mm

L = 16


@pytest.fixture(scope="module")
def f2():
    P = bi.F2TOY
    pr = O.prime_chain(P.log_n, list(P.q_bits) + list(P.p_bits))
    ctx = O.Ctx(P.log_n, pr[:len(P.q_bits)], pr[len(P.q_bits):], P.dnum)
    steps = [L << i for i in range(int(math.log2(ctx.n // L)))]
    keys = O.keygen(ctx, bi.crypto_key(4, 90), steps, relin=True)
    return ctx, keys


def enc(ctx, keys, z, cid, lvl=None):
    lvl = ctx.K - 1 if lvl is None else lvl
    return O.encrypt(ctx, bi.crypto_key(5, 90), keys.s_ntt, O.encode(ctx, z, 2.0 ** 40, lvl), lvl, cid, 2.0 ** 40)


def dec(ctx, keys, ct):
    return O.decode(ctx, O.decrypt(ctx, keys.s_ntt, ct), ct.scale)


def test_negexp_chain(f2):
    ctx, keys = f2
    rng = np.random.default_rng(91)
    x = rng.uniform(-6, 0, ctx.n)
    xbar = rng.uniform(0, 7, ctx.n)       # x - xbar in [-13, 0] (T_exp = -13)
    y = OB.negexp(ctx, keys, enc(ctx, keys, x, 1), enc(ctx, keys, xbar, 2))
    assert y.level == ctx.K - 1 - 7        # depth 7 = Table 6 block 2
    ref = (1.0 + (x - xbar) / 64.0) ** 64
    got = dec(ctx, keys, y)
    assert float(((got - ref) ** 2).mean()) < 1e-11
    assert np.abs(ref - np.exp(x - xbar)).max() < 0.02     # the Taylor form itself


def test_layernorm_head_and_tail(f2):
    ctx, keys = f2
    rng = np.random.default_rng(92)
    D = 2 * (ctx.n // L)                   # two spatial-first ciphertexts
    X = rng.normal(0, 1, (L, D))
    cts = [enc(ctx, keys, z, 10 + b) for b, z in enumerate(mm.pack_spatial(X, ctx.n))]
    xmu, var = OB.ln_head(ctx, keys, cts, L, D)
    assert var.level == ctx.K - 1 - 3
    mu = X.mean(axis=1, keepdims=True)
    got_xmu = mm.unpack_spatial([dec(ctx, keys, c) for c in xmu], L, D)
    assert float(((got_xmu - (X - mu)) ** 2).mean()) < 1e-11
    v = dec(ctx, keys, var).reshape(-1, L)               # every column block holds sigma_i^2
    ref_var = ((X - mu) ** 2).mean(axis=1)
    assert float(((v - ref_var[None, :]) ** 2).mean()) < 1e-11
    # tail: X_mu / sigma * gamma + beta (1/sigma from the MPC rsqrt, re-encrypted spatial-first)
    rs = 1.0 / np.sqrt(ref_var)
    rs_ct = enc(ctx, keys, np.tile(rs, ctx.n // L), 30, lvl=xmu[0].level)
    gamma, beta = rng.normal(1, 0.1, D), rng.normal(0, 0.1, D)
    g = mm.pack_spatial(np.tile(gamma, (L, 1)), ctx.n)
    b = mm.pack_spatial(np.tile(beta, (L, 1)), ctx.n)
    out = OB.ln_tail(ctx, keys, xmu, rs_ct, g, b)
    got = mm.unpack_spatial([dec(ctx, keys, c) for c in out], L, D)
    ref = (X - mu) / np.sqrt(ref_var)[:, None] * gamma[None, :] + beta[None, :]
    assert float(((got - ref) ** 2).mean()) < 1e-11


def test_gelu_head(f2):
    ctx, keys = f2
    rng = np.random.default_rng(93)
    x = rng.uniform(-2.7, 2.7, ctx.n)
    a, b, c, d, e = bi.GELU_COEF
    f0, f1 = OB.gelu_head(ctx, keys, enc(ctx, keys, x, 40), bi.GELU_COEF)
    assert f0.level == f1.level == ctx.K - 1 - 3
    r0 = a * x ** 4 - b * x ** 3 + c * x ** 2 + (0.5 - d) * x + e
    r1 = a * x ** 4 + b * x ** 3 + c * x ** 2 + (0.5 + d) * x + e
    g0, g1 = dec(ctx, keys, f0), dec(ctx, keys, f1)
    assert float(((g0 - r0) ** 2).mean()) < 1e-11 and float(((g1 - r1) ** 2).mean()) < 1e-11
    # the piecewise selection of Alg. GeLU line 7 (done in MPC) is GeLU within the fit's 5e-3
    from math import erf, sqrt
    gelu = np.array([0.5 * t * (1 + erf(t / sqrt(2))) for t in x])
    assert np.abs(np.where(x <= 0, g0, g1) - gelu).max() < 5e-3
