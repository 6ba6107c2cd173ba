"""Row f2 GPU parity: the fused-block chains (paper_2508_19525_b200/blocks.py) against the
oracle's (oracle/blocks.py, pinned in test_oracle_blocks.py) on the Table-6-block-3-shaped chain
{60, 40 x 7} + {60} at N = 2^12: every output limb bit-exact, the same scales."""
import math

import numpy as np
import pytest
import torch

import blb_inputs as bi
import oracle as O
import oracle.blocks as OB
import oracle.matmul as mm

pytestmark = pytest.mark.gpu

blb = pytest.importorskip("paper_2508_19525_b200")
from paper_2508_19525_b200.blocks import Chains  # noqa: E402

L = 16


@pytest.fixture(scope="module")
def pair():
    P = bi.F2TOY
    pr = O.prime_chain(P.log_n, list(P.q_bits) + list(P.p_bits))
    k = len(P.q_bits)
    ctx = O.Ctx(P.log_n, pr[:k], pr[k:], P.dnum)
    g = blb.Params(P.log_n, pr[:k], pr[k:], P.dnum)
    steps = [L << i for i in range(int(math.log2(ctx.n // L)))]
    okeys = O.keygen(ctx, bi.crypto_key(4, 95), steps, relin=True)
    gkeys, sk = blb.keygen(g, bi.crypto_key(4, 95), steps, relin=True)
    assert Chains(g, gkeys).rotation_steps(L) == steps
    return ctx, okeys, g, gkeys, sk


def enc(pair, z, cid, lvl=None):
    ctx, okeys, g, gkeys, sk = pair
    lvl = ctx.K - 1 if lvl is None else lvl
    pt = O.encode(ctx, z, 2.0 ** 40, lvl)
    o = O.encrypt(ctx, bi.crypto_key(5, 95), okeys.s_ntt, pt, lvl, cid, 2.0 ** 40)
    c = blb.encrypt(g, sk, g.encode(torch.tensor(z), 2.0 ** 40, lvl), lvl, bi.crypto_key(5, 95), cid, 2.0 ** 40)
    assert np.array_equal(blb.to_numpy_u64(c.data), o.data)
    return o, c


def same(c, o):
    assert c.level == o.level and c.scale == o.scale
    assert np.array_equal(blb.to_numpy_u64(c.data), o.data)


def test_negexp_bit_exact(pair):
    ctx, okeys, g, gkeys, _ = pair
    rng = np.random.default_rng(96)
    (ox, gx), (ob, gb) = enc(pair, rng.uniform(-6, 0, ctx.n), 1), enc(pair, rng.uniform(0, 7, ctx.n), 2)
    same(Chains(g, gkeys).negexp(gx, gb), OB.negexp(ctx, okeys, ox, ob))


def test_layernorm_bit_exact(pair):
    ctx, okeys, g, gkeys, _ = pair
    rng = np.random.default_rng(97)
    D = 2 * (ctx.n // L)
    X = rng.normal(0, 1, (L, D))
    io = [enc(pair, z, 10 + b) for b, z in enumerate(mm.pack_spatial(X, ctx.n))]
    ch = Chains(g, gkeys)
    gxmu, gvar = ch.ln_head([c for _, c in io], L, D)
    oxmu, ovar = OB.ln_head(ctx, okeys, [o for o, _ in io], L, D)
    same(gvar, ovar)
    for a, b in zip(gxmu, oxmu):
        same(a, b)
    ors, grs = enc(pair, np.tile(rng.uniform(0.5, 2, L), ctx.n // L), 30, lvl=oxmu[0].level)
    gam = mm.pack_spatial(np.tile(rng.normal(1, 0.1, D), (L, 1)), ctx.n)
    bet = mm.pack_spatial(np.tile(rng.normal(0, 0.1, D), (L, 1)), ctx.n)
    for a, b in zip(ch.ln_tail(gxmu, grs, gam, bet), OB.ln_tail(ctx, okeys, oxmu, ors, gam, bet)):
        same(a, b)


def test_gelu_head_bit_exact(pair):
    ctx, okeys, g, gkeys, _ = pair
    rng = np.random.default_rng(98)
    ox, gx = enc(pair, rng.uniform(-2.7, 2.7, ctx.n), 40)
    for a, b in zip(Chains(g, gkeys).gelu_head(gx, bi.GELU_COEF), OB.gelu_head(ctx, okeys, ox, bi.GELU_COEF)):
        same(a, b)


def test_level_ops(pair):
    """blb_drop_level keeps the low limbs exactly; blb_add_pt adds to c0 only; blb_sub = a - b."""
    ctx, okeys, g, gkeys, _ = pair
    rng = np.random.default_rng(99)
    (oa, ga), (ob, gb) = enc(pair, rng.uniform(-1, 1, ctx.n), 50), enc(pair, rng.uniform(-1, 1, ctx.n), 51)
    same(blb.drop_level(g, ga, 3), OB.drop(oa, 3))
    same(blb.sub(g, ga, gb), OB.sub(ctx, oa, ob))
    pt = O.encode(ctx, rng.uniform(-1, 1, ctx.n), oa.scale, oa.level)
    got = blb.add_pt(g, ga, blb.from_numpy_u64(pt))
    want = O.add(ctx, oa, O.Ct(np.stack([pt, np.zeros_like(pt)]), oa.level, oa.scale))
    same(got, want)


def test_batched_chains_bit_exact(pair):
    """The lockstep (batched) chains the bench runs -- blb_mul_relin_batch over several independent
    ciphertexts -- give every ciphertext the oracle's single-ciphertext bits."""
    ctx, okeys, g, gkeys, _ = pair
    rng = np.random.default_rng(100)
    xs = [enc(pair, rng.uniform(-6, 0, ctx.n), 60 + t) for t in range(3)]
    xb = [enc(pair, rng.uniform(0, 7, ctx.n), 70 + t) for t in range(3)]
    ch = Chains(g, gkeys)
    for got, (ox, _), (ob, _) in zip(ch.negexp_n([c for _, c in xs], [c for _, c in xb]), xs, xb):
        same(got, OB.negexp(ctx, okeys, ox, ob))
    gs = [enc(pair, rng.uniform(-2.7, 2.7, ctx.n), 80 + t) for t in range(3)]
    for (f0, f1), (ox, _) in zip(ch.gelu_head_n([c for _, c in gs], bi.GELU_COEF), gs):
        r0, r1 = OB.gelu_head(ctx, okeys, ox, bi.GELU_COEF)
        same(f0, r0)
        same(f1, r1)
