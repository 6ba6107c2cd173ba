"""Config 4 (BERT-large, d = 1024, 16 heads, FFN 4096, L = 128) at N = 2^16: the plans `bench.py
--dims large` times (layer.FusedLinearLayer's plans at blb_inputs.BENCH_BSGS), sampled outputs
bit-exact against the oracle.

* FFN1 (C11, 4 input ciphertexts of X in R^{128 x 1024}, W_1 in R^{1024 x 4096}): one output,
  GPU-evaluated as the output slice the plan would hand to a rank;
* Q K^T at the BERT-large shape (H = 16 = H_p, no padded heads, d_h = 64: g = 16, J = 4), level 3.

Only the tested slices are encoded (the whole layer's 91 GB of plaintexts are not needed here).
Slow: the oracle runs 2^16-point u128 NTTs on the host."""
import numpy as np
import pytest
import torch

import blb_inputs as bi
import oracle as O
import oracle.matmul as mm
import oracle.matmul_cc as cc

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

blb = pytest.importorskip("paper_2508_19525_b200")
from paper_2508_19525_b200.layer import Dims, FusedLinearLayer  # noqa: E402

DIMS = bi.BERT_LARGE
L, D, H, FFN = DIMS["L"], DIMS["d"], DIMS["H"], DIMS["ffn"]
DELTA = 2.0 ** 40


@pytest.fixture(scope="module")
def large():
    P = bi.BERT
    pr = O.prime_chain(P.log_n, list(P.q_bits) + list(P.p_bits))
    ctx = O.Ctx(P.log_n, pr[:5], pr[5:], P.dnum)
    params = blb.Params.from_preset(P)
    layer = FusedLinearLayer(params, Dims(**DIMS), bsgs=bi.BENCH_BSGS)   # plans only: no weights loaded
    return dict(ctx=ctx, params=params, layer=layer, key=bi.crypto_key(4, 44))


def encrypt_both(b, sk, s_ntt, zs, level, id0, enc_key):
    ctx, params = b["ctx"], b["params"]
    octs, gcts = [], []
    for t, z in enumerate(zs):
        pt = O.encode(ctx, z, DELTA, level)
        octs.append(O.encrypt(ctx, enc_key, s_ntt, pt, level, id0 + t, DELTA))
        gcts.append(blb.encrypt(params, sk, params.encode(torch.tensor(z), DELTA, level), level, enc_key, id0 + t,
                                DELTA))
    return octs, gcts


def same(g, o):
    assert g.level == o.level and g.scale == o.scale
    return np.array_equal(blb.to_numpy_u64(g.data), o.data)


def test_bert_large_ffn1_sampled_output_bit_exact(large):
    ctx, params, layer = large["ctx"], large["params"], large["layer"]
    F = bi.bert_ffn_inputs(L, D, H, FFN)
    plan_g = layer.plans["ffn1"]
    plan_o = mm.plan_spatial(F["W1"], L, ctx.n, bi.BENCH_BSGS["ffn1"])
    assert plan_o.n_plaintexts == plan_g.n_pt and plan_o.rotation_steps() == plan_g.rotation_steps()
    steps = plan_o.rotation_steps()
    okeys = O.keygen(ctx, large["key"], steps)
    gkeys, sk = blb.keygen(params, large["key"], steps)
    zs = list(mm.pack_spatial(F["X2"], ctx.n))
    octs, gcts = encrypt_both(large, sk, okeys.s_ntt, zs, layer.level, 4200, bi.crypto_key(5, 44))
    o = 11
    (ref,) = mm.matmul_cp(ctx, okeys, octs, plan_o, out_ids=[o])
    pts = plan_g.encode_weights(F["W1"], o, 1)
    (got,) = plan_g(gkeys, gcts, pts, o, 1)
    assert same(got, ref)


def test_bert_large_qk_sampled_output_bit_exact(large):
    """Row a7 at the BERT-large shape: H = 16 (no padding), d_h = 64, g = 16, J = 4, B = 16, level 3."""
    ctx, params, layer = large["ctx"], large["params"], large["layer"]
    rng = np.random.default_rng(44)
    Q, K = rng.normal(0, 1, (H, L, D // H)) / 8, rng.normal(0, 1, (H, L, D // H)) / 8
    plan_o = cc.plan_qk(L, H, D // H, ctx.n)
    assert (plan_o.J, plan_o.g, plan_o.B) == (4, 16, 16)
    assert layer.qk.rotation_steps() == plan_o.rotation_steps()
    steps = plan_o.rotation_steps()
    okeys = O.keygen(ctx, large["key"], steps, relin=True)
    gkeys, sk = blb.keygen(params, large["key"], steps, relin=True)
    lvl = layer.level - 1
    oq, gq = encrypt_both(large, sk, okeys.s_ntt, cc.pack_mhp(Q, plan_o), lvl, 4300, bi.crypto_key(5, 45))
    ok, gk = encrypt_both(large, sk, okeys.s_ntt, cc.pack_mhp(K, plan_o), lvl, 4310, bi.crypto_key(5, 45))
    o = 6
    (ref,) = cc.qk_encrypted(ctx, okeys, oq, ok, plan_o, out_ids=[o])
    gout = layer.qk(gkeys, gq, gk, layer.qk.encode_masks())
    assert len(gout) == plan_o.n_out and same(gout[o], ref)
