"""Full-size parity in the launch configuration bench.py times (BASELINE configs 2/3 at
N = 2^16, the BSGS splits of blb_inputs.BENCH_BSGS, the plan objects of the benched
layer.FusedLinearLayer): the GPU evaluates every output ciphertext, the oracle recomputes
sampled output ciphertexts one by one, and they must agree bit-exactly on every limb.

* QKV (C11 + MHP, B from BENCH_BSGS): a Q output and a V output; the V output also through the layer
  step's CKKS->MPC mask (masked ciphertext and server share);
* FFN1 (B = 64) and FFN2 (12 inputs, B = 16): one output each, through the layer step's mask;
* out-projection (C12, diagonal input with padded heads, B = 16) at level 1, where the layer
  runs it;
* Q K^T at the BERT-base shape (H = 12 -> H_p = 16, d_h = 64: g = 16, J = 4) at level 3;
* Softmax x V (V zero-padded to L = 128: J = 8) at level 4.

Inputs to every oracle call are fresh oracle encryptions of seeded synthetic data (never GPU
outputs); the GPU side encrypts the same messages with the same ids (bit-exact encryption is
pinned by test_gpu_parity).  Slow: the oracle runs 2^16-point u128 NTTs on the host."""
import numpy as np
import pytest
import torch

import blb_inputs as bi
import oracle as O
import oracle.layer as OL
import oracle.matmul as mm
import oracle.matmul_cc as cc

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

blb = pytest.importorskip("paper_2508_19525_b200")
from paper_2508_19525_b200 import packing  # noqa: E402
from paper_2508_19525_b200.layer import Dims, FusedLinearLayer  # noqa: E402

DIMS = bi.BERT_BASE
L, D, H, FFN = DIMS["L"], DIMS["d"], DIMS["H"], DIMS["ffn"]
DELTA = 2.0 ** 40
SEQ = 7


class Okeys:
    """Oracle rotation keys generated on demand (key material depends only on (seed, step))."""

    def __init__(self, ctx, key):
        self.ctx, self.key, self.keys = ctx, key, None

    def get(self, steps, relin=False):
        have = set(self.keys.rot) if self.keys else set()
        need = [s for s in steps if self.ctx.galois(s) not in have]
        want_rlk = relin and (self.keys is None or self.keys.rlk is None)
        if self.keys is None or need or want_rlk:
            k = O.keygen(self.ctx, self.key, need, relin=want_rlk)
            if self.keys is None:
                self.keys = k
            else:
                self.keys.rot.update(k.rot)
                if k.rlk is not None:
                    self.keys.rlk = k.rlk
        return self.keys


@pytest.fixture(scope="module")
def bert():
    P = bi.BERT
    pr = O.prime_chain(P.log_n, list(P.q_bits) + list(P.p_bits))
    ctx = O.Ctx(P.log_n, pr[:5], pr[5:], P.dnum)
    params = blb.Params.from_preset(P)
    layer = FusedLinearLayer(params, Dims(**DIMS), bsgs=bi.BENCH_BSGS)
    A = bi.bert_attention_inputs(L, D)
    F = bi.bert_ffn_inputs(L, D, H, FFN)
    keys_key = A["keys_key"]
    gkeys, sk = blb.keygen(params, keys_key, layer.rotation_steps(), relin=True)
    layer.load_weights(A["WQ"], A["WK"], A["WV"], F["WO"], F["W1"], F["W2"])
    return dict(ctx=ctx, params=params, layer=layer, A=A, F=F, gkeys=gkeys, sk=sk, okeys=Okeys(ctx, keys_key))


def encrypt_both(b, zs, level, id0, enc_key):
    ctx, params, okeys = b["ctx"], b["params"], b["okeys"]
    octs, gcts = [], []
    s_ntt = okeys.get([]).s_ntt
    for t, z in enumerate(zs):
        pt = O.encode(ctx, z, DELTA, level)
        octs.append(O.encrypt(ctx, enc_key, s_ntt, pt, level, id0 + t, DELTA))
        gcts.append(blb.encrypt(params, b["sk"], params.encode(torch.tensor(z), DELTA, level), level, enc_key,
                                id0 + t, DELTA))
        assert np.array_equal(blb.to_numpy_u64(gcts[-1].data), octs[-1].data)
    return octs, gcts


def same(g, o):
    assert g.level == o.level and g.scale == o.scale
    return np.array_equal(blb.to_numpy_u64(g.data), o.data)


def layer_inputs(b):
    """The bench step's encrypted inputs: both sides, same messages and ids."""
    if "inputs" in b:
        return b["inputs"]
    A, F, layer, ctx = b["A"], b["F"], b["layer"], b["ctx"]
    # client-side slot layouts from the oracle's packers (the product's packing.py must agree)
    sv = cc.plan_sv(L, H, ctx.n)
    S_, Kop = cc.sv_operands(F["S"], F["V"])
    slots = {"qkv": mm.pack_spatial(A["X"], ctx.n), "sv_s": cc.pack_mhp(S_, sv), "sv_v": cc.pack_mhp(Kop, sv),
             "ffn1": mm.pack_spatial(F["X2"], ctx.n), "ffn2": mm.pack_spatial(F["H1"], ctx.n)}
    ps, pv = packing.softmax_v_operands(F["S"], F["V"], ctx.n)
    assert np.array_equal(np.stack(slots["sv_s"]), ps) and np.array_equal(np.stack(slots["sv_v"]), pv)
    assert np.array_equal(np.stack(slots["qkv"]), packing.spatial_slots(A["X"], ctx.n))
    o_in, g_in, cid = {}, {}, 4096
    for name, zs in slots.items():
        o_in[name], g_in[name] = encrypt_both(b, list(zs), layer.level, cid, A["enc_key"])
        cid += len(zs)
    b["inputs"] = (o_in, g_in)
    b["step"] = {name: (id0, m, s) for name, id0, (m, s) in layer.step(b["gkeys"], g_in, A["mask_key"], seq=SEQ)}
    return b["inputs"]


def check_masked(b, name, o, oct_out):
    """Layer-step mask of output o of block name == oracle mask of the oracle's output."""
    id0, m, s = b["step"][name]
    first = b["layer"].mask_outputs(name)[0]
    om, osh = O.mask(b["ctx"], oct_out, b["A"]["mask_key"], OL.mask_id(SEQ, name, o))
    assert id0 == OL.mask_id(SEQ, name, first)
    assert np.array_equal(blb.to_numpy_u64(m[o - first]), om)
    assert np.array_equal(blb.to_numpy_u64(s[o - first]), osh)


def test_bench_plans_are_the_tested_plans(bert):
    """The layer bench.py times uses BENCH_BSGS; the oracle plans built from the same dict
    have the same rotation sets and plaintext counts (QKV 8448 / FFN 9216 / O-proj 3072: the
    diagonal input carries the H_p = 16 padded heads of the Softmax x V collapse)."""
    layer, ctx, F, A = bert["layer"], bert["ctx"], bert["F"], bert["A"]
    spec = OL.build(ctx, OL.LayerSpec(L, D, H, FFN, bi.BENCH_BSGS, layer.level), A["WQ"], A["WK"], A["WV"],
                    F["WO"], F["W1"], F["W2"])
    assert OL.rotation_steps(spec) == layer.rotation_steps()
    for name in ("qkv", "oproj", "ffn1", "ffn2"):
        pg, po = layer.plans[name], spec.plans[name]
        assert pg.n_pt == po.n_plaintexts and pg.n_rotations == po.n_rotations, name
        assert pg.rotation_steps() == po.rotation_steps(), name
    assert (layer.plans["qkv"].n_pt, layer.plans["ffn1"].n_pt, layer.plans["ffn2"].n_pt,
            layer.plans["oproj"].n_pt) == (8448, 9216, 9216, 3072)
    assert layer.qk.rotation_steps() == spec.plans["qk"].rotation_steps()
    assert layer.sv.rotation_steps() == spec.plans["sv"].rotation_steps()
    assert (spec.plans["qk"].J, spec.plans["sv"].J) == (4, 8)


def test_qkv_bench_bsgs_sampled_outputs_bit_exact(bert):
    """QKV at the bench's B (BENCH_BSGS): output 0 (Q, MHP) straight from the plan, output 9 (V) through
    the layer mask."""
    o_in, g_in = layer_inputs(bert)
    ctx, layer = bert["ctx"], bert["layer"]
    A = bert["A"]
    spec = OL.build(ctx, OL.LayerSpec(L, D, H, FFN, bi.BENCH_BSGS, layer.level), A["WQ"], A["WK"], A["WV"],
                    bert["F"]["WO"], bert["F"]["W1"], bert["F"]["W2"])
    plan_o = spec.plans["qkv"]
    okeys = bert["okeys"].get(plan_o.rotation_steps())
    sample = [0, 9]
    oout = mm.matmul_cp(ctx, okeys, o_in["qkv"], plan_o, out_ids=sample)
    gout = layer.plans["qkv"](bert["gkeys"], g_in["qkv"], layer.pts["qkv"])
    for o, ref in zip(sample, oout):
        assert same(gout[o], ref), o
    check_masked(bert, "qkv", 9, oout[1])


@pytest.mark.parametrize("name,o", [("ffn1", 5), ("ffn2", 1)])
def test_ffn_sampled_output_through_layer_mask(bert, name, o):
    o_in, _ = layer_inputs(bert)
    ctx, layer, F = bert["ctx"], bert["layer"], bert["F"]
    W = F["W1"] if name == "ffn1" else F["W2"]
    plan_o = mm.plan_spatial(W, L, ctx.n, bi.BENCH_BSGS[name])
    assert plan_o.n_plaintexts == layer.plans[name].n_pt
    okeys = bert["okeys"].get(plan_o.rotation_steps())
    (ref,) = mm.matmul_cp(ctx, okeys, o_in[name], plan_o, out_ids=[o])
    check_masked(bert, name, o, ref)


def test_oproj_level1_sampled_output_bit_exact(bert):
    """Diagonal-input W_O (C12) with padded heads at level 1, as the layer runs it."""
    ctx, layer, F = bert["ctx"], bert["layer"], bert["F"]
    lvl = layer.level - 3
    Hp = layer.Hp
    Att = np.zeros((Hp, L, D // H))
    Att[:H] = F["Att"]
    zs = mm.pack_diagonal_mh(Att, ctx.n)
    octs, gcts = encrypt_both(bert, zs, lvl, 900, bi.crypto_key(5, 33))
    plan_o = mm.plan_diagonal(cc.pad_heads_rows(F["WO"], H, Hp), Hp, L, ctx.n, bi.BENCH_BSGS["oproj"])
    okeys = bert["okeys"].get(plan_o.rotation_steps())
    (ref,) = mm.matmul_cp(ctx, okeys, octs, plan_o, out_ids=[2])
    gout = layer.plans["oproj"](bert["gkeys"], gcts, layer.pts["oproj"])
    assert ref.level == 0 and same(gout[2], ref)


def test_qk_bert_base_shape_sampled_output_bit_exact(bert):
    """Row a7 at the benched shape: H = 12 (padded to 16), d_h = 64, g = 16, J = 4, B = 16, level 3."""
    ctx, layer = bert["ctx"], bert["layer"]
    rng = np.random.default_rng(5)
    Q, K = rng.normal(0, 1, (H, L, D // H)) / 8, rng.normal(0, 1, (H, L, D // H)) / 8
    plan_o = cc.plan_qk(L, H, D // H, ctx.n)
    assert (plan_o.J, plan_o.g, plan_o.B) == (4, 16, 16)
    lvl = layer.level - 1
    oq, gq = encrypt_both(bert, cc.pack_mhp(Q, plan_o), lvl, 700, bi.crypto_key(5, 34))
    ok, gk = encrypt_both(bert, cc.pack_mhp(K, plan_o), lvl, 710, bi.crypto_key(5, 34))
    okeys = bert["okeys"].get(plan_o.rotation_steps(), relin=True)
    o = 3
    (ref,) = cc.qk_encrypted(ctx, okeys, oq, ok, plan_o, out_ids=[o])
    gout = layer.qk(bert["gkeys"], gq, gk, layer.qk_masks, ws=layer.ws)
    assert len(gout) == plan_o.n_out and same(gout[o], ref)


def test_softmax_v_j8_sampled_output_bit_exact(bert):
    """Row f1 at the benched shape: S_h (x) Vpad_h^T with d_h padded to L = 128 (J = 8), level 4."""
    ctx, layer, F = bert["ctx"], bert["layer"], bert["F"]
    plan_o = cc.plan_sv(L, H, ctx.n)
    assert plan_o.J == 8
    A_, Kop = cc.sv_operands(F["S"], F["V"])
    lvl = layer.level
    os_, gs = encrypt_both(bert, cc.pack_mhp(A_, plan_o), lvl, 800, bi.crypto_key(5, 35))
    ov, gv = encrypt_both(bert, cc.pack_mhp(Kop, plan_o), lvl, 820, bi.crypto_key(5, 35))
    okeys = bert["okeys"].get(plan_o.rotation_steps(), relin=True)
    o = 5
    (ref,) = cc.qk_encrypted(ctx, okeys, os_, ov, plan_o, out_ids=[o])
    gout = layer.sv(bert["gkeys"], gs, gv, layer.sv_masks, ws=layer.ws)
    assert len(gout) == plan_o.n_out and same(gout[o], ref)


@pytest.fixture(scope="module")
def bert_dnum1():
    P = bi.BERT_DNUM1
    pr = O.prime_chain(P.log_n, list(P.q_bits) + list(P.p_bits))
    return dict(ctx=O.Ctx(P.log_n, pr[:5], pr[5:], P.dnum), params=blb.Params.from_preset(P))


def test_dnum1_matmul_sampled_output_bit_exact(bert_dnum1):
    """The config-2 dnum = 1 variant (C23: one digit = all of Q, four special primes) at N = 2^16:
    a spatial ct-pt MatMul (3 input ciphertexts of X in R^{128 x 768}, W in R^{768 x 256}, B = 16)
    through the generic ModUp / ModDown base conversions and the fused ModDown + rescale with
    nd = 5 moduli -- one output bit-exact against the oracle."""
    ctx, params = bert_dnum1["ctx"], bert_dnum1["params"]
    rng = np.random.default_rng(61)
    X = np.clip(rng.normal(0, 1, (L, D)), -4, 4)
    W = rng.normal(0, 0.04, (D, 256))
    plan_o = mm.plan_spatial(W, L, ctx.n, 16)
    plan_g = blb.MatmulPlan(params, L, D, 256, bsgs_B=16, level=4)
    assert plan_g.n_pt == plan_o.n_plaintexts
    key = bi.crypto_key(4, 62)
    okeys = O.keygen(ctx, key, plan_o.rotation_steps())
    gkeys, sk = blb.keygen(params, key, plan_g.rotation_steps())
    zs = mm.pack_spatial(X, ctx.n)
    enc_key = bi.crypto_key(5, 62)
    octs, gcts = [], []
    for t, z in enumerate(zs):
        octs.append(O.encrypt(ctx, enc_key, okeys.s_ntt, O.encode(ctx, z, DELTA, 4), 4, 50 + t, DELTA))
        gcts.append(blb.encrypt(params, sk, params.encode(torch.tensor(z), DELTA, 4), 4, enc_key, 50 + t, DELTA))
        assert np.array_equal(blb.to_numpy_u64(gcts[-1].data), octs[-1].data)
    gout = plan_g(gkeys, gcts, plan_g.encode_weights(W))
    (ref,) = mm.matmul_cp(ctx, okeys, octs, plan_o, out_ids=[0])
    assert same(gout[0], ref)
