"""Full-size parity (BASELINE configs 2/3 at N = 2^16, the launch configuration
bench.py times): the GPU computes every output ciphertext of the BERT-base QKV
(C11 + MHP) and out-projection (C12) MatMuls; the oracle recomputes sampled
output ciphertexts one by one and they must agree bit-exactly on every limb.
Slow (the oracle runs 2^16-point NTTs in u128 C on the host)."""
import numpy as np
import pytest
import torch

import blb_inputs as bi
import oracle as O
import oracle.matmul as mm

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

blb = pytest.importorskip("paper_2508_19525_b200")
from paper_2508_19525_b200 import packing  # noqa: E402


@pytest.fixture(scope="module")
def bert():
    P = bi.BERT
    pr = O.prime_chain(P.log_n, list(P.q_bits) + list(P.p_bits))
    return O.Ctx(P.log_n, pr[:5], pr[5:], P.dnum), blb.Params(P.log_n, pr[:5], pr[5:], P.dnum)


def run(octx, g, plan_o, plan_g, zs, W, sample):
    lvl, delta = 4, 2.0 ** 40
    key, ekey = bi.crypto_key(4, 2), bi.crypto_key(5, 2)
    steps = plan_g.rotation_steps()
    assert steps == plan_o.rotation_steps()
    okeys = O.keygen(octx, key, steps)
    gkeys, sk = blb.keygen(g, key, steps)
    octs, gcts = [], []
    for b, z in enumerate(zs):
        pt = O.encode(octx, z, delta, lvl)
        octs.append(O.encrypt(octx, ekey, okeys.s_ntt, pt, lvl, b, delta))
        gcts.append(blb.encrypt(g, sk, g.encode(torch.tensor(z), delta, lvl), lvl, ekey, b, delta))
        assert np.array_equal(blb.to_numpy_u64(gcts[-1].data), octs[-1].data)
    pts = plan_g.encode_weights(W)
    gout = plan_g(gkeys, gcts, pts)
    oout = mm.matmul_cp(octx, okeys, octs, plan_o, out_ids=sample)
    for o, ref in zip(sample, oout):
        assert gout[o].level == ref.level == lvl - 1 and gout[o].scale == ref.scale
        assert np.array_equal(blb.to_numpy_u64(gout[o].data), ref.data), o
    return gout, sk


def test_bert_qkv_sampled_outputs_bit_exact(bert):
    octx, g = bert
    A = bi.bert_attention_inputs()
    L, d, H = 128, 768, 12
    cm = blb.mhp_column_map(d, H, L, 16)
    qkv_map = cm + [d + c if c >= 0 else -1 for c in cm] + list(range(2 * d, 3 * d))
    W = np.concatenate([A["WQ"], A["WK"], A["WV"]], axis=1)
    plan_g = blb.MatmulPlan(g, L, d, 3 * d, col_map=qkv_map, bsgs_B=32, level=4)
    plan_o = mm.plan_spatial(W, L, octx.n, 32, col_map=qkv_map)
    assert (plan_g.n_pt, plan_g.n_rotations) == (plan_o.n_plaintexts, plan_o.n_rotations) == (8448, 170)
    zs = list(packing.spatial_slots(A["X"], octx.n))
    gout, sk = run(octx, g, plan_o, plan_g, zs, W, sample=[0, 10])
    # every output decodes to X W (float64) within the paper's MSE bound
    Y = np.concatenate([packing.spatial_unslots(g.decode(blb.decrypt(g, sk, o), o.scale).cpu().numpy()[None], L, 256)
                        for o in gout], axis=1)
    ref = A["X"] @ W
    full = np.zeros((L, len(qkv_map)))
    for v, src in enumerate(qkv_map):
        if src >= 0:
            full[:, v] = ref[:, src]
    assert float(((Y[:, :len(qkv_map)] - full) ** 2).mean()) <= 1e-11


def test_bert_oproj_diagonal_sampled_output_bit_exact(bert):
    octx, g = bert
    F = bi.bert_ffn_inputs()
    L, d, H = 128, 768, 12
    plan_g = blb.MatmulPlan(g, L, d, d, packing=blb.PACK_DIAGONAL, heads=H, bsgs_B=16, level=4)
    plan_o = mm.plan_diagonal(F["WO"], H, L, octx.n, 16)
    assert (plan_g.n_pt, plan_g.n_rotations) == (plan_o.n_plaintexts, plan_o.n_rotations) == (2304, 90)
    zs = list(packing.diagonal_slots(F["Att"], octx.n))
    run(octx, g, plan_o, plan_g, zs, F["WO"], sample=[2])


def test_bert_size_qk_bit_exact(bert):
    """Row a7 at N = 2^16, L = 128 (16 heads of d_h = 8: g = 16, J = 1, B = 16, G = 8): the
    double-hoisted stage 1, relinearisation, step-3 rotations and deferred giant step on the
    fused N = 2^16 kernels, bit-exact against the oracle."""
    import oracle.matmul_cc as cc
    octx, g = bert
    L, H, dh = 128, 16, 8
    rng = np.random.default_rng(5)
    Q, K = rng.uniform(-1, 1, (H, L, dh)), rng.uniform(-1, 1, (H, L, dh))
    plan_o = cc.plan_qk(L, H, dh, octx.n)
    plan_g = blb.QKPlan(g, L, H, dh, level=3)
    assert plan_g.rotation_steps() == plan_o.rotation_steps()
    key, ekey = bi.crypto_key(4, 3), bi.crypto_key(5, 3)
    steps = plan_g.rotation_steps()
    okeys = O.keygen(octx, key, steps, relin=True)
    gkeys, sk = blb.keygen(g, key, steps, relin=True)
    lvl, delta = 3, 2.0 ** 40
    oq, ok, gq, gk = [], [], [], []
    for j, (zq, zk) in enumerate(zip(cc.pack_mhp(Q, plan_o), cc.pack_mhp(K, plan_o))):
        for z, cid, ol, gl in ((zq, j, oq, gq), (zk, 10 + j, ok, gk)):
            pt = O.encode(octx, z, delta, lvl)
            ol.append(O.encrypt(octx, ekey, okeys.s_ntt, pt, lvl, cid, delta))
            gl.append(blb.encrypt(g, sk, blb.from_numpy_u64(pt), lvl, ekey, cid, delta))
    gout = plan_g(gkeys, gq, gk, plan_g.encode_masks())
    oout = cc.qk_encrypted(octx, okeys, oq, ok, plan_o)
    for a, b in zip(gout, oout):
        assert a.scale == b.scale and np.array_equal(blb.to_numpy_u64(a.data), b.data)
