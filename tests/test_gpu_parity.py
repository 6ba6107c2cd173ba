"""GPU parity: the sm_100a library (through its C ABI) against the CPU oracle,
bit-exact on every RNS limb for the same seeded inputs (BASELINE.json
north_star), and decoded outputs within 2^-20 relative error.

Sizes: the tiny ring (N = 32) for edge cases, the toy preset (N = 2^12, config
1) for every operation, a 4-limb alpha = 2 preset (N = 2^10) for multi-prime
digits, and the BERT preset (N = 2^16) for the NTT / encode / rotation at full
size.  Full-size MatMul parity on sampled outputs lives in test_gpu_bert.py."""
import numpy as np
import pytest
import torch

import blb_inputs as bi
import oracle as O
import oracle.matmul as mm

pytestmark = pytest.mark.gpu

blb = pytest.importorskip("paper_2508_19525_b200")


def u64(t):
    return blb.to_numpy_u64(t)


def dev(a):
    return blb.from_numpy_u64(a)


class Pair:
    def __init__(self, preset):
        primes = O.prime_chain(preset.log_n, list(preset.q_bits) + list(preset.p_bits))
        k = len(preset.q_bits)
        self.preset = preset
        self.o = O.Ctx(preset.log_n, primes[:k], primes[k:], preset.dnum)
        self.g = blb.Params(preset.log_n, primes[:k], primes[k:], preset.dnum)
        self.N, self.n, self.K = self.o.N, self.o.n, self.o.K


@pytest.fixture(scope="module")
def tiny():
    return Pair(bi.TINY)


@pytest.fixture(scope="module")
def toy():
    return Pair(bi.TOY)


@pytest.fixture(scope="module")
def mid():
    return Pair(bi.MID)


@pytest.fixture(scope="module")
def bert():
    return Pair(bi.BERT)


@pytest.fixture(scope="module")
def f2():
    """N = 2^15 (the row-f2 Table-6 block-3 preset): the 128 x 256 two-pass NTT kernels."""
    return Pair(bi.F2)


@pytest.fixture(scope="module")
def bert_dnum1():
    return Pair(bi.BERT_DNUM1)


def rand_limbs(pair, shape_polys, limbs, seed):
    rng = np.random.default_rng(seed)
    out = np.empty((shape_polys, len(limbs), pair.N), dtype=np.uint64)
    for p in range(shape_polys):
        for j, li in enumerate(limbs):
            out[p, j] = rng.integers(0, pair.o.mods[li], pair.N, dtype=np.uint64)
    return out


# ---------------------------------------------------------------- a0 / a1
@pytest.mark.parametrize("name", ["tiny", "toy", "mid", "bert"])
def test_params_psi_match(name, request):
    pair = request.getfixturevalue(name)
    assert pair.g.moduli == pair.o.mods
    assert pair.g.psi == pair.o.psi


@pytest.mark.parametrize("name", ["tiny", "toy", "mid", "f2", "bert"])
def test_ntt_intt_bit_exact(name, request):
    pair = request.getfixturevalue(name)
    limbs = list(range(len(pair.o.mods)))
    a = rand_limbs(pair, 3, limbs, seed=11)
    t = dev(a)
    pair.g.ntt(t, limbs)
    ref = np.stack([pair.o.ntt(a[p], limbs) for p in range(3)])
    assert np.array_equal(u64(t), ref)
    pair.g.intt(t, limbs)
    assert np.array_equal(u64(t), a)


@pytest.mark.parametrize("name", ["f2", "bert"])
def test_ntt_edge_values(name, request):
    """all-zero, all q-1 and delta inputs at N = 2^15 / 2^16 (max residues exercise the lazy ranges),
    forward and back."""
    pair = request.getfixturevalue(name)
    limbs = list(range(len(pair.o.mods)))
    a = np.zeros((3, len(limbs), pair.N), dtype=np.uint64)
    for j, m in enumerate(pair.o.mods):
        a[1, j] = m - 1
        a[2, j, 0] = m - 1
        a[2, j, -1] = 1
    t = dev(a)
    pair.g.ntt(t, limbs)
    assert np.array_equal(u64(t), np.stack([pair.o.ntt(a[p], limbs) for p in range(3)]))
    pair.g.intt(t, limbs)
    assert np.array_equal(u64(t), a)


# ---------------------------------------------------------------- encode
@pytest.mark.parametrize("name", ["tiny", "toy", "bert"])
def test_encode_bit_exact(name, request):
    pair = request.getfixturevalue(name)
    rng = np.random.default_rng(5)
    zs = [rng.uniform(-1, 1, pair.n), rng.normal(0, 0.04, pair.n) * 3, np.zeros(pair.n), np.full(pair.n, 0.3125)]
    scale = float(pair.o.q[-1]) if name != "tiny" else 2.0 ** 30
    lvl = pair.K - 1
    got = u64(pair.g.encode(torch.tensor(np.stack(zs)), scale, lvl))
    for p, z in enumerate(zs):
        assert np.array_equal(got[p], O.encode(pair.o, z, scale, lvl)), p


def test_encode_overflow(toy):
    with pytest.raises(blb.BLBError) as e:
        toy.g.encode(torch.full((toy.n,), 8.0, dtype=torch.float64), 2.0 ** 52, 2)
    assert e.value.status == 7


def test_decode_close(toy):
    z = np.random.default_rng(6).uniform(-1, 1, toy.n)
    pt = O.encode(toy.o, z, 2.0 ** 40, 2)
    got = toy.g.decode(dev(pt), 2.0 ** 40).cpu().numpy()
    ref = O.decode(toy.o, pt, 2.0 ** 40)
    assert np.abs(got - ref).max() <= 2 ** -20 * max(1.0, np.abs(ref).max())


# ---------------------------------------------------------------- keys / enc
@pytest.mark.parametrize("name", ["tiny", "toy", "mid"])
def test_keygen_and_encrypt_bit_exact(name, request):
    pair = request.getfixturevalue(name)
    key = bi.crypto_key(4, 7)
    steps = [1, 3, -2]
    okeys = O.keygen(pair.o, key, steps, relin=True)
    gkeys, sk = blb.keygen(pair.g, key, steps, relin=True)
    assert np.array_equal(u64(sk), okeys.s_ntt)
    # keys are device-resident in the library: re-derive through a rotation of a known ciphertext
    lvl = pair.K - 1
    z = np.random.default_rng(1).uniform(-1, 1, pair.n)
    scale = 2.0 ** 30
    pt = O.encode(pair.o, z, scale, lvl)
    oct_ = O.encrypt(pair.o, bi.crypto_key(5, 7), okeys.s_ntt, pt, lvl, 42, scale)
    gct = blb.encrypt(pair.g, sk, dev(pt), lvl, bi.crypto_key(5, 7), 42, scale)
    assert np.array_equal(u64(gct.data), oct_.data)
    assert np.array_equal(u64(blb.decrypt(pair.g, sk, gct)), O.decrypt(pair.o, okeys.s_ntt, oct_))
    for s in steps:
        assert gkeys.has(pair.g.galois(s))
        ro = O.rotate(pair.o, oct_, okeys, s)
        rg = blb.rotate(pair.g, gkeys, gct, s)
        assert np.array_equal(u64(rg.data), ro.data), s


def test_oracle_keys_loaded_into_library(mid):
    """blb_keys_add with client-made (oracle) keys gives the same rotation."""
    key = bi.crypto_key(8, 3)
    okeys = O.keygen(mid.o, key, [5])
    g = mid.o.galois(5)
    keys = blb.Keys(mid.g)
    keys.add(g, dev(okeys.rot[g]))
    lvl = 2
    z = np.random.default_rng(2).uniform(-1, 1, mid.n)
    ct = O.encrypt(mid.o, key, okeys.s_ntt, O.encode(mid.o, z, 2.0 ** 30, lvl), lvl, 3, 2.0 ** 30)
    gct = blb.Ciphertext(dev(ct.data), lvl, ct.scale)
    assert np.array_equal(u64(blb.rotate(mid.g, keys, gct, 5).data), O.rotate(mid.o, ct, okeys, 5).data)
    with pytest.raises(blb.BLBError) as e:
        blb.rotate(mid.g, keys, gct, 6)
    assert e.value.status == 3


@pytest.mark.parametrize("name", ["toy", "mid"])
def test_rotation_all_levels_bit_exact(name, request):
    pair = request.getfixturevalue(name)
    key = bi.crypto_key(9, 9)
    okeys = O.keygen(pair.o, key, [7])
    gkeys, sk = blb.keygen(pair.g, key, [7])
    for lvl in range(pair.K):
        data = rand_limbs(pair, 2, list(range(lvl + 1)), seed=lvl)
        ct = O.Ct(data, lvl, 1.0)
        got = blb.rotate(pair.g, gkeys, blb.Ciphertext(dev(data), lvl, 1.0), 7)
        assert np.array_equal(u64(got.data), O.rotate(pair.o, ct, okeys, 7).data), lvl


@pytest.mark.parametrize("name", ["tiny", "toy", "mid", "bert"])
def test_rescale_bit_exact(name, request):
    pair = request.getfixturevalue(name)
    for lvl in range(1, pair.K):
        data = rand_limbs(pair, 2, list(range(lvl + 1)), seed=100 + lvl)
        got = blb.rescale(pair.g, blb.Ciphertext(dev(data), lvl, 2.0 ** 80))
        ref = O.rescale(pair.o, O.Ct(data, lvl, 2.0 ** 80))
        assert got.level == ref.level and got.scale == ref.scale
        assert np.array_equal(u64(got.data), ref.data), lvl


def test_mul_pt_add_bit_exact(toy):
    a = rand_limbs(toy, 2, [0, 1, 2], 1)
    b = rand_limbs(toy, 2, [0, 1, 2], 2)
    pt = rand_limbs(toy, 1, [0, 1, 2], 3)[0]
    ga, gb = blb.Ciphertext(dev(a), 2, 1.0), blb.Ciphertext(dev(b), 2, 1.0)
    got = blb.mul_pt(toy.g, ga, dev(pt), 3.0)
    assert np.array_equal(u64(got.data), O.mul_pt(toy.o, O.Ct(a, 2, 1.0), pt, 3.0).data) and got.scale == 3.0
    got = blb.add(toy.g, ga, gb)
    assert np.array_equal(u64(got.data), O.add(toy.o, O.Ct(a, 2, 1.0), O.Ct(b, 2, 1.0)).data)


@pytest.mark.parametrize("name", ["toy", "bert"])
def test_mask_bit_exact(name, request):
    pair = request.getfixturevalue(name)
    key = bytes(range(32))
    cts = [rand_limbs(pair, 2, list(range(lv + 1)), 50 + i) for i, lv in enumerate([1, 1, 1])]
    gm, gs = blb.ckks_to_mpc(pair.g, [blb.Ciphertext(dev(c), 1, 1.0) for c in cts], key, 7)
    gm, gs = u64(gm), u64(gs)
    for t, c in enumerate(cts):
        om, osh = O.mask(pair.o, O.Ct(c, 1, 1.0), key, 7 + t)
        assert np.array_equal(gm[t], om) and np.array_equal(gs[t], osh)


# ---------------------------------------------------------------- MatMul (C11 / C12)
def run_both(pair, plan_o, plan_g, zs, W, key_seed=4, delta=2.0 ** 40, lvl=None, out_first=0, out_count=None):
    lvl = pair.K - 1 if lvl is None else lvl
    key, ekey = bi.crypto_key(key_seed, 1), bi.crypto_key(5, 1)
    steps = plan_g.rotation_steps()
    assert steps == plan_o.rotation_steps()
    okeys = O.keygen(pair.o, key, steps)
    gkeys, sk = blb.keygen(pair.g, key, steps)
    octs, gcts = [], []
    for b, z in enumerate(zs):
        pt = O.encode(pair.o, z, delta, lvl)
        octs.append(O.encrypt(pair.o, ekey, okeys.s_ntt, pt, lvl, b, delta))
        gpt = pair.g.encode(torch.tensor(z), delta, lvl)
        gcts.append(blb.encrypt(pair.g, sk, gpt, lvl, ekey, b, delta))
        assert np.array_equal(u64(gcts[-1].data), octs[-1].data)
    out_count = plan_g.n_out - out_first if out_count is None else out_count
    pts = plan_g.encode_weights(W, out_first, out_count)
    gout = plan_g(gkeys, gcts, pts, out_first, out_count)
    oout = mm.matmul_cp(pair.o, okeys, octs, plan_o, out_ids=range(out_first, out_first + out_count))
    return okeys, sk, oout, gout


def test_toy_config_matmul_and_mask_bit_exact(toy):
    d = bi.toy_inputs()
    plan_o = mm.plan_spatial(d["W"], 16, toy.n, 16)
    plan_g = blb.MatmulPlan(toy.g, 16, 16, 16, bsgs_B=16)
    assert (plan_g.n_pt, plan_g.n_rotations) == (plan_o.n_plaintexts, plan_o.n_rotations) == (31, 16)
    from paper_2508_19525_b200 import packing
    zs = list(packing.spatial_slots(d["X"], toy.n))
    okeys, sk, oout, gout = run_both(toy, plan_o, plan_g, zs, d["W"])
    assert gout[0].level == oout[0].level == 1 and gout[0].scale == oout[0].scale == 2.0 ** 40
    assert np.array_equal(u64(gout[0].data), oout[0].data)
    # decoded parity within 2^-20 relative, and accuracy vs X W
    dec_g = toy.g.decode(blb.decrypt(toy.g, sk, gout[0]), gout[0].scale).cpu().numpy()
    dec_o = O.decode(toy.o, O.decrypt(toy.o, okeys.s_ntt, oout[0]), oout[0].scale)
    assert np.abs(dec_g - dec_o).max() <= 2 ** -20 * np.abs(dec_o).max()
    Y = packing.spatial_unslots(dec_g[None], 16, 16)
    assert float(((Y - d["X"] @ d["W"]) ** 2).mean()) <= 1e-11
    # CKKS -> MPC mask of the result (row a8)
    gm, gs = blb.ckks_to_mpc(toy.g, gout, d["mask_key"], 0)
    om, osh = O.mask(toy.o, oout[0], d["mask_key"], 0)
    assert np.array_equal(u64(gm)[0], om) and np.array_equal(u64(gs)[0], osh)


@pytest.mark.parametrize("L,D,Dout,B", [(16, 200, 136, 8), (32, 64, 300, 4)])
def test_spatial_matmul_ragged_bit_exact(toy, L, D, Dout, B):
    X = bi.uniform(70 + D, (L, D), -1, 1)
    W = bi.normal(71 + D, (D, Dout), 0.1)
    plan_o = mm.plan_spatial(W, L, toy.n, B)
    plan_g = blb.MatmulPlan(toy.g, L, D, Dout, bsgs_B=B)
    assert (plan_g.n_in, plan_g.n_out, plan_g.n_pt) == (plan_o.n_in, plan_o.n_out, plan_o.n_plaintexts)
    from paper_2508_19525_b200 import packing
    zs = list(packing.spatial_slots(X, toy.n))
    _, _, oout, gout = run_both(toy, plan_o, plan_g, zs, W)
    for a, b in zip(gout, oout):
        assert np.array_equal(u64(a.data), b.data)


def test_mhp_matmul_output_slice_bit_exact(toy):
    """MHP-reordered output columns and an output slice (multi-GPU sharding unit)."""
    L, d, H = 16, 64, 4
    X = bi.uniform(80, (L, d), -1, 1)
    W = bi.normal(81, (d, d), 0.1)
    cmap = blb.mhp_column_map(d, H, L, toy.o.log_n)
    assert cmap == mm.mhp_column_map(d, H, L, toy.n)
    plan_o = mm.plan_spatial(W, L, toy.n, 16, col_map=cmap)
    plan_g = blb.MatmulPlan(toy.g, L, d, d, col_map=cmap, bsgs_B=16)
    from paper_2508_19525_b200 import packing
    zs = list(packing.spatial_slots(X, toy.n))
    _, _, oout, gout = run_both(toy, plan_o, plan_g, zs, W, out_first=0, out_count=plan_g.n_out)
    for a, b in zip(gout, oout):
        assert np.array_equal(u64(a.data), b.data)


def test_diagonal_matmul_bit_exact(toy):
    L, H, dh, Dout = 16, 4, 16, 144
    Att = bi.normal(62, (H, L, dh), 1.0)
    WO = bi.normal(63, (H * dh, Dout), 0.05)
    plan_o = mm.plan_diagonal(WO, H, L, toy.n, 16)
    plan_g = blb.MatmulPlan(toy.g, L, H * dh, Dout, packing=blb.PACK_DIAGONAL, heads=H, bsgs_B=16)
    assert (plan_g.n_pt, plan_g.n_rotations) == (plan_o.n_plaintexts, plan_o.n_rotations)
    from paper_2508_19525_b200 import packing
    zs = list(packing.diagonal_slots(Att, toy.n))
    _, _, oout, gout = run_both(toy, plan_o, plan_g, zs, WO, out_first=1, out_count=1)
    assert np.array_equal(u64(gout[0].data), oout[0].data)


def test_matmul_alpha2_digits_bit_exact(mid):
    L, D, Dout = 8, 40, 40
    X = bi.uniform(90, (L, D), -1, 1)
    W = bi.normal(91, (D, Dout), 0.1)
    plan_o = mm.plan_spatial(W, L, mid.n, 8)
    plan_g = blb.MatmulPlan(mid.g, L, D, Dout, bsgs_B=8)
    from paper_2508_19525_b200 import packing
    zs = list(packing.spatial_slots(X, mid.n))
    _, _, oout, gout = run_both(mid, plan_o, plan_g, zs, W, delta=2.0 ** 36)
    for a, b in zip(gout, oout):
        assert np.array_equal(u64(a.data), b.data)


def test_matmul_errors(toy):
    plan_g = blb.MatmulPlan(toy.g, 16, 16, 16, bsgs_B=16)
    keys = blb.Keys(toy.g)
    ct = blb.Ciphertext.empty(toy.g, 2, 1.0)
    pts = plan_g.encode_weights(np.eye(16))
    with pytest.raises(blb.BLBError) as e:
        plan_g(keys, [ct], pts)
    assert e.value.status == 3  # missing keys
    with pytest.raises(blb.BLBError) as e:
        blb.MatmulPlan(toy.g, 15, 16, 16)
    assert e.value.status == 6


# ---------------------------------------------------------------- ct-ct Q K^T (row a7)
@pytest.fixture(scope="module")
def qktoy():
    return Pair(bi.QKTOY)


@pytest.mark.parametrize("H,L,dh,B", [(4, 32, 32, 0), (3, 32, 16, 0), (2, 32, 32, 32), (4, 32, 32, 32)])
def test_qk_ct_ct_bit_exact(qktoy, H, L, dh, B):
    import oracle.matmul_cc as cc
    d = bi.qk_toy_inputs(H, L, dh)
    plan_o = cc.plan_qk(L, H, dh, qktoy.n, B or None)
    plan_g = blb.QKPlan(qktoy.g, L, H, dh, bsgs_B=B, level=3)
    assert plan_g.rotation_steps() == plan_o.rotation_steps()
    assert (plan_g.J, plan_g.n_out, plan_g.n_rotations) == (plan_o.J, plan_o.n_out, plan_o.counts()["rotations"])
    steps = plan_g.rotation_steps()
    okeys = O.keygen(qktoy.o, d["keys_key"], steps, relin=True)
    gkeys, sk = blb.keygen(qktoy.g, d["keys_key"], steps, relin=True)
    lvl, delta = 3, 2.0 ** 40
    oq, ok, gq, gk = [], [], [], []
    for j, (zq, zk) in enumerate(zip(cc.pack_mhp(d["Q"], plan_o), cc.pack_mhp(d["K"], plan_o))):
        for z, cid, ol, gl in ((zq, j, oq, gq), (zk, 100 + j, ok, gk)):
            pt = O.encode(qktoy.o, z, delta, lvl)
            ol.append(O.encrypt(qktoy.o, d["enc_key"], okeys.s_ntt, pt, lvl, cid, delta))
            gl.append(blb.encrypt(qktoy.g, sk, dev(pt), lvl, d["enc_key"], cid, delta))
    masks = plan_g.encode_masks()
    gout = plan_g(gkeys, gq, gk, masks)
    oout = cc.qk_encrypted(qktoy.o, okeys, oq, ok, plan_o)
    assert len(gout) == len(oout)
    for a, b in zip(gout, oout):
        assert a.level == b.level == 0 and a.scale == b.scale
        assert np.array_equal(u64(a.data), b.data)
    dec = [qktoy.g.decode(blb.decrypt(qktoy.g, sk, o), o.scale).cpu().numpy() for o in gout]
    C = cc.unpack_diag(dec, plan_o)
    ref = np.einsum("hik,hjk->hij", d["Q"], d["K"])
    assert float(((C - ref) ** 2).mean()) <= 1e-11


def test_softmax_v_wo_chain_bit_exact(qktoy):
    """Row f1: Softmax x V_h (C13 with d_h zero-padded to L) -> dense-diagonal collapse
     -> diagonal ct-pt W_O with MHP-padded rows (C12) at level 1."""
    import oracle.matmul_cc as cc
    L, H, n = 32, 4, qktoy.n
    dh = L // 2
    rng = np.random.default_rng(7)
    S = rng.uniform(0, 1.0 / L, size=(H, L, L))
    V = rng.normal(0, 1, size=(H, L, dh))
    WO = rng.normal(0, 0.1, size=(H * dh, 48))
    p = cc.plan_sv(L, H, n)
    A, Kop = cc.sv_operands(S, V)
    key, ekey = bi.crypto_key(4, 77), bi.crypto_key(5, 77)
    qk_g = blb.QKPlan(qktoy.g, L, H, L, level=4)
    WOp = cc.pad_heads_rows(WO, H, p.Hp)
    diag_g = blb.MatmulPlan(qktoy.g, L, p.Hp * dh, 48, packing=blb.PACK_DIAGONAL, heads=p.Hp, bsgs_B=16, level=1)
    diag_o = mm.plan_diagonal(WOp, p.Hp, L, n, 16)
    steps = sorted(set(qk_g.rotation_steps()) | set(diag_g.rotation_steps()))
    okeys = O.keygen(qktoy.o, key, steps, relin=True)
    gkeys, sk = blb.keygen(qktoy.g, key, steps, relin=True)
    lvl, delta = 4, 2.0 ** 40
    oa, ok, ga, gk = [], [], [], []
    for j, (za, zk) in enumerate(zip(cc.pack_mhp(A, p), cc.pack_mhp(Kop, p))):
        for z, cid, ol, gl in ((za, j, oa, ga), (zk, 50 + j, ok, gk)):
            pt = O.encode(qktoy.o, z, delta, lvl)
            ol.append(O.encrypt(qktoy.o, ekey, okeys.s_ntt, pt, lvl, cid, delta))
            gl.append(blb.encrypt(qktoy.g, sk, dev(pt), lvl, ekey, cid, delta))
    # oracle chain
    oout = cc.qk_encrypted(qktoy.o, okeys, oa, ok, p)
    odense = cc.collapse_dense(oout, p, dh, add_fn=lambda a, b: O.add(qktoy.o, a, b))
    ofin = mm.matmul_cp(qktoy.o, okeys, odense, diag_o)
    # GPU chain
    gout = qk_g(gkeys, ga, gk, qk_g.encode_masks())
    half = len(gout) // 2
    gdense = [blb.add(qktoy.g, gout[o], gout[o + half]) for o in range(half)]
    gfin = diag_g(gkeys, gdense, diag_g.encode_weights(WOp))
    for a, b in zip(gdense, odense):
        assert np.array_equal(u64(a.data), b.data)
    for a, b in zip(gfin, ofin):
        assert a.level == b.level == 0 and a.scale == b.scale
        assert np.array_equal(u64(a.data), b.data)
    from paper_2508_19525_b200 import packing
    Y = packing.spatial_unslots(np.stack([qktoy.g.decode(blb.decrypt(qktoy.g, sk, o), o.scale).cpu().numpy()
                                          for o in gfin]), L, 48)
    Att = np.concatenate([S[h] @ V[h] for h in range(H)], axis=1)
    assert float(((Y - Att @ WO) ** 2).mean()) <= 1e-11


# ---------------------------------------------------------------- row f2
def test_f2_ops_bit_exact(qktoy):
    key = bi.crypto_key(4, 88)
    L, D = 32, 8
    steps = [L, 2 * L, 4 * L, -L, -2 * L, -4 * L]
    okeys = O.keygen(qktoy.o, key, steps, relin=True)
    gkeys, sk = blb.keygen(qktoy.g, key, steps, relin=True)
    lvl = 4
    a = rand_limbs(qktoy, 2, list(range(lvl + 1)), 1)
    b = rand_limbs(qktoy, 2, list(range(lvl + 1)), 2)
    oa, ob = O.Ct(a, lvl, 2.0 ** 40), O.Ct(b, lvl, 2.0 ** 40)
    ga, gb = blb.Ciphertext(dev(a), lvl, 2.0 ** 40), blb.Ciphertext(dev(b), lvl, 2.0 ** 40)
    r = blb.mul_relin(qktoy.g, gkeys, ga, gb)
    assert np.array_equal(u64(r.data), O.mul_relin(qktoy.o, oa, ob, okeys).data) and r.scale == 2.0 ** 80
    for bc in (False, True):
        r = blb.rotate_sum(qktoy.g, gkeys, ga, L, D, broadcast=bc)
        assert np.array_equal(u64(r.data), O.rotate_sum(qktoy.o, oa, okeys, L, D, broadcast=bc).data)


def test_f2_preset_keyswitch_bit_exact(f2):
    """N = 2^15 (row f2's Table-6 block-3 preset, dnum = 8): rotations (fused ModUp / ModDown NTT passes
    of the 2^15 kernels, bulk key switch with beta up to 8) and the relinearised product (fused
    ModDown + rescale, C17), bit-exact against the oracle."""
    key = bi.crypto_key(9, 15)
    okeys = O.keygen(f2.o, key, [5], relin=True)
    gkeys, sk = blb.keygen(f2.g, key, [5], relin=True)
    for lvl in (f2.K - 1, 4, 1):
        data = rand_limbs(f2, 2, list(range(lvl + 1)), seed=30 + lvl)
        got = blb.rotate(f2.g, gkeys, blb.Ciphertext(dev(data), lvl, 1.0), 5)
        assert np.array_equal(u64(got.data), O.rotate(f2.o, O.Ct(data, lvl, 1.0), okeys, 5).data), lvl
    lvl = f2.K - 1
    a = rand_limbs(f2, 2, list(range(lvl + 1)), 41)
    b = rand_limbs(f2, 2, list(range(lvl + 1)), 42)
    r = blb.mul_relin(f2.g, gkeys, blb.Ciphertext(dev(a), lvl, 2.0 ** 40), blb.Ciphertext(dev(b), lvl, 2.0 ** 40))
    ref = O.mul_relin(f2.o, O.Ct(a, lvl, 2.0 ** 40), O.Ct(b, lvl, 2.0 ** 40), okeys)
    assert np.array_equal(u64(r.data), ref.data)


@pytest.mark.parametrize("name", ["bert", "bert_dnum1"])
def test_bert_size_keyswitch_bit_exact(name, request):
    """N = 2^16: rotation at every level, relinearised product, rotate-and-sum -- bit-exact against
    the oracle; dnum = 5 takes the fused ModUp / ModDown NTT path, the dnum = 1 variant (C23) the
    generic base conversions with four special primes."""
    bert = request.getfixturevalue(name)
    key = bi.crypto_key(4, 99)
    steps = [128, -256, 5]
    okeys = O.keygen(bert.o, key, steps, relin=True)
    gkeys, sk = blb.keygen(bert.g, key, steps, relin=True)
    for lvl in (4, 2, 0):
        data = rand_limbs(bert, 2, list(range(lvl + 1)), 40 + lvl)
        oc, gc = O.Ct(data, lvl, 2.0 ** 40), blb.Ciphertext(dev(data), lvl, 2.0 ** 40)
        for s in steps:
            assert np.array_equal(u64(blb.rotate(bert.g, gkeys, gc, s).data), O.rotate(bert.o, oc, okeys, s).data), (lvl, s)
        assert np.array_equal(u64(blb.mul_relin(bert.g, gkeys, gc, gc).data), O.mul_relin(bert.o, oc, oc, okeys).data)
    data = rand_limbs(bert, 2, list(range(5)), 7)
    oc, gc = O.Ct(data, 4, 1.0), blb.Ciphertext(dev(data), 4, 1.0)
    assert np.array_equal(u64(blb.rotate_sum(bert.g, gkeys, gc, 128, 2).data), O.rotate_sum(bert.o, oc, okeys, 128, 2).data)


def test_matmul_long_mac_fold_bit_exact(toy):
    """192 products per output (12 inputs x B = 16) exceed the 128-bit lazy bound for the
    60-bit q_0 limb: the MAC folds its accumulator every 64 products."""
    L, D, Dout = 16, 1536, 16
    X = bi.uniform(95, (L, D), -1, 1)
    W = bi.normal(96, (D, Dout), 0.02)
    plan_o = mm.plan_spatial(W, L, toy.n, 16)
    plan_g = blb.MatmulPlan(toy.g, L, D, Dout, bsgs_B=16)
    assert plan_g.n_in == 12 and plan_g.n_pt == plan_o.n_plaintexts
    from paper_2508_19525_b200 import packing
    zs = list(packing.spatial_slots(X, toy.n))
    _, _, oout, gout = run_both(toy, plan_o, plan_g, zs, W)
    assert np.array_equal(u64(gout[0].data), oout[0].data)


def test_matmul_fp64_fold_bit_exact(toy):
    """640 products per output (40 inputs x B = 16): the FP64-pipe accumulator of the 40-bit limbs
    folds every 512 products (AccF64), the 60-bit limb every 64 (Acc128)."""
    L, D, Dout = 16, 5120, 16
    X = bi.uniform(97, (L, D), -1, 1)
    W = bi.normal(98, (D, Dout), 0.01)
    plan_o = mm.plan_spatial(W, L, toy.n, 16)
    plan_g = blb.MatmulPlan(toy.g, L, D, Dout, bsgs_B=16)
    assert plan_g.n_in == 40 and plan_g.n_pt == plan_o.n_plaintexts
    from paper_2508_19525_b200 import packing
    zs = list(packing.spatial_slots(X, toy.n))
    _, _, oout, gout = run_both(toy, plan_o, plan_g, zs, W)
    assert np.array_equal(u64(gout[0].data), oout[0].data)


# ---------------------------------------------------------------- row f3: MPC -> CKKS ingest
@pytest.mark.parametrize("name,w", [("toy", 64), ("toy", 41), ("bert", 64)])
def test_mpc_to_ckks_bit_exact(name, w, request):
    pair = request.getfixturevalue(name)
    rng = np.random.default_rng(60 + w)
    lvl = pair.K - 1
    x = rng.integers(0, 2 ** min(w, 63), pair.N, dtype=np.uint64)
    if w == 64:
        x |= rng.integers(0, 2, pair.N, dtype=np.uint64) << np.uint64(63)
    x[:4] = [0, 1, (2 ** w - 1) if w < 64 else 2 ** 64 - 1, 2 ** (w - 1)]
    for sub in (False, True):
        got = u64(blb.share_to_rns(pair.g, dev(x), w, sub, lvl))
        assert np.array_equal(got, O.share_to_rns(pair.o, x, w, sub, lvl))
    c = rand_limbs(pair, 2, list(range(lvl + 1)), 61)
    gct = blb.Ciphertext(dev(c), lvl, 2.0 ** 40)
    blb.mpc_to_ckks(pair.g, gct, dev(x), w)
    want = O.mpc_to_ckks(pair.o, O.Ct(c, lvl, 2.0 ** 40), x, w)
    assert np.array_equal(u64(gct.data), want.data)


@pytest.mark.parametrize("name", ["toy", "bert"])
def test_share_decode_bit_exact(name, request):
    """Row f3 local fixed-point Decode (C18): bit-exact over Z_{2^128} for a uniform share and
    for a small signed message, incl. the extreme words."""
    pair = request.getfixturevalue(name)
    rng = np.random.default_rng(70)
    x = rng.integers(0, 2 ** 63, (pair.N, 2), dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, (pair.N, 2),
                                                                                            dtype=np.uint64)
    x[0] = [0, 0]
    x[1] = [2 ** 64 - 1, 2 ** 64 - 1]
    x[2] = [0, 2 ** 63]
    z = rng.uniform(-1, 1, pair.n)
    m = O.int_to_u128([int(v) for v in O.encode_coeffs(pair.o, z, 2.0 ** 30)])
    for xs, ft, s_out in ((x, 30, 18), (m, 30, 18), (m, 40, 0), (x, 52, 126)):
        got = u64(blb.share_decode(pair.g, dev(xs), ft, s_out))
        assert np.array_equal(got, O.share_decode(pair.o, xs, ft, s_out))


@pytest.mark.parametrize("name", ["toy", "bert"])
def test_share_encode_bit_exact(name, request):
    """Row f3 local fixed-point Encode (Alg. 2 line 1, C20): bit-exact over Z_{2^128} for a uniform
    share, a fixed-point message, and the extreme words; the GPU encode then GPU decode round trip
    returns Delta z."""
    pair = request.getfixturevalue(name)
    rng = np.random.default_rng(71)
    y = rng.integers(0, 2 ** 63, (pair.n, 2), dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, (pair.n, 2),
                                                                                            dtype=np.uint64)
    y[0] = [0, 0]
    y[1] = [2 ** 64 - 1, 2 ** 64 - 1]
    y[2] = [0, 2 ** 63]
    z = rng.uniform(-1, 1, pair.n)
    f = 50
    m = O.int_to_u128([int(round(v * 2.0 ** f)) for v in z])
    s_out = f + pair.o.log_n - 40
    for ys, ft, so in ((y, 50, s_out), (m, 50, s_out), (m, 30, 0), (y, 52, 126)):
        got = u64(blb.share_encode(pair.g, dev(ys), ft, so))
        assert np.array_equal(got, O.share_encode(pair.o, ys, ft, so))
    back = O.u128_to_int(u64(blb.share_decode(pair.g, blb.share_encode(pair.g, dev(m), 50, s_out), 30, 0)))
    # the decode's 2^-30 twiddles over log N stages bound the error (< 2^-22 of Delta at N = 2^16)
    assert np.abs(np.array(back, dtype=np.float64) - z * 2.0 ** 40).max() < 2.0 ** 18


# ---------------------------------------------------------------- error behaviour (include/blb.h)
def test_api_error_statuses(toy):
    """Each documented error status is raised before any launch, and degenerate calls are no-ops."""
    g = toy.g
    a = blb.Ciphertext(dev(rand_limbs(toy, 2, [0, 1, 2], 80)), 2, 2.0 ** 40)
    b1 = blb.Ciphertext(dev(rand_limbs(toy, 2, [0, 1], 81)), 1, 2.0 ** 40)
    with pytest.raises(blb.BLBError) as e:          # level mismatch
        blb.add(g, a, b1)
    assert e.value.status == 4
    b2 = blb.Ciphertext(dev(rand_limbs(toy, 2, [0, 1, 2], 82)), 2, 2.0 ** 43)
    with pytest.raises(blb.BLBError) as e:          # scale mismatch > 1 bit
        blb.add(g, a, b2)
    assert e.value.status == 5
    z0 = blb.Ciphertext(dev(rand_limbs(toy, 2, [0], 83)), 0, 2.0 ** 40)
    with pytest.raises(blb.BLBError):               # rescale below level 0
        blb.rescale(g, z0)
    keys = blb.Keys(g)
    with pytest.raises(blb.BLBError) as e:          # rotation without its key
        blb.rotate(g, keys, a, 3)
    assert e.value.status == 3
    plan = blb.MatmulPlan(g, 16, 16, 16, bsgs_B=16)
    with pytest.raises(blb.BLBError) as e:          # input at the wrong level
        plan(keys, [b1], plan.encode_weights(np.eye(16)))
    assert e.value.status in (3, 4)
    # degenerate inputs
    m, s = blb.ckks_to_mpc(g, [], bytes(32), 0)
    assert m.numel() == 0 and s.numel() == 0
    x = dev(np.zeros(toy.N, dtype=np.uint64))
    for w in (0, 65):
        with pytest.raises(blb.BLBError) as e:
            blb.share_to_rns(g, x, w, False, 2)
        assert e.value.status == 1
    with pytest.raises(blb.BLBError) as e:
        blb.share_decode(g, dev(np.zeros((toy.N, 2), dtype=np.uint64)), 60, 0)
    assert e.value.status == 1


# ---------------------------------------------------------------- row f4: batched inputs
def test_batched_inputs_bit_exact(toy):
    """Row f4 (App. D): B = 4 same-user inputs of 8 tokens packed along the spatial
    dimension (L' = 32 rows per block) run through one ct-pt MatMul plan; bit-exact against the
    oracle and each input's rows decode to its own X_b W."""
    from paper_2508_19525_b200 import packing
    Bt, L, D, Dout = 4, 8, 64, 48
    Xs = [bi.uniform(100 + b, (L, D), -1, 1) for b in range(Bt)]
    W = bi.normal(99, (D, Dout), 0.05)
    X = np.concatenate(Xs, axis=0)                      # (B L) x D: spatial-first with L' = B L
    plan_o = mm.plan_spatial(W, Bt * L, toy.n, 8)
    plan_g = blb.MatmulPlan(toy.g, Bt * L, D, Dout, bsgs_B=8)
    zs = list(packing.spatial_slots(X, toy.n))
    okeys, sk, oout, gout = run_both(toy, plan_o, plan_g, zs, W)
    for a, b in zip(gout, oout):
        assert np.array_equal(u64(a.data), b.data)
    dec = np.stack([toy.g.decode(blb.decrypt(toy.g, sk, c), c.scale).cpu().numpy() for c in gout])
    Y = packing.spatial_unslots(dec, Bt * L, Dout)
    for b in range(Bt):
        assert np.abs(Y[b * L:(b + 1) * L] - Xs[b] @ W).max() < 1e-5


# ---------------------------------------------------------------- S13 re-randomisation (C22)
@pytest.mark.parametrize("name,flood", [("toy", 0), ("toy", 20), ("bert", 30)])
def test_ckks_to_mpc_rerandomised_bit_exact(name, flood, request):
    """Optional re-randomisation before the mask: the public key, the re-randomised masked
    ciphertexts and the server shares are bit-exact against the oracle (two conversions, so the
    per-conversion ids are exercised)."""
    pair = request.getfixturevalue(name)
    okeys = O.keygen(pair.o, bi.crypto_key(4, 62))
    gkeys, sk = blb.keygen(pair.g, bi.crypto_key(4, 62), [])
    lvl = min(2, pair.K - 1)
    rng = np.random.default_rng(63)
    octs, gcts = [], []
    for t in range(2):
        pt = O.encode(pair.o, rng.uniform(-1, 1, pair.n), 2.0 ** 40, lvl)
        octs.append(O.encrypt(pair.o, bi.crypto_key(5, 62), okeys.s_ntt, pt, lvl, 20 + t, 2.0 ** 40))
        gcts.append(blb.encrypt(pair.g, sk, dev(pt), lvl, bi.crypto_key(5, 62), 20 + t, 2.0 ** 40))
    opk = O.public_key(pair.o, bi.crypto_key(5, 62), okeys.s_ntt)
    gpk = blb.public_key(pair.g, sk, bi.crypto_key(5, 62))
    assert np.array_equal(u64(gpk.data), opk.data)
    mk, rk = bi.crypto_key(3, 62), bi.crypto_key(6, 62)
    m, s = blb.ckks_to_mpc_rr(pair.g, gpk, gcts, mk, rk, 500, flood)
    for t in range(2):
        rr = O.rerandomize(pair.o, octs[t], opk, rk, 500 + t, flood)
        om, osh = O.mask(pair.o, rr, mk, 500 + t)
        assert np.array_equal(u64(m[t]), om) and np.array_equal(u64(s[t]), osh)


@pytest.mark.parametrize("name", ["toy", "bert"])
def test_algorithm2_chain_bit_exact(name, request):
    """Alg. 2 on the GPU: local fixed-point encode of both slot shares (C20), zero-sharing
    re-randomisation, reduction to Z_{2^83} (w = l + 40), ring-to-field of both shares on 128-bit
    words, P0's encryption + P1's ingest: every limb bit-exact against the oracle, and the result
    decodes to the shared vector."""
    pair = request.getfixturevalue(name)
    rng = np.random.default_rng(72)
    z = rng.uniform(-1, 1, pair.n)
    f, ft, w = 50, 50, 83
    s_out = f + pair.o.log_n - 40
    y = [int(round(v * 2.0 ** f)) for v in z]
    rnd = lambda n: [int(a) | (int(b) << 64) for a, b in zip(rng.integers(0, 2 ** 63, n, dtype=np.uint64),  # noqa
                                                          rng.integers(0, 2 ** 63, n, dtype=np.uint64))]
    y0 = rnd(pair.n)
    y1 = [(v - a) % (1 << 128) for v, a in zip(y, y0)]
    e0 = u64(blb.share_encode(pair.g, dev(O.int_to_u128(y0)), ft, s_out))
    e1 = u64(blb.share_encode(pair.g, dev(O.int_to_u128(y1)), ft, s_out))
    assert np.array_equal(e0, O.share_encode(pair.o, O.int_to_u128(y0), ft, s_out))
    assert np.array_equal(e1, O.share_encode(pair.o, O.int_to_u128(y1), ft, s_out))
    u = rnd(pair.N)
    x0 = O.int_to_u128([(a + r) % (1 << w) for a, r in zip(O.u128_to_int(e0), u)])
    x1 = O.int_to_u128([(b - r) % (1 << w) for b, r in zip(O.u128_to_int(e1), u)])
    lvl = min(2, pair.K - 1)
    for sub, xs in ((False, x0), (True, x1)):
        assert np.array_equal(u64(blb.share_to_rns(pair.g, dev(xs), w, sub, lvl)),
                              O.share_to_rns(pair.o, xs, w, sub, lvl))
    okeys = O.keygen(pair.o, bi.crypto_key(4, 73))
    gkeys, sk = blb.keygen(pair.g, bi.crypto_key(4, 73), [])
    f0 = O.share_to_rns(pair.o, x0, w, False, lvl)
    oct_ = O.mpc_to_ckks(pair.o, O.encrypt(pair.o, bi.crypto_key(5, 73), okeys.s_ntt, f0, lvl, 9, 2.0 ** 40), x1, w)
    gct = blb.mpc_to_ckks(pair.g, blb.encrypt(pair.g, sk, dev(f0), lvl, bi.crypto_key(5, 73), 9, 2.0 ** 40),
                          dev(x1), w)
    assert np.array_equal(u64(gct.data), oct_.data)
    dec = pair.g.decode(blb.decrypt(pair.g, sk, gct), gct.scale).cpu().numpy()
    assert np.abs(dec - z).max() < 1e-6
