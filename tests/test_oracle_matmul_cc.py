"""Oracle pins: ct-ct MatMul Q_h K_h^T (sec. 5.1; App. C.1 P:1203-1207;
reading C13).  Slot-level execution of the schedule equals Q_h K_h^T; Table 5's
CMult count is exact and its rotation count within 3%; the depth is
4 including the QKV ct-pt MatMul; the encrypted toy meets MSE < 1e-11
(P:698)."""
import numpy as np
import pytest

import blb_inputs as bi
import oracle as O
import oracle.matmul as mm
import oracle.matmul_cc as cc


@pytest.mark.parametrize("L,H,dh,n,B", [(32, 4, 32, 2048, None), (16, 3, 16, 512, None), (32, 4, 16, 2048, 32),
                                        (8, 2, 8, 64, None), (16, 2, 24, 256, 16)])
def test_slot_level_exact(L, H, dh, n, B):
    p = cc.plan_qk(L, H, dh, n, B)
    rng = np.random.default_rng(L + H + dh)
    Q, K = rng.normal(size=(H, L, dh)), rng.normal(size=(H, L, dh))
    C = cc.unpack_diag(cc.slot_level(cc.pack_mhp(Q, p), cc.pack_mhp(K, p), p), p)
    assert np.abs(C - np.einsum("hik,hjk->hij", Q, K)).max() < 1e-12


def test_figure6_observations():
    """Obs. 1: A{:,k} (.) B{k,:} = k-th partial sum of the main diagonal;
    Obs. 2: rotating B{k,:} left by t gives the k-th partial of diagonal t."""
    rng = np.random.default_rng(0)
    L, D = 4, 2
    A, Bm = rng.normal(size=(L, D)), rng.normal(size=(D, L))
    C = A @ Bm
    for t in range(L):
        diag = sum(A[:, k] * np.roll(Bm[k], -t) for k in range(D))
        assert np.allclose(diag, [C[i, (i + t) % L] for i in range(L)])


def test_table5_counts_bert_large():
    """Table 5, BERT-large dims, s = 16384 slots: #CMult = 1024 exactly, #Rot = 640."""
    p = cc.plan_qk(128, 16, 64, 16384)
    cnt = p.counts()
    assert cnt["cmult"] == 1024 == 128 * 128 * 1024 // 16384   # m^2 d / s
    assert abs(cnt["rotations"] - 640) <= 0.03 * 640
    assert cnt["relin"] == 128


def test_bert_base_counts():
    cnt = cc.plan_qk(128, 12, 64, 32768).counts()
    assert (cnt["rotations"], cnt["cmult"], cnt["relin"]) == (444, 512, 128)


@pytest.fixture(scope="module")
def qktoy():
    P = bi.QKTOY
    pr = O.prime_chain(P.log_n, list(P.q_bits) + list(P.p_bits))
    return O.Ctx(P.log_n, pr[:5], pr[5:], P.dnum)


def test_encrypted_toy_accuracy_and_depth(qktoy):
    d = bi.qk_toy_inputs()
    plan = cc.plan_qk(32, 4, 32, qktoy.n)
    keys = O.keygen(qktoy, d["keys_key"], plan.rotation_steps(), relin=True)
    lvl, delta = 3, 2.0 ** 40
    Q = [O.encrypt(qktoy, d["enc_key"], keys.s_ntt, O.encode(qktoy, z, delta, lvl), lvl, j, delta)
         for j, z in enumerate(cc.pack_mhp(d["Q"], plan))]
    K = [O.encrypt(qktoy, d["enc_key"], keys.s_ntt, O.encode(qktoy, z, delta, lvl), lvl, 10 + j, delta)
         for j, z in enumerate(cc.pack_mhp(d["K"], plan))]
    outs = cc.qk_encrypted(qktoy, keys, Q, K, plan)
    assert len(outs) == plan.n_out and all(o.level == lvl - 3 for o in outs)   # 3 levels here (+1 QKV = 4)
    C = cc.unpack_diag([O.decode(qktoy, O.decrypt(qktoy, keys.s_ntt, o), o.scale) for o in outs], plan)
    ref = np.einsum("hik,hjk->hij", d["Q"], d["K"])
    assert float(((C - ref) ** 2).mean()) <= 1e-11
    assert np.abs(C - ref).max() <= 2 ** -16 * max(1.0, np.abs(ref).max())


def test_qkv_then_qk_chain_slot_level():
    """Fused attention flow: MHP-reordered QKV ct-pt MatMul feeds the ct-ct
    protocol directly; result = (X W_Q)_h (X W_K)_h^T per head."""
    L, d, H, n = 16, 32, 2, 512
    X = bi.uniform(1, (L, d), -1, 1)
    WQ, WK = bi.normal(2, (d, d), 0.2), bi.normal(3, (d, d), 0.2)
    cm = mm.mhp_column_map(d, H, L, n)
    xz = mm.pack_spatial(X, n)
    Qz = mm.slot_level(xz, mm.plan_spatial(WQ, L, n, 8, col_map=cm))
    Kz = mm.slot_level(xz, mm.plan_spatial(WK, L, n, 8, col_map=cm))
    p = cc.plan_qk(L, H, d // H, n)
    C = cc.unpack_diag(cc.slot_level(Qz, Kz, p), p)
    dh = d // H
    Qm, Km = X @ WQ, X @ WK
    ref = np.stack([Qm[:, h * dh:(h + 1) * dh] @ Km[:, h * dh:(h + 1) * dh].T for h in range(H)])
    assert np.abs(C - ref).max() < 1e-12


@pytest.mark.parametrize("L,H,n", [(16, 2, 256), (32, 3, 2048), (16, 4, 512)])
def test_softmax_v_then_wo_chain_slot_level(L, H, n):
    """Row f1: Att_h = S_h V_h by the C13 protocol with V zero-padded d_h -> L,
    adjacent outputs added into a dense diagonal packing, then the diagonal-input
    ct-pt MatMul with the MHP row reorder of W_O (App. C.2) gives Concat(Att_h) W_O."""
    dh = L // 2
    rng = np.random.default_rng(L + H)
    S = rng.uniform(0, 1, size=(H, L, L))
    V = rng.normal(size=(H, L, dh))
    WO = rng.normal(size=(H * dh, 24))
    p = cc.plan_sv(L, H, n)
    A, Kop = cc.sv_operands(S, V)
    outs = cc.slot_level(cc.pack_mhp(A, p), cc.pack_mhp(Kop, p), p)
    full = cc.unpack_diag(outs, p)
    assert np.abs(full[:, :, :dh] - np.einsum("hik,hkj->hij", S, V)).max() < 1e-12
    assert np.abs(full[:, :, dh:]).max() < 1e-12
    dense = cc.collapse_dense(outs, p, dh)
    WOp = cc.pad_heads_rows(WO, H, p.Hp)
    plan_o = mm.plan_diagonal(WOp, p.Hp, L, n, 8)
    assert plan_o.n_in == len(dense)
    Y = mm.unpack_spatial(mm.slot_level(dense, plan_o), L, WO.shape[1])
    Att = np.concatenate([S[h] @ V[h] for h in range(H)], axis=1)
    assert np.abs(Y - Att @ WO).max() < 1e-11


def test_table5_softmax_v_counts():
    """Table 5, Softmax x V_h, BERT-large dims, s = 16384: #CMult = m^3 H / s = 2048
    exactly; #Rot = 1056 (we reconstruct 1092, within the 2x envelope of S:416)."""
    p = cc.plan_sv(128, 16, 16384)
    cnt = p.counts()
    assert cnt["cmult"] == 2048 == 128 ** 3 * 16 // 16384
    assert cnt["rotations"] <= 2 * 1056


def test_sampled_outputs_equal_full_schedule(qktoy):
    """qk_encrypted(out_ids=...) (used for sampled parity at N = 2^16) returns exactly the
    ciphertexts the full schedule computes for those outputs."""
    d = bi.qk_toy_inputs(H=4, L=32, dh=16)
    plan = cc.plan_qk(32, 4, 16, qktoy.n)
    keys = O.keygen(qktoy, d["keys_key"], plan.rotation_steps(), relin=True)
    lvl, delta = 3, 2.0 ** 40
    Q = [O.encrypt(qktoy, d["enc_key"], keys.s_ntt, O.encode(qktoy, z, delta, lvl), lvl, j, delta)
         for j, z in enumerate(cc.pack_mhp(d["Q"], plan))]
    K = [O.encrypt(qktoy, d["enc_key"], keys.s_ntt, O.encode(qktoy, z, delta, lvl), lvl, 10 + j, delta)
         for j, z in enumerate(cc.pack_mhp(d["K"], plan))]
    full = cc.qk_encrypted(qktoy, keys, Q, K, plan)
    sample = [plan.n_out - 1, 0]
    part = cc.qk_encrypted(qktoy, keys, Q, K, plan, out_ids=sample)
    for o, ct in zip(sample, part):
        assert np.array_equal(ct.data, full[o].data) and ct.scale == full[o].scale
