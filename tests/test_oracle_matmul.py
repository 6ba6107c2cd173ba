"""Oracle pins: ct-pt MatMul (C11 spatial-first BSGS; MHP reorder
P:463-466; C12 diagonal input, App. C.2).

Pins: slot-level execution of the schedule equals X W (App. A item 6);
decoded encrypted output vs float64 X W within the paper's MSE < 1e-11;
W = I gives X back; rotation / plaintext counts equal the closed form
(B-1)*n_in + (G-1)*n_out and the SURVEY 8(d) table."""
import math

import numpy as np
import pytest

import blb_inputs as bi
import oracle as O
import oracle.matmul as mm


@pytest.fixture(scope="module")
def toy():
    P = bi.TOY
    q = O.prime_chain(P.log_n, list(P.q_bits) + list(P.p_bits))
    return O.Ctx(P.log_n, q[:3], q[3:], P.dnum)


def run_encrypted(ctx, X_zs, plan, seed=4, delta=2.0 ** 40, level=2):
    keys = O.keygen(ctx, bi.crypto_key(seed, 1), plan.rotation_steps())
    ek = bi.crypto_key(5, 1)
    cts = [O.encrypt(ctx, ek, keys.s_ntt, O.encode(ctx, z, delta, level), level, b, delta) for b, z in enumerate(X_zs)]
    outs = mm.matmul_cp(ctx, keys, cts, plan)
    return keys, outs, [O.decode(ctx, O.decrypt(ctx, keys.s_ntt, o), o.scale) for o in outs]


def check_accuracy(Y, ref):
    mse = float(((Y - ref) ** 2).mean())
    assert mse <= 1e-11, mse                                        # P:698 acceptance
    assert np.abs(Y - ref).max() <= 2 ** -16 * max(1.0, np.abs(ref).max())


def test_toy_config_counts_and_accuracy(toy):
    d = bi.toy_inputs()
    plan = mm.plan_spatial(d["W"], 16, toy.n, 16)
    assert (plan.n_plaintexts, plan.n_rotations) == (31, 16)
    assert plan.baby_steps == {0: list(range(1, 16))} and plan.giant_steps == {0: [7]}
    zs = mm.pack_spatial(d["X"], toy.n)
    keys, outs, dec = run_encrypted(toy, zs, plan)
    assert outs[0].level == 1 and outs[0].scale == 2.0 ** 40
    check_accuracy(mm.unpack_spatial(dec, 16, 16), d["X"] @ d["W"])


def test_identity_weight(toy):
    X = bi.uniform(31, (16, 24), -1, 1)
    W = np.eye(24)
    plan = mm.plan_spatial(W, 16, toy.n, 16)
    _, _, dec = run_encrypted(toy, mm.pack_spatial(X, toy.n), plan)
    assert np.abs(mm.unpack_spatial(dec, 16, 24) - X).max() < 1e-6


@pytest.mark.parametrize("L,D,Dout,B", [(16, 16, 16, 16), (8, 40, 24, 4), (32, 200, 72, 8), (4, 300, 260, 32)])
def test_slot_level_schedule_exact(L, D, Dout, B):
    n = 512
    X = bi.uniform(40 + D, (L, D), -1, 1)
    W = bi.uniform(41 + D, (D, Dout), -1, 1)
    plan = mm.plan_spatial(W, L, n, B)
    Y = mm.unpack_spatial(mm.slot_level(mm.pack_spatial(X, n), plan), L, Dout)
    assert np.abs(Y - X @ W).max() < 1e-12
    c = n // L
    n_in, n_out = math.ceil(D / c), math.ceil(Dout / c)
    G = math.ceil(c / B)
    assert plan.n_rotations <= (B - 1) * n_in + (G - 1) * n_out


def test_mhp_reorder_layout():
    """(L, H, D/H) packing of P:463 / Fig. 6(e): block cc*H_p + h of ciphertext j
    holds column j*g + cc of head h."""
    L, d, H, n = 4, 8, 2, 16    # c = 4 blocks, H_p = 2, g = 2, d_h = 4 -> J = 2
    cmap = mm.mhp_column_map(d, H, L, n)
    assert cmap == [0, 4, 1, 5, 2, 6, 3, 7]
    cmap = mm.mhp_column_map(768, 12, 128, 32768)   # BERT-base: 12 heads padded to 16
    assert len(cmap) == 1024 and cmap.count(-1) == 256 and sorted(c for c in cmap if c >= 0) == list(range(768))
    X = bi.uniform(50, (L, d), -1, 1)
    W = bi.uniform(51, (d, d), -1, 1)
    plan = mm.plan_spatial(W, L, n, 2, col_map=mm.mhp_column_map(d, H, L, n))
    Y = mm.unpack_spatial(mm.slot_level(mm.pack_spatial(X, n), plan), L, d)
    Yref = X @ W
    assert np.allclose(Y[:, 1], Yref[:, 4]) and np.allclose(Y[:, 2], Yref[:, 1])


def test_diagonal_slot_level_exact():
    L, H, dh, Dout, n = 16, 4, 8, 40, 512
    Att = bi.normal(60, (H, L, dh), 1.0)
    WO = bi.normal(61, (H * dh, Dout), 0.1)
    plan = mm.plan_diagonal(WO, H, L, n, 8)
    Y = mm.unpack_spatial(mm.slot_level(mm.pack_diagonal_mh(Att, n), plan), L, Dout)
    ref = np.concatenate([Att[h] for h in range(H)], axis=1) @ WO
    assert np.abs(Y - ref).max() < 1e-12


def test_diagonal_encrypted_toy(toy):
    L, H, dh, Dout = 16, 4, 16, 48     # 64 input blocks, c = 128
    Att = bi.normal(62, (H, L, dh), 1.0)
    WO = bi.normal(63, (H * dh, Dout), 0.05)
    plan = mm.plan_diagonal(WO, H, L, toy.n, 16)
    _, _, dec = run_encrypted(toy, mm.pack_diagonal_mh(Att, toy.n), plan)
    ref = np.concatenate([Att[h] for h in range(H)], axis=1) @ WO
    check_accuracy(mm.unpack_spatial(dec, L, Dout), ref)


def test_bert_plan_counts():
    """SURVEY 8(d) config 2/3 counts at N = 2^16, L = 128 (c = 256)."""
    n, L = 32768, 128
    rng = np.random.default_rng(0)
    W = rng.normal(size=(768, 768))
    cm = mm.mhp_column_map(768, 12, L, n)
    qkv_map = cm + [768 + c if c >= 0 else -1 for c in cm] + [1536 + c for c in range(768)]
    Wqkv = rng.normal(size=(768, 2304))
    p = mm.plan_spatial(Wqkv, L, n, 32, col_map=qkv_map)
    assert (p.n_in, p.n_out, p.n_plaintexts, p.n_rotations) == (3, 11, 8448, 170)
    assert sum(len(v) for v in p.baby_steps.values()) == 93
    p = mm.plan_diagonal(W, 12, L, n, 16)
    assert (p.n_in, p.n_out, p.n_plaintexts, p.n_rotations) == (3, 3, 2304, 90)
    p = mm.plan_spatial(rng.normal(size=(768, 3072)), L, n, 32)
    assert (p.n_plaintexts, p.n_rotations) == (9216, 177)
    p = mm.plan_spatial(rng.normal(size=(3072, 768)), L, n, 8)
    assert (p.n_plaintexts, p.n_rotations) == (9216, 177)
