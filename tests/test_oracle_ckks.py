"""Oracle pins: encryption (C6), keys (C5), base conversion / ModUp / ModDown
(C7), hoisted rotation (C8), relinearisation (C9), rescale (C10) and the
CKKS->MPC mask (C14; Alg. 1, Theorem 1).

Exact checks use big-integer CRT and an independent ChaCha20 (`cryptography`);
noise checks use bounds derived in DESIGN.md."""
import struct

import numpy as np
import pytest
from cryptography.hazmat.primitives.ciphers import Cipher, algorithms

import blb_inputs as bi
import oracle as O


def keystream_draw(key, tag, objid, x):
    nonce = struct.pack("<IQ", tag, objid)
    enc = Cipher(algorithms.ChaCha20(key, struct.pack("<I", x // 4) + nonce), mode=None).encryptor()
    blk = enc.update(bytes(64))
    d = x % 4
    return int.from_bytes(blk[16 * d:16 * d + 16], "little")


def cbd_ref(key, tag, objid, N):
    m = (1 << 21) - 1
    out = []
    for x in range(N):
        lo = keystream_draw(key, tag, objid, x) & (2**64 - 1)
        out.append(bin(lo & m).count("1") - bin((lo >> 21) & m).count("1"))
    return out


def brv(x, bits):
    return int(format(x, "0%db" % bits)[::-1], 2)


def closed_ntt(a, psi, q, logn):
    N = 1 << logn
    out = []
    for k in range(N):
        w = pow(psi, 2 * brv(k, logn) + 1, q)
        out.append(sum(int(a[j]) * pow(w, j, q) for j in range(N)) % q)
    return out


def crt(vals, mods):
    Q = 1
    for m in mods:
        Q *= m
    x = 0
    for v, m in zip(vals, mods):
        qh = Q // m
        x += int(v) * qh * pow(qh % m, -1, m)
    return x % Q, Q


@pytest.fixture(scope="module")
def tiny():
    P = bi.TINY
    q = O.prime_chain(P.log_n, list(P.q_bits) + list(P.p_bits))
    return O.Ctx(P.log_n, q[:3], q[3:], P.dnum)


@pytest.fixture(scope="module")
def mid():
    P = bi.MID
    q = O.prime_chain(P.log_n, list(P.q_bits) + list(P.p_bits))
    return O.Ctx(P.log_n, q[:4], q[4:], P.dnum)


@pytest.fixture(scope="module")
def toy():
    P = bi.TOY
    q = O.prime_chain(P.log_n, list(P.q_bits) + list(P.p_bits))
    return O.Ctx(P.log_n, q[:3], q[3:], P.dnum)


# ---------------------------------------------------------------- enc / dec
def test_encrypt_decrypt_exact(tiny):
    key = bi.crypto_key(9, 0)
    keys = O.keygen(tiny, key)
    pt = O.encode(tiny, np.random.default_rng(0).uniform(-1, 1, tiny.n), 2.0 ** 20, 2)
    ct = O.encrypt(tiny, key, keys.s_ntt, pt, 2, ct_id=5, scale=2.0 ** 20)
    d = O.decrypt(tiny, keys.s_ntt, ct)
    e = cbd_ref(key, O.TAG_ENC_E, 5 << 8, tiny.N)
    for i in range(3):
        q = tiny.mods[i]
        # c1 is the uniform draw (NTT domain, per limb)
        assert [int(v) for v in ct.data[1, i]] == [keystream_draw(key, O.TAG_ENC_A, (5 << 8) | i, x) % q
                                                  for x in range(tiny.N)]
        diff = [(int(a) - int(b)) % q for a, b in zip(d[i], pt[i])]
        assert diff == closed_ntt([v % q for v in e], tiny.psi[i], q, tiny.log_n)
    # secret is ternary from the SECRET draws
    s_ref = [(keystream_draw(key, O.TAG_SECRET, 0, x) & (2**64 - 1)) % 3 - 1 for x in range(tiny.N)]
    assert keys.s_coef.tolist() == s_ref


def test_fresh_encryptions_differ(tiny):
    key = bi.crypto_key(9, 0)
    keys = O.keygen(tiny, key)
    pt = O.encode(tiny, np.zeros(tiny.n), 2.0 ** 20, 2)
    a = O.encrypt(tiny, key, keys.s_ntt, pt, 2, 0, 1.0)
    b = O.encrypt(tiny, key, keys.s_ntt, pt, 2, 1, 1.0)
    assert not np.array_equal(a.data, b.data)


def test_switching_key_structure(mid):
    """b_j + a_j s - P pi_j s' == NTT(e_j) exactly (C5)."""
    key = bi.crypto_key(4, 99)
    keys = O.keygen(mid, key, rot_steps=[3])
    g = mid.galois(3)
    rk = keys.rot[g]
    sp = mid.automorphism_ntt(keys.s_ntt, g)
    P = mid.P()
    for j in range(mid.beta_top):
        e = cbd_ref(key, O.TAG_KEY_E, (g * 64 + j) << 8, mid.N)
        for i, q in enumerate(mid.mods):
            in_digit = i < mid.K and j * mid.alpha <= i < (j + 1) * mid.alpha
            b, a, s, t = rk[j, 0, i], rk[j, 1, i], keys.s_ntt[i], sp[i]
            lhs = [(int(b[x]) + int(a[x]) * int(s[x]) - (P * int(t[x]) if in_digit else 0)) % q for x in range(mid.N)]
            en = O.Ctx.ntt(mid, np.array([v % q for v in e], dtype=np.uint64)[None], [i])[0]
            assert lhs == [int(v) for v in en]


# ------------------------------------------------------------- base conversion
def test_fastbconv_exact_invariant():
    rng = np.random.default_rng(5)
    cm = O.prime_chain(5, [40, 41, 45])
    dm = O.prime_chain(5, [60])[0]
    N = 32
    src = np.stack([rng.integers(0, m, N, dtype=np.uint64) for m in cm])
    out = O.fastbconv(src, cm, dm)
    for x in range(N):
        X, C = crt([src[i, x] for i in range(3)], cm)
        u = [u for u in range(3) if (X + u * C) % dm == int(out[x])]
        assert u, "FastBConv(x) != x + u*C for u in [0, |C|)"


def test_modup_exact_invariant(mid):
    """INTT(ModUp(D_j(x))) == [x]_{C_j} + u*C_j on every limb, 0 <= u < |C_j| (C7)."""
    rng = np.random.default_rng(6)
    lvl = 3
    k = lvl + 1
    d = np.stack([rng.integers(0, mid.mods[i], mid.N, dtype=np.uint64) for i in range(k)])
    ext = O.modup(mid, d, lvl)
    coef = mid.intt(d, list(range(k)))
    E = k + mid.np_
    pidx = list(range(k)) + [mid.K + t for t in range(mid.np_)]
    for j in range(mid.beta(lvl)):
        dig = list(range(j * mid.alpha, min((j + 1) * mid.alpha, k)))
        ext_coef = mid.intt(ext[j], pidx)
        for x in range(0, mid.N, 37):
            X, C = crt([coef[i, x] for i in dig], [mid.mods[i] for i in dig])
            us = set()
            for m in range(E):
                mod = mid.mods[pidx[m]]
                cand = {u for u in range(len(dig)) if (X + u * C) % mod == int(ext_coef[m, x])}
                us = cand if m == 0 else us & cand
            assert us, "no common u"


def test_moddown_exact_invariant(mid):
    """ModDown(y) == (Y - [Y]_P)/P - u  (mod q_i), u in [0, np) (C7, no rounding)."""
    rng = np.random.default_rng(7)
    lvl = 2
    k = lvl + 1
    pidx = list(range(k)) + [mid.K + t for t in range(mid.np_)]
    mods = [mid.mods[i] for i in pidx]
    y = np.stack([rng.integers(0, m, mid.N, dtype=np.uint64) for m in mods])
    out = O.moddown(mid, y, lvl)
    ycoef = mid.intt(y, pidx)
    ocoef = mid.intt(out, list(range(k)))
    P = mid.P()
    for x in range(0, mid.N, 29):
        Y, QP = crt([ycoef[m, x] for m in range(len(pidx))], mods)
        YP = Y % P
        base = (Y - YP) // P
        Qk = QP // P
        got, _ = crt([ocoef[i, x] for i in range(k)], mods[:k])
        assert any((base - u) % Qk == got for u in range(mid.np_))


def test_rescale_is_exact_rounding(mid):
    rng = np.random.default_rng(8)
    lvl = 3
    data = np.stack([np.stack([rng.integers(0, mid.mods[i], mid.N, dtype=np.uint64) for i in range(lvl + 1)])
                     for _ in range(2)])
    ct = O.Ct(data, lvl, 2.0 ** 80)
    out = O.rescale(mid, ct)
    assert out.level == lvl - 1 and out.scale == 2.0 ** 80 / mid.q[lvl]
    ql = mid.q[lvl]
    for p in range(2):
        c_in = mid.intt(data[p], list(range(lvl + 1)))
        c_out = mid.intt(out.data[p], list(range(lvl)))
        for x in range(0, mid.N, 17):
            X, Q = crt(c_in[:, x], mid.q[:lvl + 1])
            Y, Qo = crt(c_out[:, x], mid.q[:lvl])
            # centred lift, then round(X / q_l) (q_l odd: no ties)
            Xc = X - Q if X > Q // 2 else X
            r = (2 * Xc + ql) // (2 * ql)
            assert Y == r % Qo


# --------------------------------------------------------------- rotations
@pytest.fixture(scope="module")
def toy_keys(toy):
    return O.keygen(toy, bi.crypto_key(4, 1), rot_steps=[1, 5, 16, 21, -16], relin=True)


def enc(toy, keys, z, cid, delta=2.0 ** 40):
    return O.encrypt(toy, bi.crypto_key(5, 1), keys.s_ntt, O.encode(toy, z, delta, 2), 2, cid, delta)


def dec(toy, keys, ct):
    return O.decode(toy, O.decrypt(toy, keys.s_ntt, ct), ct.scale)


def test_rotation_left_roll(toy, toy_keys):
    z = np.random.default_rng(1).uniform(-1, 1, toy.n)
    ct = enc(toy, toy_keys, z, 0)
    for r in [1, 16, -16]:
        got = dec(toy, toy_keys, O.rotate(toy, ct, toy_keys, r))
        assert np.abs(got - np.roll(z, -r)).max() < 1e-6
    # Rot_n == identity (5^n == 1 mod 2N): no key needed, exact copy
    assert np.array_equal(O.rotate(toy, ct, toy_keys, toy.n).data, ct.data)
    # composition: Rot_5 o Rot_16 == Rot_21 after decryption
    a = dec(toy, toy_keys, O.rotate(toy, O.rotate(toy, ct, toy_keys, 16), toy_keys, 5))
    b = dec(toy, toy_keys, O.rotate(toy, ct, toy_keys, 21))
    assert np.abs(a - b).max() < 1e-6
    with pytest.raises(KeyError):
        O.rotate(toy, ct, toy_keys, 2)


def test_keyswitch_noise_bound(toy, toy_keys):
    """Coefficient-domain key-switch error: ||Dec(Rot(ct)) - sigma(Dec(ct))||_inf stays
    within 2^18 (estimate sigma*N*sqrt(beta/12)*Q_j/P ~ 2^14 for the toy preset)."""
    z = np.random.default_rng(2).uniform(-1, 1, toy.n)
    ct = enc(toy, toy_keys, z, 1)
    g = toy.galois(5)
    lhs = O.decrypt(toy, toy_keys.s_ntt, O.rotate(toy, ct, toy_keys, 5))
    rhs = toy.automorphism_ntt(O.decrypt(toy, toy_keys.s_ntt, ct), g)
    diff = toy.intt(np.stack([(lhs[i].astype(object) - rhs[i].astype(object)) % toy.mods[i] for i in range(3)])
                    .astype(np.uint64), [0, 1, 2])
    cen = O.crt_centered(toy, diff)
    assert max(abs(v) for v in cen) < 2 ** 18


def test_relinearized_product(toy, toy_keys):
    rng = np.random.default_rng(3)
    a, b = rng.uniform(-1, 1, toy.n), rng.uniform(-1, 1, toy.n)
    ca, cb = enc(toy, toy_keys, a, 10), enc(toy, toy_keys, b, 11)
    prod = O.rescale(toy, O.relinearize(toy, O.tensor(toy, ca, cb), toy_keys))
    assert prod.level == 1
    assert np.abs(dec(toy, toy_keys, prod) - a * b).max() < 1e-6


def test_pt_mult_scale_bookkeeping(toy, toy_keys):
    z = np.random.default_rng(4).uniform(-1, 1, toy.n)
    w = np.random.default_rng(5).uniform(-1, 1, toy.n)
    ct = enc(toy, toy_keys, z, 2)
    ql = float(toy.q[2])
    out = O.rescale(toy, O.mul_pt(toy, ct, O.encode(toy, w, ql, 2), ql))
    assert out.scale == 2.0 ** 40   # Delta * q_l / q_l, exact
    assert np.abs(dec(toy, toy_keys, out) - z * w).max() < 1e-7


# --------------------------------------------------------------- mask (C14)
def test_mask_shares_reconstruct_exactly(toy, toy_keys):
    z = np.random.default_rng(6).uniform(-1, 1, toy.n)
    ct = enc(toy, toy_keys, z, 3)
    mkey = bi.crypto_key(3, 1)
    masked, share = O.mask(toy, ct, mkey, 77)
    q0 = toy.q[0]
    r = O.sample_uniform(mkey, O.TAG_MASK, 77 << 8, q0, toy.N)
    c0 = toy.intt(ct.data[0, :1], [0])[0]
    assert np.array_equal((masked[0].astype(object) - r.astype(object)) % q0, c0.astype(object))
    assert np.array_equal(masked[1], toy.intt(ct.data[1, :1], [0])[0])
    assert np.array_equal((share.astype(object) + r.astype(object)) % q0, np.zeros(toy.N, dtype=object))
    # client side (test only): tmp0 = masked_c0 + masked_c1 * s (mod q0); tmp0 + share == Dec(ct) mod q0
    s0 = toy_keys.s_ntt[:1]
    m0 = toy.ntt(masked[0][None], [0])[0].astype(object)
    m1 = toy.ntt(masked[1][None], [0])[0].astype(object)
    tmp0 = toy.intt(((m0 + m1 * s0[0].astype(object)) % q0).astype(np.uint64)[None], [0])[0]
    decc = toy.intt(O.decrypt(toy, toy_keys.s_ntt, ct)[:1], [0])[0]
    assert np.array_equal((tmp0.astype(object) + share.astype(object)) % q0, decc.astype(object))


@pytest.mark.parametrize("offset", [0.0, 1000.0])
def test_masked_decryption_uniform(toy, toy_keys, offset):
    """Theorem 1: P0's view Dec(ct + r) is uniform over Z_q0 -- chi-square,
    64 bins, alpha = 0.01, for zero-mean and large-offset messages."""
    from scipy.stats import chisquare
    z = np.random.default_rng(7).uniform(-1, 1, toy.n) + offset
    ct = enc(toy, toy_keys, z, 4)
    counts = np.zeros(64)
    q0 = toy.q[0]
    s0 = toy_keys.s_ntt[0].astype(object)
    for cid in range(8):
        masked, _ = O.mask(toy, ct, bi.crypto_key(3, 1), 1000 + cid)
        m0 = toy.ntt(masked[0][None], [0])[0].astype(object)
        m1 = toy.ntt(masked[1][None], [0])[0].astype(object)
        tmp0 = toy.intt(((m0 + m1 * s0) % q0).astype(np.uint64)[None], [0])[0]
        counts += np.bincount((tmp0.astype(object) * 64 // q0).astype(np.int64), minlength=64)
    assert chisquare(counts).pvalue > 0.01


# --------------------------------------------------------------- row f2
def test_rotate_sum_table3_and_values(toy, toy_keys):
    """Table 3: fused summation = log2 D rotations, 0 multiplications; the
    first column block holds the row sums; all-ones L x D -> every slot = D."""
    import oracle.matmul as mm
    L, D = 16, 4
    keys = O.keygen(toy, bi.crypto_key(4, 5), rot_steps=[L, 2 * L, -L, -2 * L])
    X = np.random.default_rng(9).uniform(-1, 1, (L, D))
    z = mm.pack_spatial(X, toy.n)[0]
    ct = enc(toy, keys, z, 20)
    out = O.rotate_sum(toy, ct, keys, L, D)
    got = dec(toy, keys, out)
    assert np.abs(got[:L] - X.sum(axis=1)).max() < 1e-6
    ones = enc(toy, keys, np.concatenate([np.ones(L * D), np.zeros(toy.n - L * D)]), 21)
    assert np.abs(dec(toy, keys, O.rotate_sum(toy, ones, keys, L, D))[:L] - D).max() < 1e-6
    # broadcast of an (L, 1) column: replicated into D column blocks
    col = np.zeros(toy.n)
    col[:L] = X[:, 0]
    got = dec(toy, keys, O.rotate_sum(toy, enc(toy, keys, col, 22), keys, L, D, broadcast=True))
    assert np.abs(got[:L * D] - np.tile(X[:, 0], D)).max() < 1e-6


def test_squaring_chain(qk_ctx=None):
    """ewmul_cc chain: three relinearised squarings + rescales (the depth pattern of
    negExp's (1 + x/2^6)^{2^6}) decode to x^8."""
    P = bi.QKTOY
    q = O.prime_chain(P.log_n, list(P.q_bits) + list(P.p_bits))
    ctx = O.Ctx(P.log_n, q[:5], q[5:], P.dnum)
    keys = O.keygen(ctx, bi.crypto_key(4, 6), relin=True)
    z = np.random.default_rng(10).uniform(0.5, 1.0, ctx.n)
    ct = O.encrypt(ctx, bi.crypto_key(5, 6), keys.s_ntt, O.encode(ctx, z, 2.0 ** 40, 4), 4, 1, 2.0 ** 40)
    for _ in range(3):
        ct = O.rescale(ctx, O.mul_relin(ctx, ct, ct, keys))
    assert ct.level == 1
    got = O.decode(ctx, O.decrypt(ctx, keys.s_ntt, ct), ct.scale)
    assert np.abs(got - z ** 8).max() < 1e-6


def test_extended_basis_identities(toy, toy_keys):
    """Double hoisting (DESIGN C13): ModDown(P*x + y) = x + ModDown(y) exactly, because P*x
    vanishes mod P and (P*x)*P^-1 = x mod Q (C7).  Hence ModDown(rotate_ext(ct)) equals the
    plain hoisted rotation bit for bit, ModDown of the step-0 lift (P c0, P c1) is ct itself,
    and an extended-basis plaintext restricted to Q_l is the ordinary encoding (C3)."""
    z = np.random.default_rng(21).uniform(-1, 1, toy.n)
    for lvl in (2, 1):
        ct = enc(toy, toy_keys, z, 7)
        if lvl < 2:
            ct = O.Ct(ct.data[:, :lvl + 1].copy(), lvl, ct.scale)
        lift = O.rotate_ext(toy, ct, toy_keys, 0)
        assert lift.data.shape == (2, lvl + 1 + toy.np_, toy.N)
        assert np.array_equal(O.moddown_ct(toy, lift).data, ct.data)
        for r in (1, 16, -16):
            got = O.moddown_ct(toy, O.rotate_ext(toy, ct, toy_keys, r))
            assert np.array_equal(got.data, O.rotate(toy, ct, toy_keys, r).data)
        m = np.random.default_rng(22).uniform(-1, 1, toy.n)
        pe = O.encode_ext(toy, m, float(toy.q[lvl]), lvl)
        assert np.array_equal(pe[:lvl + 1], O.encode(toy, m, float(toy.q[lvl]), lvl))
        # the special-prime residue is the same rounded integer mod p
        coef_q = toy.intt(pe[:1], [0])[0]
        coef_p = toy.intt(pe[lvl + 1:], O.ext_pidx(toy, lvl)[lvl + 1:])[0]
        q0, p0 = int(toy.mods[0]), int(toy.mods[O.ext_pidx(toy, lvl)[lvl + 1]])
        cq = [int(v) if int(v) < q0 // 2 else int(v) - q0 for v in coef_q]
        assert all((c - int(v)) % p0 == 0 for c, v in zip(cq, coef_p))


@pytest.mark.parametrize("lvl", [1, 2])
def test_moddown_rescale_is_exact_rounding(mid, lvl):
    """C17: out == round(X / (q_l P)) mod q_i for every coefficient, X the CRT integer of the
    input over Q_l u P (big-integer CRT, independent of the oracle's Garner code); np = 2 here."""
    rng = np.random.default_rng(30 + lvl)
    k = lvl + 1
    pidx = list(range(k)) + [mid.K + t for t in range(mid.np_)]
    mods = [mid.mods[i] for i in pidx]
    y = np.stack([np.stack([rng.integers(0, m, mid.N, dtype=np.uint64) for m in mods]) for _ in range(2)])
    out = O.moddown_rescale(mid, O.CtExt(y, lvl, 1.0))
    assert out.level == lvl - 1 and out.data.shape == (2, lvl, mid.N)
    M = int(mid.mods[lvl]) * mid.P()
    for p in range(2):
        ycoef = mid.intt(y[p], pidx)
        ocoef = mid.intt(out.data[p], list(range(lvl)))
        for x in list(range(0, mid.N, 37)) + [mid.N - 1]:
            X, _ = crt([ycoef[m, x] for m in range(len(pidx))], mods)
            want = (X + (M - 1) // 2) // M
            assert all(int(ocoef[i, x]) == want % int(mid.mods[i]) for i in range(lvl))


def test_moddown_rescale_of_lift_is_rescale(toy, toy_keys):
    """round(P x / (q_l P)) = round(x / q_l): on the step-0 lift C17 reduces to C10 exactly."""
    z = np.random.default_rng(23).uniform(-1, 1, toy.n)
    ct = enc(toy, toy_keys, z, 9)
    got = O.moddown_rescale(toy, O.rotate_ext(toy, ct, toy_keys, 0))
    want = O.rescale(toy, ct)
    assert np.array_equal(got.data, want.data) and got.scale == want.scale and got.level == want.level
