"""Row f3 oracle pins: MPC -> CKKS ingest (Algorithm 2) with the ring-to-field local
step of App. C.3.  Independent checks: Python-integer residues, the decrypted
message, and the paper's correctness identity x0 + x1 - 2^w = m when x0 + x1 >= 2^w."""
import numpy as np
import pytest

import blb_inputs as bi
import oracle as O


@pytest.fixture(scope="module")
def toy():
    P = bi.TOY
    q = O.prime_chain(P.log_n, list(P.q_bits) + list(P.p_bits))
    return O.Ctx(P.log_n, q[:3], q[3:], P.dnum)


def test_share_to_rns_residues(toy):
    rng = np.random.default_rng(40)
    for w in (24, 40, 64):
        x = rng.integers(0, 2 ** min(w, 63), toy.N, dtype=np.uint64)
        if w == 64:
            x |= rng.integers(0, 2, toy.N, dtype=np.uint64) << np.uint64(63)
        for sub in (False, True):
            got = toy.intt(O.share_to_rns(toy, x, w, sub, 2), [0, 1, 2])
            for i in range(3):
                q = int(toy.mods[i])
                want = [(int(v) - (2 ** w if sub else 0)) % q for v in x[:64]]
                assert [int(v) for v in got[i, :64]] == want


def test_mpc_to_ckks_reconstructs_message(toy):
    """Client P0 encrypts x0 mod q, server P1 adds x1 - 2^w mod q: the ciphertext decrypts to
    m + e exactly (e = the encryption noise), so it decodes to the shared message."""
    rng = np.random.default_rng(41)
    z = rng.uniform(-1, 1, toy.n)
    delta, w, lvl = 2.0 ** 40, 64, 2
    m = np.array(O.encode_coeffs(toy, z, delta), dtype=object)        # signed integer coefficients
    x0 = [int(a) * 2 for a in rng.integers(2 ** 46, 2 ** 62, toy.N, dtype=np.uint64)]  # in [2^47, 2^63): no wrap
    x1 = [(int(mm) - int(a)) % 2 ** w for mm, a in zip(m, x0)]
    assert all(int(a) + b == int(mm) + 2 ** w for a, b, mm in zip(x0, x1, m))  # P:1222 success event
    x0u = np.array(x0, dtype=np.uint64)
    x1u = np.array(x1, dtype=np.uint64)
    key = bi.crypto_key(6, 1)
    keys = O.keygen(toy, key)
    pt0 = O.share_to_rns(toy, x0u, w, False, lvl)
    ct = O.encrypt(toy, bi.crypto_key(7, 1), keys.s_ntt, pt0, lvl, 3, delta)
    ct2 = O.mpc_to_ckks(toy, ct, x1u, w)
    d_before = O.decrypt(toy, keys.s_ntt, ct)
    d_after = O.decrypt(toy, keys.s_ntt, ct2)
    add = O.share_to_rns(toy, x1u, w, True, lvl)
    for i in range(lvl + 1):
        q = np.uint64(toy.mods[i])
        assert np.array_equal(d_after[i], (d_before[i] + add[i]) % q)
    got = O.decode(toy, d_after, delta)
    assert np.abs(got - z).max() < 1e-6


# ---------------------------------------------------------------- f3: local fixed-point Decode (C18)
def _slot_sums(ctx, m):
    """sum_k m_k Re(zeta_j^k) for every real slot j, in float64 via numpy's FFT-free direct
    evaluation at zeta^{5^j} (zeta = e^{i pi / N}), independent of the oracle's network."""
    N, n = ctx.N, ctx.n
    e = np.array([pow(5, j, 2 * N) for j in range(n)], dtype=np.int64)
    k = np.arange(N, dtype=np.int64)
    ang = np.pi * ((e[:, None] * k[None, :]) % (2 * N)) / N
    return (np.cos(ang) * np.asarray(m, dtype=np.float64)[None, :]).sum(axis=1)


def test_share_decode_single_party_matches_decode(toy):
    """One party holding the whole message: y = 2^-s_out sum_k m_k Re(zeta_j^k) up to the
    fixed-point error (twiddles rounded at 2^-ft, one truncation per stage), and with
    Delta = 2^30, s_out = 18 it is round(2^12 z) within 2 ulps."""
    rng = np.random.default_rng(42)
    z = rng.uniform(-1, 1, toy.n)
    m = [int(v) for v in O.encode_coeffs(toy, z, 2.0 ** 30)]
    ft, s_out = 30, 18
    y = O.u128_to_int(O.share_decode(toy, O.int_to_u128(m), ft, s_out))
    exact = _slot_sums(toy, m) / 2.0 ** s_out
    assert np.abs(np.array(y, dtype=np.float64) - exact).max() < 4.0
    assert np.abs(np.array(y, dtype=np.float64) - np.round(z * 2.0 ** 12)).max() <= 2
    # a wrong twiddle sign or index would be off by ~|m| / 2^s_out >> 4: check one such perturbation
    assert np.abs(_slot_sums(toy, m[1:] + m[:1]) / 2.0 ** s_out - exact).max() > 100


def test_share_decode_two_party_reconstruction(toy):
    """Additive shares x0 + x1 = m over Z_{2^128} (x0 uniform): the local decodes add up to the
    single-party decode of m within the local-truncation error (SecureML: each truncation adds
    at most 1 ulp of disagreement; failure probability |v| / 2^127 per truncation)."""
    rng = np.random.default_rng(43)
    z = rng.uniform(-1, 1, toy.n)
    m = [int(v) for v in O.encode_coeffs(toy, z, 2.0 ** 30)]
    x0 = [int(a) | (int(b) << 64) for a, b in zip(rng.integers(0, 2 ** 63, toy.N, dtype=np.uint64),
                                                  rng.integers(0, 2 ** 63, toy.N, dtype=np.uint64))]
    x1 = [(mm - a) % (1 << 128) for mm, a in zip(m, x0)]
    ft, s_out = 30, 18
    y0 = O.u128_to_int(O.share_decode(toy, O.int_to_u128(x0), ft, s_out))
    y1 = O.u128_to_int(O.share_decode(toy, O.int_to_u128(x1), ft, s_out))
    ym = O.u128_to_int(O.share_decode(toy, O.int_to_u128(m), ft, s_out))
    rec = [((a + b + (1 << 127)) % (1 << 128)) - (1 << 127) for a, b in zip(y0, y1)]
    assert max(abs(r - t) for r, t in zip(rec, ym)) <= 2


# ---------------------------------------------------------------- f3: local fixed-point Encode (C20)
def _fx(z, f):
    return [int(round(v * 2.0 ** f)) for v in z]


def test_share_encode_single_party_is_the_ckks_encode(toy):
    """One party holding the whole slot vector y = round(2^f z): the local fixed-point Encode
    (Alg. 2 line 1) equals the correctly rounded CKKS encode Delta pi^{-1}(y / 2^f) (C3, the
    oracle's __float128 encode) within 1, for Delta = 2^(f + log N - s_out)."""
    rng = np.random.default_rng(44)
    z = rng.uniform(-1, 1, toy.n)
    f, ft = 50, 50
    s_out = f + toy.log_n - 40                     # Delta = 2^40
    y = _fx(z, f)
    x = O.u128_to_int(O.share_encode(toy, O.int_to_u128(y), ft, s_out))
    exact = [int(v) for v in O.encode_coeffs(toy, np.array(y, dtype=np.float64) / 2.0 ** f, 2.0 ** 40)]
    assert max(abs(a - b) for a, b in zip(x, exact)) <= 1
    # constants encode to Delta c at coefficient 0 only; zero to zero
    c = O.u128_to_int(O.share_encode(toy, O.int_to_u128([3 << (f - 2)] * toy.n), ft, s_out))
    assert abs(c[0] - 3 * 2 ** 38) <= 1 and max(abs(v) for v in c[1:]) <= 1
    assert O.u128_to_int(O.share_encode(toy, O.int_to_u128([0] * toy.n), ft, s_out)) == [0] * toy.N


def test_share_encode_two_party_reconstruction(toy):
    """Additive shares y0 + y1 = y over Z_{2^128}: the two local encodes add up to the encode of y
    within the SecureML local-truncation error (App. C.4)."""
    rng = np.random.default_rng(45)
    z = rng.uniform(-1, 1, toy.n)
    f, ft = 50, 50
    s_out = f + toy.log_n - 40
    y = _fx(z, f)
    y0 = [int(a) | (int(b) << 64) for a, b in zip(rng.integers(0, 2 ** 63, toy.n, dtype=np.uint64),
                                                  rng.integers(0, 2 ** 63, toy.n, dtype=np.uint64))]
    y1 = [(v - a) % (1 << 128) for v, a in zip(y, y0)]
    x0 = O.u128_to_int(O.share_encode(toy, O.int_to_u128(y0), ft, s_out))
    x1 = O.u128_to_int(O.share_encode(toy, O.int_to_u128(y1), ft, s_out))
    x = O.u128_to_int(O.share_encode(toy, O.int_to_u128(y), ft, s_out))
    rec = [((a + b + (1 << 127)) % (1 << 128)) - (1 << 127) for a, b in zip(x0, x1)]
    assert max(abs(r - t) for r, t in zip(rec, x)) <= 2


def test_share_encode_then_decode_round_trip(toy):
    """share_decode(share_encode(y)) returns Delta z (C18 after C20) within the fixed-point error."""
    rng = np.random.default_rng(46)
    z = rng.uniform(-1, 1, toy.n)
    f, ft = 50, 50
    s_out = f + toy.log_n - 40
    x = O.share_encode(toy, O.int_to_u128(_fx(z, f)), ft, s_out)
    back = O.u128_to_int(O.share_decode(toy, x, 30, 0))        # sum_k x_k Re(zeta^{k 5^j}) = Delta z_j
    assert np.abs(np.array(back, dtype=np.float64) - z * 2.0 ** 40).max() < 2.0 ** 12   # |err| < 2^-28 of 1.0


def test_share_to_rns_wide_residues(toy):
    """Ring-to-field on Z_{2^w}, w = l + 40 = 83 (l = 43) and w = 128: residues of
    the 128-bit shares, the P1 variant subtracting 2^w mod q_i (Python integers)."""
    rng = np.random.default_rng(47)
    for w in (83, 128):
        xs = [int(a) | (int(b) << 64) for a, b in zip(rng.integers(0, 2 ** 63, toy.N, dtype=np.uint64),
                                                      rng.integers(0, 2 ** 63, toy.N, dtype=np.uint64))]
        xs = [v % (1 << w) for v in xs]
        x = O.int_to_u128(xs)
        for sub in (False, True):
            got = toy.intt(O.share_to_rns(toy, x, w, sub, 2), [0, 1, 2])
            for i in range(3):
                q = int(toy.mods[i])
                assert [int(v) for v in got[i, :64]] == [(v - (2 ** w if sub else 0)) % q for v in xs[:64]]


def test_algorithm2_chain_encode_ring_to_field_ingest(toy):
    """Alg. 2 end to end on the toy ring: each party encodes its slot share locally
    (C20), the shares are reduced to Z_{2^w} with w = l + 40 = 83, ring-to-field maps them to the
    field (App. C.3), P0 encrypts its field share and P1 adds its own: the ciphertext decodes to the
    shared vector (the paper's success event x0 + x1 >= 2^w holds for these shares)."""
    rng = np.random.default_rng(48)
    z = rng.uniform(-1, 1, toy.n)
    f, ft, w = 50, 50, 83
    s_out = f + toy.log_n - 40                     # Delta = 2^40
    y = [int(round(v * 2.0 ** f)) for v in z]
    y0 = [int(a) | (int(b) << 64) for a, b in zip(rng.integers(0, 2 ** 63, toy.n, dtype=np.uint64),
                                                  rng.integers(0, 2 ** 63, toy.n, dtype=np.uint64))]
    y1 = [(v - a) % (1 << 128) for v, a in zip(y, y0)]
    x0 = [v % (1 << w) for v in O.u128_to_int(O.share_encode(toy, O.int_to_u128(y0), ft, s_out))]
    x1 = [v % (1 << w) for v in O.u128_to_int(O.share_encode(toy, O.int_to_u128(y1), ft, s_out))]
    # coefficient N/2 of the encode of ANY real vector is exactly 0 (zeta^{-N/2 5^j} = +-i), so both
    # local encodes are 0 there and ring-to-field's success event x0 + x1 >= 2^w fails; the parties
    # re-randomise with a zero sharing (u from a shared PRF) first (reading C20)
    assert x0[toy.N // 2] == 0 and x1[toy.N // 2] == 0
    u = [int(a) | (int(b) << 64) for a, b in zip(rng.integers(0, 2 ** 63, toy.N, dtype=np.uint64),
                                                 rng.integers(0, 2 ** 63, toy.N, dtype=np.uint64))]
    x0 = [(a + r) % (1 << w) for a, r in zip(x0, u)]
    x1 = [(b - r) % (1 << w) for b, r in zip(x1, u)]
    keys = O.keygen(toy, bi.crypto_key(4, 49))
    lvl = 2
    f0 = O.share_to_rns(toy, O.int_to_u128(x0), w, False, lvl)
    ct = O.encrypt(toy, bi.crypto_key(5, 49), keys.s_ntt, f0, lvl, 3, 2.0 ** 40)
    out = O.mpc_to_ckks(toy, ct, O.int_to_u128(x1), w)
    dec = O.decode(toy, O.decrypt(toy, keys.s_ntt, out), out.scale)
    assert np.abs(dec - z).max() < 1e-6
