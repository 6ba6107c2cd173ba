"""Oracle pins: CKKS encode / decode (Eq. eq:ckks_encode; C3) against
mpmath direct evaluation, the SURVEY KAT, closed forms and round trips."""
import json
import os

import mpmath
import numpy as np
import pytest

import oracle as O

KAT = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "encode_kat.json")))


def ctx_for(logn):
    q = O.prime_chain(logn, [60, 50, 50, 60])
    return O.Ctx(logn, q[:3], q[3:], 3)


def exact_scaled(z, k, N, delta, dps=50):
    """Delta * m_k = Delta * (2/N) sum_j z_j cos(pi (k 5^j mod 2N) / N), in mpmath."""
    with mpmath.workdps(dps):
        acc = mpmath.mpf(0)
        e = 1
        for j in range(N // 2):
            a = (k * e) % (2 * N)
            acc += mpmath.mpf(z[j]) * mpmath.cos(mpmath.pi * a / N)
            e = e * 5 % (2 * N)
        return acc * 2 / N * mpmath.mpf(delta)


def round_half_even(x):
    with mpmath.workdps(60):
        f = mpmath.floor(x)
        r = x - f
        if r > 0.5 or (r == 0.5 and int(f) % 2 == 1):
            return int(f) + 1
        return int(f)


def test_encode_matches_mpmath_small():
    c = ctx_for(5)
    rng = np.random.default_rng(7)
    z = rng.uniform(-1, 1, c.n)
    delta = 2.0 ** 30
    got = O.encode_coeffs(c, z, delta)
    ref = [round_half_even(exact_scaled(z, k, c.N, delta)) for k in range(c.N)]
    assert got.tolist() == ref
    assert O.encode_direct(c, z, delta).tolist() == ref


def test_encode_kat_n4096():
    c = ctx_for(KAT["log_n"])
    z = np.arange(c.n) / c.n
    delta = 2.0 ** KAT["log_delta"]
    got = O.encode_coeffs(c, z, delta)
    for k, exact_str, rounded in KAT["rows"]:
        assert int(got[k]) == rounded
        ex = exact_scaled(z, k, c.N, delta, dps=40)
        assert abs(ex - mpmath.mpf(exact_str)) < 1e-6
        assert round_half_even(ex) == rounded


def test_encode_fft_equals_direct_n1024():
    c = ctx_for(10)
    z = np.random.default_rng(3).normal(0, 1, c.n)
    assert np.array_equal(O.encode_coeffs(c, z, 2.0 ** 40), O.encode_direct(c, z, 2.0 ** 40))


def test_encode_constant_and_zero():
    c = ctx_for(10)
    coef = O.encode_coeffs(c, np.full(c.n, 0.75), 2.0 ** 40)
    assert coef[0] == int(0.75 * 2 ** 40) and not coef[1:].any()
    assert not O.encode_coeffs(c, np.zeros(c.n), 2.0 ** 40).any()
    # ties-to-even on an exactly representable half: 2.5 * 2^0 scale 1 -> 2
    coef = O.encode_coeffs(c, np.full(c.n, 2.5), 1.0)
    assert coef[0] == 2
    coef = O.encode_coeffs(c, np.full(c.n, 3.5), 1.0)
    assert coef[0] == 4


def test_encode_overflow():
    c = ctx_for(5)
    with pytest.raises(O.EncodeOverflow):
        O.encode_coeffs(c, np.full(c.n, 4.0), 2.0 ** 61)


def test_decode_matches_direct_sum():
    c = ctx_for(5)
    rng = np.random.default_rng(11)
    coef = rng.integers(-2**40, 2**40, c.N)
    got = O.decode_coeffs(c, coef.tolist(), 2.0 ** 30)
    N = c.N
    ref = []
    for j in range(c.n):
        e = pow(5, j, 2 * N)
        ref.append(sum(float(coef[k]) * np.cos(np.pi * ((k * e) % (2 * N)) / N) for k in range(N)) / 2.0 ** 30)
    assert np.allclose(got, ref, rtol=0, atol=1e-9)


@pytest.mark.parametrize("logn", [5, 12])
def test_decode_encode_roundtrip(logn):
    c = ctx_for(logn)
    z = np.random.default_rng(logn).uniform(-1, 1, c.n)
    delta = 2.0 ** 40
    pt = O.encode(c, z, delta, 2)
    back = O.decode(c, pt, delta)
    assert np.abs(back - z).max() < c.N / delta
    # level-0 decode (single prime) gives the same values
    assert np.allclose(O.decode(c, pt[:1], delta), back, atol=1e-12)
