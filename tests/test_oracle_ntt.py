"""Oracle pins: negacyclic NTT (C2), automorphisms (C3), by closed form and brute force."""
import numpy as np
import pytest

import oracle as O


def brv(x, bits):
    return int(format(x, "0%db" % bits)[::-1], 2)


def closed_form_ntt(a, psi, q, logn, ks=None):
    N = 1 << logn
    ks = range(N) if ks is None else ks
    out = {}
    for k in ks:
        w = pow(psi, 2 * brv(k, logn) + 1, q)
        acc, wj = 0, 1
        for j in range(N):
            acc += int(a[j]) * wj
            wj = wj * w % q
        out[k] = acc % q
    return out


def negacyclic_py(a, b, q):
    N = len(a)
    out = [0] * N
    for i in range(N):
        for j in range(N):
            v = int(a[i]) * int(b[j])
            if i + j < N:
                out[i + j] += v
            else:
                out[i + j - N] -= v
    return [x % q for x in out]


@pytest.fixture(scope="module")
def tiny():
    q = O.prime_chain(5, [50, 40, 40, 60])
    return O.Ctx(5, q[:3], q[3:], 3)


@pytest.fixture(scope="module")
def mid():
    q = O.prime_chain(10, [60, 40, 61])
    return O.Ctx(10, q[:2], q[2:], 2)


def test_ntt_closed_form_tiny(tiny):
    rng = np.random.default_rng(0)
    for i, q in enumerate(tiny.mods):
        a = rng.integers(0, q, tiny.N, dtype=np.uint64)
        got = tiny.ntt(a[None, :], [i])[0]
        ref = closed_form_ntt(a, tiny.psi[i], q, 5)
        assert [int(x) for x in got] == [ref[k] for k in range(tiny.N)]


def test_ntt_closed_form_n1024_sampled(mid):
    rng = np.random.default_rng(1)
    q = mid.mods[0]
    a = rng.integers(0, q, mid.N, dtype=np.uint64)
    got = mid.ntt(a[None, :], [0])[0]
    ks = [0, 1, 2, 511, 512, 1000, 1023]
    ref = closed_form_ntt(a, mid.psi[0], q, 10, ks)
    assert all(int(got[k]) == ref[k] for k in ks)


def test_ntt_special_inputs(mid):
    for i, q in enumerate(mid.mods):
        one = np.zeros(mid.N, dtype=np.uint64); one[0] = 1
        assert np.all(mid.ntt(one[None], [i])[0] == 1)
        x = np.zeros(mid.N, dtype=np.uint64); x[1] = 1
        got = mid.ntt(x[None], [i])[0]
        assert all(int(got[k]) == pow(mid.psi[i], 2 * brv(k, 10) + 1, q) for k in range(mid.N))


@pytest.mark.parametrize("logn", [5, 12, 16])
def test_ntt_roundtrip(logn):
    q = O.prime_chain(logn, [60, 40, 61])
    c = O.Ctx(logn, q[:2], q[2:], 2)
    rng = np.random.default_rng(logn)
    a = np.stack([rng.integers(0, m, c.N, dtype=np.uint64) for m in c.mods])
    idx = list(range(3))
    assert np.array_equal(c.intt(c.ntt(a, idx), idx), a)
    assert not np.array_equal(c.ntt(a, idx), a)


def test_pointwise_is_negacyclic_bruteforce(tiny):
    rng = np.random.default_rng(2)
    for i, q in enumerate(tiny.mods):
        a = rng.integers(0, q, tiny.N, dtype=np.uint64)
        b = rng.integers(0, q, tiny.N, dtype=np.uint64)
        ref = negacyclic_py(a, b, q)
        assert [int(x) for x in O.schoolbook(a, b, q)] == ref
        fa, fb = tiny.ntt(a[None], [i])[0], tiny.ntt(b[None], [i])[0]
        prod = np.array([int(x) * int(y) % q for x, y in zip(fa, fb)], dtype=np.uint64)
        assert [int(x) for x in tiny.intt(prod[None], [i])[0]] == ref


def test_pointwise_is_negacyclic_n1024(mid):
    rng = np.random.default_rng(3)
    q = mid.mods[1]
    a = rng.integers(0, q, mid.N, dtype=np.uint64)
    b = rng.integers(0, q, mid.N, dtype=np.uint64)
    fa, fb = mid.ntt(a[None], [1])[0], mid.ntt(b[None], [1])[0]
    prod = np.array([int(x) * int(y) % q for x, y in zip(fa, fb)], dtype=np.uint64)
    assert np.array_equal(mid.intt(prod[None], [1])[0], O.schoolbook(a, b, q))


def test_automorphism_ntt_equals_coefficient_map(mid):
    rng = np.random.default_rng(4)
    for i, q in enumerate(mid.mods):
        a = rng.integers(0, q, mid.N, dtype=np.uint64)
        fa = mid.ntt(a[None], [i])
        for g in [mid.galois(1), mid.galois(7), mid.galois(-3), 2 * mid.N - 1]:
            lhs = mid.ntt(O.automorphism_coef(a, g, q)[None], [i])
            rhs = mid.automorphism_ntt(fa, g)
            assert np.array_equal(lhs, rhs)


def test_automorphism_coef_definition():
    # a(X) = X  ->  X^g ; with g >= N the sign flips (X^N = -1)
    N, q = 8, 17
    a = np.zeros(N, dtype=np.uint64); a[1] = 1
    out = O.automorphism_coef(a, 5, q)
    assert out[5] == 1 and out.sum() == 1
    out = O.automorphism_coef(a, 11, q)   # X^11 = -X^3
    assert out[3] == 16 and out.sum() == 16


def test_galois_rotation_group():
    q = O.prime_chain(10, [60, 61])
    c = O.Ctx(10, q[:1], q[1:], 1)
    assert c.galois(0) == 1 and c.galois(c.n) == 1       # 5 has order n mod 2N
    assert c.galois(3) * c.galois(-3) % (2 * c.N) == 1
