"""Oracle pins: prime chain and minimal psi (C1; SURVEY 8(c) KAT), checked with sympy."""
import json
import os

import pytest
import sympy

import oracle as O

KAT = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "kat_primes.json")))


@pytest.mark.parametrize("name", ["toy", "bert"])
def test_prime_chain_kat(name):
    k = KAT[name]
    assert O.prime_chain(k["log_n"], k["bits"]) == k["primes"]


@pytest.mark.parametrize("name", ["toy", "bert"])
def test_primes_are_largest_ntt_friendly(name):
    k = KAT[name]
    twoN = 2 << k["log_n"]
    used = []
    for q, b in zip(k["primes"], k["bits"]):
        assert sympy.isprime(q) and q % twoN == 1 and q < 2 ** b
        x = q + twoN
        while x < 2 ** b:  # every larger candidate is composite or already used
            assert (not sympy.isprime(x)) or x in used
            x += twoN
        used.append(q)
    assert len(set(k["primes"])) == len(k["primes"])


@pytest.mark.parametrize("name", ["toy", "bert"])
def test_min_psi_kat_and_minimality(name):
    k = KAT[name]
    N = 1 << k["log_n"]
    for q, psi in zip(k["primes"], k["psi"]):
        assert O.min_psi(q, k["log_n"]) == psi
        assert pow(psi, N, q) == q - 1
        # minimality over the set of all primitive 2N-th roots {r^k : k odd},
        # r derived from sympy's primitive root (independent of the oracle)
        g = sympy.primitive_root(q)
        r = pow(g, (q - 1) // (2 * N), q)
        r2 = r * r % q
        cur, best = r, r
        for _ in range(N):
            best = min(best, cur)
            cur = cur * r2 % q
        assert best == psi


def test_min_psi_bruteforce_small():
    for q, logn in [(17, 3), (97, 4), (193, 5), (257, 7)]:
        N = 1 << logn
        brute = min(x for x in range(2, q) if pow(x, N, q) == q - 1)
        assert O.min_psi(q, logn) == brute


def test_ctx_rejects_bad_params():
    q = O.prime_chain(5, [40, 40, 50])
    with pytest.raises(O.ParamError):
        O.Ctx(5, [q[0], q[0]], [q[2]], 2)            # duplicate prime
    with pytest.raises(O.ParamError):
        O.Ctx(5, [q[0], 1099511627791], [q[2]], 2)   # not 1 mod 2N
    with pytest.raises(O.ParamError):
        O.Ctx(5, [q[0], q[1]], [q[2]], 0)            # bad dnum
    c = O.Ctx(5, [q[0], q[1]], [q[2]], 1)
    assert c.alpha == 2 and c.beta_top == 1
