"""CPU pin of the exactness argument behind the grid-split FP64 accumulator AccG
(paper_2508_19525_b200/csrc/blb_internal.cuh): its device formula is replayed
here in IEEE double arithmetic (Python floats; fma evaluated exactly with Fraction and rounded
once, round-half-even) and compared with the exact integer sum of the products.  This checks
the bounds the kernels rely on -- running sum s in [2^92, 2^93) for <= 512 products of residues
< 2^41, every rounding error recovered exactly -- independently of any GPU."""
from fractions import Fraction

import numpy as np
import pytest

M = 1.5 * 2.0 ** 92
MAGIC = 6755399441055744.0  # 1.5 * 2^52


def fma(a: float, b: float, c: float) -> float:
    return float(Fraction(a) * Fraction(b) + Fraction(c))  # exact, then one correct rounding


def accg_sum(A, B):
    """AccG.macd over the products A[t] * B[t]: returns (s, l)."""
    s, l = M, 0.0
    for a, b in zip(A, B):
        sn = fma(a, b, s)
        l = l + fma(a, b, s - sn)
        s = sn
    return s, l


def accg_rem(s, l, q):
    """AccG.rem: (s - M) + l reduced to a double congruent mod q, |value| < q + 2^49."""
    qd, qinv = float(q), 1.0 / float(q)
    Hd = (s - M) * 2.0 ** -40
    Hm = fma(-(fma(Hd, qinv, MAGIC) - MAGIC), qd, Hd)
    two40 = float(2 ** 40)
    c40 = fma(-(fma(two40, qinv, MAGIC) - MAGIC), qd, two40)
    p = Hm * c40
    e = fma(Hm, c40, -p)
    c = fma(p, qinv, MAGIC) - MAGIC
    return (fma(-c, qd, p) + e) + l


@pytest.mark.parametrize("seed,n,top", [(1, 512, 41), (2, 512, 40), (3, 7, 41), (4, 100, 41)])
def test_accg_sum_is_exact(seed, n, top):
    rng = np.random.default_rng(seed)
    A = [int(x) for x in rng.integers(0, 2 ** top, n, dtype=np.int64)]
    B = [int(x) for x in rng.integers(0, 2 ** top, n, dtype=np.int64)]
    if seed == 1:  # the extreme: every product at the top of the range
        A = [2 ** 41 - 1] * n
        B = [2 ** 41 - 1] * n
    s, l = accg_sum([float(a) for a in A], [float(b) for b in B])
    assert 2.0 ** 92 <= s < 2.0 ** 93
    assert abs(l) < 2.0 ** 49
    assert Fraction(s) - Fraction(M) + Fraction(l) == sum(a * b for a, b in zip(A, B))


@pytest.mark.parametrize("seed", [5, 6, 7])
def test_accg_remainder_mod_q(seed):
    import oracle as O
    q = O.prime_chain(16, [60, 40])[1]  # the BERT chain's first 40-bit prime (q = 1 mod 2^17)
    assert q.bit_length() == 40 and q % (2 ** 17) == 1
    rng = np.random.default_rng(seed)
    A = [int(x) for x in rng.integers(0, q, 512, dtype=np.int64)]
    B = [int(x) for x in rng.integers(0, q, 512, dtype=np.int64)]
    s, l = accg_sum([float(a) for a in A], [float(b) for b in B])
    r = accg_rem(s, l, q)
    assert r == int(r) and abs(r) < q + 2 ** 49
    assert int(r) % q == sum(a * b for a, b in zip(A, B)) % q


def accg_fold(s, l, q):
    """AccG.fold: s = M, l = rem(s, l) re-centred mod q."""
    qd, qinv = float(q), 1.0 / float(q)
    r = accg_rem(s, l, q)
    c = fma(r, qinv, MAGIC) - MAGIC
    return M, fma(-c, qd, r)


def test_accg_many_folds_stay_exact():
    """64 fold periods of 512 top-range products (32k products per accumulator, twice the point
    where an unreduced l would pass 2^53): every fold keeps |l| <= q/2 + 1 and the final
    remainder is the exact sum mod q."""
    import oracle as O
    q = O.prime_chain(16, [60, 40])[1]
    qd, qinv = float(q), 1.0 / float(q)
    s, l = M, 0.0
    exact = 0
    a = float(q - 1)
    for period in range(64):
        for _ in range(512):
            sn = fma(a, a, s)
            l = l + fma(a, a, s - sn)
            s = sn
        exact += 512 * (q - 1) ** 2
        s, l = accg_fold(s, l, q)
        assert s == M and l == int(l) and abs(l) <= q / 2 + 1
    assert int(accg_rem(s, l, q)) % q == exact % q
