// host_tables.cpp -- host-side setup tables of the B200 BLB library (row a0).
// Compiled by g++ (needs __float128 / libquadmath for the double-double
// encode twiddles).  Product code: independent of oracle/.
//
//   * primes by the C1 rule (largest unused p < 2^b, p == 1 mod 2N),
//   * psi = minimal primitive 2N-th root (C1),
//   * bit-reversed twiddle tables with Shoup companions (C2),
//   * zeta^{brv(i)} = exp(i pi brv(i) / N) as double-double pairs (C3).
#include <stdint.h>
#include <string.h>
#include <quadmath.h>

typedef uint64_t u64;
typedef unsigned __int128 u128;

static u64 mm(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
static u64 pw(u64 a, u64 e, u64 q) {
    u64 r = 1 % q;
    a %= q;
    while (e) {
        if (e & 1) r = mm(r, a, q);
        a = mm(a, a, q);
        e >>= 1;
    }
    return r;
}

extern "C" int blbh_is_prime(u64 n) {
    if (n < 2) return 0;
    static const u64 bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    for (u64 b : bases) {
        if (n % b == 0) return n == b;
    }
    u64 d = n - 1;
    int s = 0;
    while (!(d & 1)) { d >>= 1; ++s; }
    for (u64 a : bases) {
        u64 x = pw(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool witness = true;
        for (int r = 1; r < s && witness; ++r) {
            x = mm(x, x, n);
            if (x == n - 1) witness = false;
        }
        if (witness) return 0;
    }
    return 1;
}

extern "C" int blbh_prime_chain(int logN, const int *bits, int count, u64 *out) {
    const u64 step = 2ull << logN;
    for (int c = 0; c < count; ++c) {
        if (bits[c] < logN + 2 || bits[c] > 61) return -1;
        const u64 limit = 1ull << bits[c];
        u64 cand = ((limit - 1) / step) * step + 1;
        if (cand >= limit) cand -= step;
        for (;;) {
            bool taken = false;
            for (int u = 0; u < c; ++u) taken |= (out[u] == cand);
            if (!taken && blbh_is_prime(cand)) break;
            if (cand <= step) return -2;
            cand -= step;
        }
        out[c] = cand;
    }
    return 0;
}

// minimal x with x^N == -1 mod q, searched over the odd powers of one root
extern "C" u64 blbh_min_psi(u64 q, int logN) {
    const u64 N = 1ull << logN, twoN = N << 1;
    if ((q - 1) % twoN) return 0;
    u64 root = 0;
    for (u64 g = 2; g < q && !root; ++g) {
        u64 cand = pw(g, (q - 1) / twoN, q);
        if (pw(cand, N, q) == q - 1) root = cand;
    }
    const u64 sq = mm(root, root, q);
    u64 best = root, cur = root;
    for (u64 k = 1; k < N; ++k) {
        cur = mm(cur, sq, q);
        if (cur < best) best = cur;
    }
    return best;
}

static inline u64 bitrev(u64 x, int bits) {
    u64 r = 0;
    for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1ull) << (bits - 1 - i);
    return r;
}

extern "C" u64 blbh_shoup(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
extern "C" u64 blbh_mulmod(u64 a, u64 b, u64 q) { return mm(a, b, q); }
extern "C" u64 blbh_powmod(u64 a, u64 e, u64 q) { return pw(a, e, q); }
extern "C" u64 blbh_invmod(u64 a, u64 q) { return pw(a, q - 2, q); }

// out: [2][N][2] = (psi^{brv(i)}, Shoup) pairs, then (psi^{-brv(i)}, Shoup) pairs
extern "C" void blbh_twiddles(u64 q, u64 psi, int logN, u64 *out) {
    const u64 N = 1ull << logN;
    const u64 ipsi = pw(psi, q - 2, q);
    // powers in natural order, then scatter by bit reversal
    u64 f = 1, b = 1;
    for (u64 e = 0; e < N; ++e) {
        const u64 i = bitrev(e, logN);
        out[2 * i] = f;
        out[2 * i + 1] = blbh_shoup(f, q);
        out[2 * N + 2 * i] = b;
        out[2 * N + 2 * i + 1] = blbh_shoup(b, q);
        f = mm(f, psi, q);
        b = mm(b, ipsi, q);
    }
}

// out: [N][4] doubles = (Re hi, Re lo, Im hi, Im lo) of zeta^{brv(i)}, zeta = e^{i pi / N}
extern "C" void blbh_zeta_dd(int logN, double *out) {
    const u64 N = 1ull << logN;
    for (u64 i = 0; i < N; ++i) {
        const __float128 ang = M_PIq * (__float128)bitrev(i, logN) / (__float128)N;
        const __float128 c = cosq(ang), s = sinq(ang);
        const double ch = (double)c, sh = (double)s;
        out[4 * i + 0] = ch;
        out[4 * i + 1] = (double)(c - (__float128)ch);
        out[4 * i + 2] = sh;
        out[4 * i + 3] = (double)(s - (__float128)sh);
    }
}
