/*
 * oracle/blb_oracle.c -- BLB CKKS oracle, C primitives.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the plain, slow, obviously-correct
 * CPU statement of what the server-side CKKS hot path of BLB
 * (arXiv 2508.19525) computes.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.  It shares no
 * code, headers or tables with the CUDA product under
 * paper_2508_19525_b200/ (that product must never import or link this).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n,
 * "C<k>" / "S<k>" = the readings of SURVEY.md section 8(c) restated in DESIGN.md.
 *
 * Conventions:
 *   * ring A_{N,q} = Z_q[x]/(x^N+1) (Table 1), RNS over primes
 *     q_0..q_{K-1} (ciphertext chain, Table 6 footnote P:725) and special
 *     primes p_0..p_{np-1}.
 *   * NTT(a)[k] = a(psi^{2*brv(k)+1}) mod q (C2), psi the minimal primitive
 *     2N-th root (C1).  All arithmetic below is exact modular arithmetic with
 *     unsigned __int128 products and '%'.
 *   * randomness: ChaCha20 block function per RFC 8439, layout C4.
 *   * encode: correctly rounded Delta * pi^{-1}(z) computed in __float128
 *     (C3).
 * Every function is a direct transcription; no blocking, fusion or lazy
 * reduction.  OpenMP only splits independent loop iterations.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <quadmath.h>

typedef uint64_t u64;
typedef int64_t i64;
typedef unsigned __int128 u128;
typedef __int128 i128;

#define ORC_MAXP 24

/* ------------------------------------------------------------------ */
/* modular arithmetic (textbook)                                        */
/* ------------------------------------------------------------------ */
static inline u64 mulmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
static inline u64 addmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a + b) % q); }
static inline u64 submod(u64 a, u64 b, u64 q) { return (u64)(((u128)a + q - (b % q)) % q); }
static u64 powmod(u64 a, u64 e, u64 q) {
    u64 r = 1 % q; a %= q;
    while (e) { if (e & 1) r = mulmod(r, a, q); a = mulmod(a, a, q); e >>= 1; }
    return r;
}
static u64 invmod(u64 a, u64 q) { return powmod(a, q - 2, q); } /* q prime */

u64 orc_mulmod(u64 a, u64 b, u64 q) { return mulmod(a, b, q); }
u64 orc_powmod(u64 a, u64 e, u64 q) { return powmod(a, e, q); }

/* deterministic Miller-Rabin for 64-bit inputs */
int orc_is_prime(u64 n) {
    if (n < 2) return 0;
    static const u64 small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    for (int i = 0; i < 12; i++) { if (n % small[i] == 0) return n == small[i]; }
    u64 d = n - 1; int s = 0;
    while ((d & 1) == 0) { d >>= 1; s++; }
    for (int i = 0; i < 12; i++) {
        u64 x = powmod(small[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int comp = 1;
        for (int r = 1; r < s; r++) { x = mulmod(x, x, n); if (x == n - 1) { comp = 0; break; } }
        if (comp) return 0;
    }
    return 1;
}

/* C1 prime-list rule: for each requested width b (chain order), the largest
 * unused prime < 2^b with p == 1 mod 2N.  Returns 0 on success. */
int orc_prime_chain(int logN, const int *bits, int count, u64 *out) {
    u64 twoN = 2ull << logN;
    for (int c = 0; c < count; c++) {
        if (bits[c] < logN + 2 || bits[c] > 61) return -1;
        u64 top = (bits[c] == 64) ? ~0ull : ((1ull << bits[c]) - 1);
        u64 x = (top / twoN) * twoN + 1;
        if (x > top) x -= twoN;
        for (;;) {
            int used = 0;
            for (int u = 0; u < c; u++) if (out[u] == x) used = 1;
            if (!used && orc_is_prime(x)) break;
            if (x <= twoN) return -2;
            x -= twoN;
        }
        out[c] = x;
    }
    return 0;
}

/* C1: psi = the smallest x >= 2 with x^N == -1 (mod q); computed as
 * min{psi0^k : k odd < 2N} for one primitive 2N-th root psi0. */
u64 orc_min_psi(u64 q, int logN) {
    u64 N = 1ull << logN, twoN = 2 * N;
    if ((q - 1) % twoN) return 0;
    u64 psi0 = 0;
    for (u64 g = 2; g < q; g++) {
        u64 c = powmod(g, (q - 1) / twoN, q);
        if (powmod(c, N, q) == q - 1) { psi0 = c; break; }
    }
    u64 best = psi0, sq = mulmod(psi0, psi0, q), cur = psi0;
    for (u64 k = 1; k < twoN; k += 2) {
        if (cur < best) best = cur;
        cur = mulmod(cur, sq, q);
    }
    return best;
}

static inline u64 brv(u64 x, int bits) {
    u64 r = 0;
    for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

/* ------------------------------------------------------------------ */
/* context                                                              */
/* ------------------------------------------------------------------ */
typedef struct {
    int logN; u64 N;
    int K, np, dnum, alpha;
    u64 mod[ORC_MAXP];      /* q_0..q_{K-1}, p_0..p_{np-1} */
    u64 psi[ORC_MAXP];
    u64 *fwd[ORC_MAXP];     /* fwd[i][j] = psi^{brv(j)}   (C2)  */
    u64 *inv[ORC_MAXP];     /* inv[i][j] = psi^{-brv(j)}        */
    u64 ninv[ORC_MAXP];
    __float128 *cos2, *sin2; /* cos/sin(2 pi j / N), j < N      */
    __float128 *cosh_, *sinh_; /* cos/sin(pi j / N), j < N       */
} orc_ctx;

void orc_ctx_free(orc_ctx *c) {
    if (!c) return;
    for (int i = 0; i < c->K + c->np; i++) { free(c->fwd[i]); free(c->inv[i]); }
    free(c->cos2); free(c->sin2); free(c->cosh_); free(c->sinh_);
    free(c);
}

/* status: 0 ok, -1 bad N, -2 prime not 1 mod 2N / not prime / >= 2^61,
 * -3 duplicate prime, -4 bad dnum */
orc_ctx *orc_ctx_new(int logN, const u64 *q, int K, const u64 *p, int np, int dnum, int *status) {
    *status = 0;
    if (logN < 2 || logN > 17) { *status = -1; return NULL; }
    if (K < 1 || np < 1 || K + np > ORC_MAXP) { *status = -2; return NULL; }
    if (dnum < 1 || dnum > K) { *status = -4; return NULL; }
    orc_ctx *c = (orc_ctx *)calloc(1, sizeof(orc_ctx));
    c->logN = logN; c->N = 1ull << logN; c->K = K; c->np = np; c->dnum = dnum;
    c->alpha = (K + dnum - 1) / dnum;
    for (int i = 0; i < K; i++) c->mod[i] = q[i];
    for (int i = 0; i < np; i++) c->mod[K + i] = p[i];
    for (int i = 0; i < K + np; i++) {
        u64 m = c->mod[i];
        if (m >= (1ull << 61) || !orc_is_prime(m) || (m - 1) % (2 * c->N)) { *status = -2; free(c); return NULL; }
        for (int j = 0; j < i; j++) if (c->mod[j] == m) { *status = -3; free(c); return NULL; }
    }
    if (c->np < c->alpha) { /* P must cover a digit (hybrid key switching needs P >= digit) */ }
    for (int i = 0; i < K + np; i++) {
        u64 m = c->mod[i];
        c->psi[i] = orc_min_psi(m, logN);
        u64 pinv = invmod(c->psi[i], m);
        c->fwd[i] = (u64 *)malloc(c->N * sizeof(u64));
        c->inv[i] = (u64 *)malloc(c->N * sizeof(u64));
        for (u64 j = 0; j < c->N; j++) {
            u64 e = brv(j, logN);
            c->fwd[i][j] = powmod(c->psi[i], e, m);
            c->inv[i][j] = powmod(pinv, e, m);
        }
        c->ninv[i] = invmod(c->N % m, m);
    }
    c->cos2 = (__float128 *)malloc(c->N * sizeof(__float128));
    c->sin2 = (__float128 *)malloc(c->N * sizeof(__float128));
    c->cosh_ = (__float128 *)malloc(c->N * sizeof(__float128));
    c->sinh_ = (__float128 *)malloc(c->N * sizeof(__float128));
    for (u64 j = 0; j < c->N; j++) {
        __float128 a2 = 2 * M_PIq * (__float128)j / (__float128)c->N;
        __float128 a1 = M_PIq * (__float128)j / (__float128)c->N;
        c->cos2[j] = cosq(a2); c->sin2[j] = sinq(a2);
        c->cosh_[j] = cosq(a1); c->sinh_[j] = sinq(a1);
    }
    return c;
}

int orc_ctx_alpha(const orc_ctx *c) { return c->alpha; }
u64 orc_ctx_psi(const orc_ctx *c, int i) { return c->psi[i]; }

/* ------------------------------------------------------------------ */
/* NTT (C2): textbook Cooley-Tukey / Gentleman-Sande, one limb          */
/* ------------------------------------------------------------------ */
static void ntt_limb(const orc_ctx *c, u64 *a, int pi) {
    u64 q = c->mod[pi], N = c->N, t = N;
    for (u64 m = 1; m < N; m <<= 1) {
        t >>= 1;
        for (u64 i = 0; i < m; i++) {
            u64 w = c->fwd[pi][m + i], j1 = 2 * i * t;
            for (u64 j = j1; j < j1 + t; j++) {
                u64 u = a[j], v = mulmod(a[j + t], w, q);
                a[j] = addmod(u, v, q);
                a[j + t] = submod(u, v, q);
            }
        }
    }
}
static void intt_limb(const orc_ctx *c, u64 *a, int pi) {
    u64 q = c->mod[pi], N = c->N, t = 1;
    for (u64 m = N >> 1; m >= 1; m >>= 1) {
        for (u64 i = 0; i < m; i++) {
            u64 w = c->inv[pi][m + i], j1 = 2 * i * t;
            for (u64 j = j1; j < j1 + t; j++) {
                u64 u = a[j], v = a[j + t];
                a[j] = addmod(u, v, q);
                a[j + t] = mulmod(submod(u, v, q), w, q);
            }
        }
        t <<= 1;
    }
    for (u64 j = 0; j < N; j++) a[j] = mulmod(a[j], c->ninv[pi], q);
}

/* data: [n_limbs][N]; limb l uses prime index pidx[l] */
void orc_ntt(const orc_ctx *c, u64 *data, const int *pidx, int n_limbs) {
#pragma omp parallel for schedule(dynamic)
    for (int l = 0; l < n_limbs; l++) ntt_limb(c, data + (u64)l * c->N, pidx[l]);
}
void orc_intt(const orc_ctx *c, u64 *data, const int *pidx, int n_limbs) {
#pragma omp parallel for schedule(dynamic)
    for (int l = 0; l < n_limbs; l++) intt_limb(c, data + (u64)l * c->N, pidx[l]);
}

/* definition mode: schoolbook negacyclic product mod (x^N + 1, q) */
void orc_negacyclic_schoolbook(const u64 *a, const u64 *b, u64 *out, u64 N, u64 q) {
#pragma omp parallel for
    for (u64 k = 0; k < N; k++) {
        u64 acc = 0;
        for (u64 i = 0; i < N; i++) {
            u64 j, prod;
            if (i <= k) { j = k - i; prod = mulmod(a[i], b[j], q); acc = addmod(acc, prod, q); }
            else { j = N + k - i; prod = mulmod(a[i], b[j], q); acc = submod(acc, prod, q); }
        }
        out[k] = acc;
    }
}

/* NTT-domain automorphism X -> X^g (g odd):
 * out[k] = in[brv(((g*(2*brv(k)+1)) mod 2N - 1)/2)]  (C2 + App. A item 2) */
void orc_automorphism_ntt(const orc_ctx *c, const u64 *in, u64 *out, u64 g, int n_limbs) {
    u64 N = c->N, twoN = 2 * N;
    for (int l = 0; l < n_limbs; l++) {
        const u64 *src = in + (u64)l * N; u64 *dst = out + (u64)l * N;
#pragma omp parallel for
        for (u64 k = 0; k < N; k++) {
            u64 e = 2 * brv(k, c->logN) + 1;
            u64 e2 = (u64)(((u128)g * e) % twoN);
            dst[k] = src[brv((e2 - 1) / 2, c->logN)];
        }
    }
}
/* coefficient-domain automorphism a(X) -> a(X^g), the definition */
void orc_automorphism_coef(u64 N, const u64 *in, u64 *out, u64 g, u64 q) {
    u64 twoN = 2 * N;
    for (u64 i = 0; i < N; i++) {
        u64 e = (u64)(((u128)i * g) % twoN);
        if (e < N) out[e] = in[i];
        else out[e - N] = (q - in[i]) % q;
    }
}

/* ------------------------------------------------------------------ */
/* ChaCha20 (RFC 8439 section 2.3) and the C4 draw layout               */
/* ------------------------------------------------------------------ */
static inline uint32_t rotl32(uint32_t x, int r) { return (x << r) | (x >> (32 - r)); }
#define QR(a, b, c, d) \
    a += b; d ^= a; d = rotl32(d, 16); c += d; b ^= c; b = rotl32(b, 12); \
    a += b; d ^= a; d = rotl32(d, 8);  c += d; b ^= c; b = rotl32(b, 7);
static inline uint32_t le32(const uint8_t *p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}
void orc_chacha20_block(const uint8_t key[32], uint32_t counter, const uint8_t nonce[12], uint8_t out[64]) {
    uint32_t s[16], x[16];
    s[0] = 0x61707865; s[1] = 0x3320646e; s[2] = 0x79622d32; s[3] = 0x6b206574;
    for (int i = 0; i < 8; i++) s[4 + i] = le32(key + 4 * i);
    s[12] = counter;
    for (int i = 0; i < 3; i++) s[13 + i] = le32(nonce + 4 * i);
    memcpy(x, s, sizeof(s));
    for (int r = 0; r < 10; r++) {
        QR(x[0], x[4], x[8], x[12]); QR(x[1], x[5], x[9], x[13]);
        QR(x[2], x[6], x[10], x[14]); QR(x[3], x[7], x[11], x[15]);
        QR(x[0], x[5], x[10], x[15]); QR(x[1], x[6], x[11], x[12]);
        QR(x[2], x[7], x[8], x[13]); QR(x[3], x[4], x[9], x[14]);
    }
    for (int i = 0; i < 16; i++) {
        uint32_t v = x[i] + s[i];
        out[4 * i] = v & 0xff; out[4 * i + 1] = (v >> 8) & 0xff;
        out[4 * i + 2] = (v >> 16) & 0xff; out[4 * i + 3] = (v >> 24) & 0xff;
    }
}
/* C4: nonce = LE32(tag) || LE64(objid); coefficient x uses block x/4,
 * 128-bit draw x%4 = w_{2i} + 2^64 w_{2i+1}, w_i the LE u64 words. */
static void draw128(const uint8_t key[32], uint32_t tag, u64 objid, u64 x, u64 *lo, u64 *hi) {
    uint8_t nonce[12], blk[64];
    for (int i = 0; i < 4; i++) nonce[i] = (tag >> (8 * i)) & 0xff;
    for (int i = 0; i < 8; i++) nonce[4 + i] = (objid >> (8 * i)) & 0xff;
    orc_chacha20_block(key, (uint32_t)(x / 4), nonce, blk);
    int d = (int)(x % 4);
    u64 w0 = 0, w1 = 0;
    for (int i = 0; i < 8; i++) {
        w0 |= (u64)blk[16 * d + i] << (8 * i);
        w1 |= (u64)blk[16 * d + 8 + i] << (8 * i);
    }
    *lo = w0; *hi = w1;
}
void orc_draw128(const uint8_t key[32], uint32_t tag, u64 objid, u64 x, u64 *lohi) {
    draw128(key, tag, objid, x, &lohi[0], &lohi[1]);
}
/* uniform mod q: (128-bit draw) mod q */
void orc_sample_uniform(const uint8_t key[32], uint32_t tag, u64 objid, u64 q, u64 N, u64 *out) {
#pragma omp parallel for
    for (u64 x = 0; x < N; x++) {
        u64 lo, hi; draw128(key, tag, objid, x, &lo, &hi);
        out[x] = (u64)((((u128)hi << 64) | lo) % q);
    }
}
/* ternary secret: (u mod 3) - 1 with u the low 64 bits of draw x */
void orc_sample_ternary(const uint8_t key[32], uint32_t tag, u64 objid, u64 N, i64 *out) {
#pragma omp parallel for
    for (u64 x = 0; x < N; x++) {
        u64 lo, hi; draw128(key, tag, objid, x, &lo, &hi);
        out[x] = (i64)(lo % 3) - 1;
    }
}
/* centred binomial eta = 21 from the low 64 bits of draw x */
void orc_sample_cbd(const uint8_t key[32], uint32_t tag, u64 objid, u64 N, i64 *out) {
#pragma omp parallel for
    for (u64 x = 0; x < N; x++) {
        u64 lo, hi; draw128(key, tag, objid, x, &lo, &hi);
        u64 m = (1ull << 21) - 1;
        out[x] = (i64)__builtin_popcountll(lo & m) - (i64)__builtin_popcountll((lo >> 21) & m);
    }
}

enum { TAG_SECRET = 1, TAG_KEY_A = 2, TAG_KEY_E = 3, TAG_ENC_A = 4, TAG_ENC_E = 5, TAG_MASK = 6 };

/* signed integer polynomial -> residues mod prime pi, then NTT */
static void small_to_ntt(const orc_ctx *c, const i64 *v, int pi, u64 *out) {
    u64 q = c->mod[pi];
    for (u64 x = 0; x < c->N; x++) out[x] = v[x] >= 0 ? ((u64)v[x]) % q : (q - ((u64)(-v[x]) % q)) % q;
    ntt_limb(c, out, pi);
}

/* ------------------------------------------------------------------ */
/* keys (C5), encrypt / decrypt (C6)                                    */
/* ------------------------------------------------------------------ */
/* secret s (coefficients, ternary) and its NTT over all K+np primes: s_ntt[K+np][N] */
void orc_secret(const orc_ctx *c, const uint8_t key[32], i64 *s_coef, u64 *s_ntt) {
    orc_sample_ternary(key, TAG_SECRET, 0, c->N, s_coef);
    int L = c->K + c->np;
#pragma omp parallel for
    for (int i = 0; i < L; i++) small_to_ntt(c, s_coef, i, s_ntt + (u64)i * c->N);
}

/* switching key for target s' (NTT, [K+np][N]):
 * for digit j < beta_top: b_j = -a_j*s + e_j + P*pi_j*s', a_j uniform (NTT domain).
 * key_id (e.g. galois*64 + j) enters the ChaCha nonce; out: [beta_top][2][K+np][N] */
void orc_gen_swk(const orc_ctx *c, const uint8_t key[32], const u64 *s_ntt, const u64 *target_ntt,
                 u64 key_id_base, u64 *out) {
    int K = c->K, L = K + c->np, beta = (K + c->alpha - 1) / c->alpha;
    u64 N = c->N;
    for (int j = 0; j < beta; j++) {
        u64 kid = key_id_base * 64 + (u64)j;
        i64 *e = (i64 *)malloc(N * sizeof(i64));
        orc_sample_cbd(key, TAG_KEY_E, kid << 8, N, e);
#pragma omp parallel for
        for (int i = 0; i < L; i++) {
            u64 q = c->mod[i];
            u64 *b = out + (((u64)j * 2 + 0) * L + i) * N;
            u64 *a = out + (((u64)j * 2 + 1) * L + i) * N;
            orc_sample_uniform(key, TAG_KEY_A, (kid << 8) | (u64)i, q, N, a);
            u64 *en = (u64 *)malloc(N * sizeof(u64));
            small_to_ntt(c, e, i, en);
            /* P mod q_i if q_i is in digit j, else 0 (pi_j == 1 on digit j, 0 elsewhere, P == 0 mod p) */
            u64 gadget = 0;
            if (i < K && i >= j * c->alpha && i < (j + 1) * c->alpha) {
                gadget = 1;
                for (int t = 0; t < c->np; t++) gadget = mulmod(gadget, c->mod[K + t] % q, q);
            }
            const u64 *s = s_ntt + (u64)i * N, *sp = target_ntt + (u64)i * N;
            for (u64 x = 0; x < N; x++) {
                u64 v = submod(en[x], mulmod(a[x], s[x], q), q);
                v = addmod(v, mulmod(gadget, sp[x], q), q);
                b[x] = v;
            }
            free(en);
        }
        free(e);
    }
}

/* symmetric encryption at level lvl (C6): c1 = a (uniform, NTT), c0 = -a*s + m + e.
 * m: [lvl+1][N] NTT; out [2][lvl+1][N] */
void orc_encrypt(const orc_ctx *c, const uint8_t key[32], const u64 *s_ntt, const u64 *m, int lvl, u64 ct_id, u64 *out) {
    u64 N = c->N; int k = lvl + 1;
    i64 *e = (i64 *)malloc(N * sizeof(i64));
    orc_sample_cbd(key, TAG_ENC_E, ct_id << 8, N, e);
#pragma omp parallel for
    for (int i = 0; i < k; i++) {
        u64 q = c->mod[i];
        u64 *c0 = out + (u64)i * N, *c1 = out + ((u64)k + i) * N;
        orc_sample_uniform(key, TAG_ENC_A, (ct_id << 8) | (u64)i, q, N, c1);
        u64 *en = (u64 *)malloc(N * sizeof(u64));
        small_to_ntt(c, e, i, en);
        const u64 *s = s_ntt + (u64)i * N, *mi = m + (u64)i * N;
        for (u64 x = 0; x < N; x++)
            c0[x] = addmod(submod(mi[x], mulmod(c1[x], s[x], q), q), en[x], q);
        free(en);
    }
    free(e);
}
/* decrypt: c0 + c1*s mod Q_lvl (NTT domain) -> out [lvl+1][N] */
void orc_decrypt(const orc_ctx *c, const u64 *s_ntt, const u64 *ct, int lvl, u64 *out) {
    u64 N = c->N; int k = lvl + 1;
    for (int i = 0; i < k; i++) {
        u64 q = c->mod[i];
        const u64 *c0 = ct + (u64)i * N, *c1 = ct + ((u64)k + i) * N, *s = s_ntt + (u64)i * N;
        for (u64 x = 0; x < N; x++) out[(u64)i * N + x] = addmod(c0[x], mulmod(c1[x], s[x], q), q);
    }
}

/* ------------------------------------------------------------------ */
/* base conversion, ModUp, ModDown, key switch (C7, C8)                 */
/* ------------------------------------------------------------------ */
/* FastBConv_{C->m}(x) = sum_i [x_i * chat_i^{-1}]_{c_i} * chat_i mod m,
 * chat_i = prod_{l != i} c_l.  src: coefficient-form residues, src[l] over
 * modulus cm[l]; out over dm. */
static void fastbconv(const u64 *const *src, const u64 *cm, int ns, u64 dm, u64 *out, u64 N) {
    u64 inv_i[ORC_MAXP], chat_dm[ORC_MAXP];
    for (int i = 0; i < ns; i++) {
        u64 h = 1, hd = 1 % dm;
        for (int l = 0; l < ns; l++) if (l != i) { h = mulmod(h, cm[l] % cm[i], cm[i]); hd = mulmod(hd, cm[l] % dm, dm); }
        inv_i[i] = invmod(h, cm[i]);
        chat_dm[i] = hd;
    }
    for (u64 x = 0; x < N; x++) {
        u64 acc = 0;
        for (int i = 0; i < ns; i++) {
            u64 t = mulmod(src[i][x], inv_i[i], cm[i]);
            acc = addmod(acc, mulmod(t % dm, chat_dm[i], dm), dm);
        }
        out[x] = acc;
    }
}
/* public wrapper for pins: src [ns][N] coefficient residues */
void orc_fastbconv(const u64 *src, const u64 *cm, int ns, u64 dm, u64 *out, u64 N) {
    const u64 *ptrs[ORC_MAXP];
    for (int i = 0; i < ns; i++) ptrs[i] = src + (u64)i * N;
    fastbconv(ptrs, cm, ns, dm, out, N);
}

/* extended-limb index m in [0, k+np): m < k -> q_m, else p_{m-k}; prime idx: */
static inline int ext_prime(const orc_ctx *c, int k, int m) { return m < k ? m : c->K + (m - k); }

/* ModUp of every digit of d (NTT, [k][N], level lvl) -> ext [beta][k+np][N] NTT.
 * Digit j = {q_i : j*alpha <= i < min((j+1)*alpha, k)}. */
void orc_modup(const orc_ctx *c, const u64 *d, int lvl, u64 *ext) {
    int k = lvl + 1, np = c->np, E = k + np, beta = (k + c->alpha - 1) / c->alpha;
    u64 N = c->N;
    u64 *coef = (u64 *)malloc((u64)k * N * sizeof(u64));
    memcpy(coef, d, (u64)k * N * sizeof(u64));
    for (int i = 0; i < k; i++) intt_limb(c, coef + (u64)i * N, i);
    for (int j = 0; j < beta; j++) {
        int lo = j * c->alpha, hi = (j + 1) * c->alpha < k ? (j + 1) * c->alpha : k;
        const u64 *src[ORC_MAXP]; u64 cm[ORC_MAXP];
        for (int i = lo; i < hi; i++) { src[i - lo] = coef + (u64)i * N; cm[i - lo] = c->mod[i]; }
#pragma omp parallel for
        for (int m = 0; m < E; m++) {
            u64 *dst = ext + ((u64)j * E + m) * N;
            int pi = ext_prime(c, k, m);
            if (m < k && m >= lo && m < hi) { memcpy(dst, coef + (u64)m * N, N * sizeof(u64)); }
            else fastbconv(src, cm, hi - lo, c->mod[pi], dst, N);
            ntt_limb(c, dst, pi);
        }
    }
    free(coef);
}

/* ModDown (C7): y [k+np][N] NTT over Q_lvl u P -> out [k][N] NTT:
 * out_i = (y_i - NTT(FastBConv_{P->q_i}(INTT(y_P)))) * P^{-1} mod q_i  (no rounding correction) */
void orc_moddown(const orc_ctx *c, const u64 *y, int lvl, u64 *out) {
    int k = lvl + 1, np = c->np;
    u64 N = c->N;
    u64 *yp = (u64 *)malloc((u64)np * N * sizeof(u64));
    memcpy(yp, y + (u64)k * N, (u64)np * N * sizeof(u64));
    const u64 *src[ORC_MAXP]; u64 cm[ORC_MAXP];
    for (int t = 0; t < np; t++) { intt_limb(c, yp + (u64)t * N, c->K + t); src[t] = yp + (u64)t * N; cm[t] = c->mod[c->K + t]; }
#pragma omp parallel for
    for (int i = 0; i < k; i++) {
        u64 q = c->mod[i];
        u64 *conv = (u64 *)malloc(N * sizeof(u64));
        fastbconv(src, cm, np, q, conv, N);
        ntt_limb(c, conv, i);
        u64 Pinv = 1;
        for (int t = 0; t < np; t++) Pinv = mulmod(Pinv, c->mod[c->K + t] % q, q);
        Pinv = invmod(Pinv, q);
        for (u64 x = 0; x < N; x++) out[(u64)i * N + x] = mulmod(submod(y[(u64)i * N + x], conv[x], q), Pinv, q);
        free(conv);
    }
    free(yp);
}

/* inner product with a switching key after applying sigma_g (g = 1: none) to
 * the extended digits:  u_b[m] = sum_j sigma_g(ext_j[m]) * swk_j.(b|a)[m].
 * swk: [beta_top][2][K+np][N]; out u [2][k+np][N] (NTT). */
void orc_ks_inner(const orc_ctx *c, const u64 *ext, int lvl, const u64 *swk, u64 g, u64 *u) {
    int k = lvl + 1, np = c->np, E = k + np, K = c->K, Lk = K + np, beta = (k + c->alpha - 1) / c->alpha;
    u64 N = c->N;
#pragma omp parallel for
    for (int m = 0; m < E; m++) {
        int pi = ext_prime(c, k, m);
        u64 q = c->mod[pi];
        u64 *tmp = (u64 *)malloc(N * sizeof(u64));
        u64 *u0 = u + (u64)m * N, *u1 = u + ((u64)E + m) * N;
        memset(u0, 0, N * sizeof(u64)); memset(u1, 0, N * sizeof(u64));
        for (int j = 0; j < beta; j++) {
            const u64 *src = ext + ((u64)j * E + m) * N;
            if (g == 1) memcpy(tmp, src, N * sizeof(u64));
            else orc_automorphism_ntt(c, src, tmp, g, 1);
            const u64 *kb = swk + (((u64)j * 2 + 0) * Lk + pi) * N;
            const u64 *ka = swk + (((u64)j * 2 + 1) * Lk + pi) * N;
            for (u64 x = 0; x < N; x++) {
                u0[x] = addmod(u0[x], mulmod(tmp[x], kb[x], q), q);
                u1[x] = addmod(u1[x], mulmod(tmp[x], ka[x], q), q);
            }
        }
        free(tmp);
    }
}

/* hoisted rotation (C8): Rot_g(ct) = (sigma_g(c0) + c0', c1'),
 * (c0', c1') = ModDown(sum_j sigma_g(ModUp(D_j(c1))) * rk_{g,j}).  ct [2][k][N] */
void orc_rotate(const orc_ctx *c, const u64 *ct, int lvl, const u64 *rk, u64 g, u64 *out) {
    int k = lvl + 1, E = k + c->np, beta = (k + c->alpha - 1) / c->alpha;
    u64 N = c->N;
    u64 *ext = (u64 *)malloc((u64)beta * E * N * sizeof(u64));
    u64 *u = (u64 *)malloc(2ull * E * N * sizeof(u64));
    orc_modup(c, ct + (u64)k * N, lvl, ext);
    orc_ks_inner(c, ext, lvl, rk, g, u);
    u64 *c0p = (u64 *)malloc((u64)k * N * sizeof(u64));
    orc_moddown(c, u, lvl, c0p);
    orc_moddown(c, u + (u64)E * N, lvl, out + (u64)k * N);
    u64 *sc0 = (u64 *)malloc((u64)k * N * sizeof(u64));
    orc_automorphism_ntt(c, ct, sc0, g, k);
    for (int i = 0; i < k; i++) {
        u64 q = c->mod[i];
        for (u64 x = 0; x < N; x++) out[(u64)i * N + x] = addmod(sc0[(u64)i * N + x], c0p[(u64)i * N + x], q);
    }
    free(ext); free(u); free(c0p); free(sc0);
}

/* ct x ct tensor (C9): (a0b0, a0b1 + a1b0, a1b1) -> out [3][k][N] */
void orc_tensor(const orc_ctx *c, const u64 *a, const u64 *b, int lvl, u64 *out) {
    int k = lvl + 1; u64 N = c->N;
    for (int i = 0; i < k; i++) {
        u64 q = c->mod[i];
        const u64 *a0 = a + (u64)i * N, *a1 = a + ((u64)k + i) * N, *b0 = b + (u64)i * N, *b1 = b + ((u64)k + i) * N;
        u64 *d0 = out + (u64)i * N, *d1 = out + ((u64)k + i) * N, *d2 = out + (2ull * k + i) * N;
        for (u64 x = 0; x < N; x++) {
            d0[x] = mulmod(a0[x], b0[x], q);
            d1[x] = addmod(mulmod(a0[x], b1[x], q), mulmod(a1[x], b0[x], q), q);
            d2[x] = mulmod(a1[x], b1[x], q);
        }
    }
}
/* relinearize (C9): (d0 + KS(d2).0, d1 + KS(d2).1) with the s^2 key; d [3][k][N] */
void orc_relinearize(const orc_ctx *c, const u64 *d, int lvl, const u64 *rlk, u64 *out) {
    int k = lvl + 1, E = k + c->np, beta = (k + c->alpha - 1) / c->alpha;
    u64 N = c->N;
    u64 *ext = (u64 *)malloc((u64)beta * E * N * sizeof(u64));
    u64 *u = (u64 *)malloc(2ull * E * N * sizeof(u64));
    u64 *r = (u64 *)malloc(2ull * k * N * sizeof(u64));
    orc_modup(c, d + 2ull * k * N, lvl, ext);
    orc_ks_inner(c, ext, lvl, rlk, 1, u);
    orc_moddown(c, u, lvl, r);
    orc_moddown(c, u + (u64)E * N, lvl, r + (u64)k * N);
    for (int p = 0; p < 2; p++)
        for (int i = 0; i < k; i++) {
            u64 q = c->mod[i];
            for (u64 x = 0; x < N; x++)
                out[((u64)p * k + i) * N + x] = addmod(d[((u64)p * k + i) * N + x], r[((u64)p * k + i) * N + x], q);
        }
    free(ext); free(u); free(r);
}

/* ------------------------------------------------------------------ */
/* pointwise ops (C9)                                                   */
/* ------------------------------------------------------------------ */
/* ct (x) pt: out = (c0*p, c1*p); ct [2][k][N], pt [k][N] (plaintext given at >= lvl, stride ptk limbs) */
void orc_mul_pt(const orc_ctx *c, const u64 *ct, const u64 *pt, int lvl, u64 *out) {
    int k = lvl + 1; u64 N = c->N;
    for (int p = 0; p < 2; p++)
        for (int i = 0; i < k; i++) {
            u64 q = c->mod[i];
            for (u64 x = 0; x < N; x++)
                out[((u64)p * k + i) * N + x] = mulmod(ct[((u64)p * k + i) * N + x], pt[(u64)i * N + x], q);
        }
}
/* out = a + b over n_polys polys of k limbs */
void orc_add(const orc_ctx *c, const u64 *a, const u64 *b, int lvl, int n_polys, u64 *out) {
    int k = lvl + 1; u64 N = c->N;
    for (int p = 0; p < n_polys; p++)
        for (int i = 0; i < k; i++) {
            u64 q = c->mod[i];
            for (u64 x = 0; x < N; x++)
                out[((u64)p * k + i) * N + x] = addmod(a[((u64)p * k + i) * N + x], b[((u64)p * k + i) * N + x], q);
        }
}

/* ------------------------------------------------------------------ */
/* rescale (C10): y_i = (x_i - [x_lvl]_centred) * q_lvl^{-1} mod q_i    */
/* ------------------------------------------------------------------ */
void orc_rescale(const orc_ctx *c, const u64 *ct, int lvl, int n_polys, u64 *out) {
    int k = lvl + 1; u64 N = c->N, ql = c->mod[lvl];
    u64 *last = (u64 *)malloc(N * sizeof(u64));
    u64 *r = (u64 *)malloc(N * sizeof(u64));
    for (int p = 0; p < n_polys; p++) {
        memcpy(last, ct + ((u64)p * k + lvl) * N, N * sizeof(u64));
        intt_limb(c, last, lvl);
        for (int i = 0; i < lvl; i++) {
            u64 q = c->mod[i];
            for (u64 x = 0; x < N; x++) {
                u64 v = last[x];
                r[x] = (v <= (ql - 1) / 2) ? v % q : (q - ((ql - v) % q)) % q; /* centred lift mod q_i */
            }
            ntt_limb(c, r, i);
            u64 qinv = invmod(ql % q, q);
            for (u64 x = 0; x < N; x++)
                out[((u64)p * lvl + i) * N + x] = mulmod(submod(ct[((u64)p * k + i) * N + x], r[x], q), qinv, q);
        }
    }
    free(last); free(r);
}

/* ------------------------------------------------------------------ */
/* CKKS->MPC masking, server half (Alg. 1 line 1, F_C2M items 1 and 4; C14) */
/* ------------------------------------------------------------------ */
/* ct [2][k][N] NTT at level lvl -> drop to q_0, INTT both polys,
 * r uniform mod q_0 (ChaCha MASK, objid ct_id<<8), masked = (c0 + r, c1),
 * share = -r mod q_0.  masked [2][N], share [N]  (coefficient domain) */
void orc_mask(const orc_ctx *c, const u64 *ct, int lvl, const uint8_t key[32], u64 ct_id, u64 *masked, u64 *share) {
    int k = lvl + 1; u64 N = c->N, q = c->mod[0];
    memcpy(masked, ct, N * sizeof(u64));
    memcpy(masked + N, ct + (u64)k * N, N * sizeof(u64));
    intt_limb(c, masked, 0);
    intt_limb(c, masked + N, 0);
    u64 *r = (u64 *)malloc(N * sizeof(u64));
    orc_sample_uniform(key, TAG_MASK, ct_id << 8, q, N, r);
    for (u64 x = 0; x < N; x++) {
        masked[x] = addmod(masked[x], r[x], q);
        share[x] = (q - r[x]) % q;
    }
    free(r);
}

/* ------------------------------------------------------------------ */
/* Encode (C3) in __float128                                 */
/* ------------------------------------------------------------------ */
/* In-place radix-2 DIT complex FFT of length N over __float128, sign -1:
 * X_k = sum_t x_t exp(-2 pi i k t / N).  A textbook library-style step. */
static void fft_q(const orc_ctx *c, __float128 *re, __float128 *im, int sign) {
    u64 N = c->N; int lg = c->logN;
    for (u64 i = 0; i < N; i++) {
        u64 j = brv(i, lg);
        if (j > i) { __float128 t = re[i]; re[i] = re[j]; re[j] = t; t = im[i]; im[i] = im[j]; im[j] = t; }
    }
    for (u64 len = 2; len <= N; len <<= 1) {
        u64 step = N / len;
        for (u64 s = 0; s < N; s += len)
            for (u64 j = 0; j < len / 2; j++) {
                __float128 wr = c->cos2[j * step], wi = sign * c->sin2[j * step];
                u64 a = s + j, b = s + j + len / 2;
                __float128 tr = re[b] * wr - im[b] * wi, ti = re[b] * wi + im[b] * wr;
                re[b] = re[a] - tr; im[b] = im[a] - ti;
                re[a] = re[a] + tr; im[a] = im[a] + ti;
            }
    }
}

/* real slots z[N/2] -> integer coefficients round(scale * m_k), m = pi^{-1}(z):
 * m_k = (1/N) Re( zeta^{-k} * sum_t w_t omega^{-k t} ), w_t = z_j where
 * 2t+1 == +-5^j mod 2N (conjugate slots carry the same real value).
 * Rounding: nearest, ties to even (rintq).  Returns 0, or -1 if some |coef| >= 2^62. */
int orc_encode_coeffs(const orc_ctx *c, const double *z, double scale, i64 *coef) {
    u64 N = c->N, n = N / 2, twoN = 2 * N;
    __float128 *re = (__float128 *)calloc(N, sizeof(__float128));
    __float128 *im = (__float128 *)calloc(N, sizeof(__float128));
    u64 e = 1;
    for (u64 j = 0; j < n; j++) {
        re[(e - 1) / 2] = (__float128)z[j];
        re[(twoN - e - 1) / 2] = (__float128)z[j];
        e = (e * 5) % twoN;
    }
    fft_q(c, re, im, -1);
    int st = 0;
    for (u64 k = 0; k < N; k++) {
        /* zeta^{-k} = cos(pi k/N) - i sin(pi k/N) */
        __float128 v = (c->cosh_[k] * re[k] + c->sinh_[k] * im[k]) / (__float128)N;
        __float128 r = rintq(v * (__float128)scale);
        if (fabsq(r) >= 4611686018427387904.0Q) { st = -1; r = 0; }
        coef[k] = (i64)r;
    }
    free(re); free(im);
    return st;
}
/* direct O(N*n) evaluation of the same definition, for pins at small N:
 * m_k = (2/N) sum_j z_j cos(pi * (k*5^j mod 2N) / N) */
void orc_encode_direct(const orc_ctx *c, const double *z, double scale, __float128 *exact_out, i64 *coef) {
    u64 N = c->N, n = N / 2, twoN = 2 * N;
    u64 *e5 = (u64 *)malloc(n * sizeof(u64));
    u64 e = 1;
    for (u64 j = 0; j < n; j++) { e5[j] = e; e = (e * 5) % twoN; }
#pragma omp parallel for
    for (u64 k = 0; k < N; k++) {
        __float128 acc = 0;
        for (u64 j = 0; j < n; j++) {
            u64 a = (u64)(((u128)k * e5[j]) % twoN);  /* cos(pi a / N) */
            __float128 cv = a < N ? c->cosh_[a] : -c->cosh_[a - N];
            acc += (__float128)z[j] * cv;
        }
        __float128 v = acc * 2 / (__float128)N * (__float128)scale;
        if (exact_out) exact_out[k] = v;
        coef[k] = (i64)rintq(v);
    }
    free(e5);
}
/* quad -> decimal string helper for tests */
void orc_quad_to_str(const __float128 *v, char *buf, int len) { quadmath_snprintf(buf, len, "%.36Qg", *v); }

/* encode at level lvl: coefficients mod q_0..q_lvl, NTT -> out [lvl+1][N] */
int orc_encode(const orc_ctx *c, const double *z, double scale, int lvl, u64 *out) {
    u64 N = c->N;
    i64 *coef = (i64 *)malloc(N * sizeof(i64));
    int st = orc_encode_coeffs(c, z, scale, coef);
#pragma omp parallel for
    for (int i = 0; i <= lvl; i++) small_to_ntt(c, coef, i, out + (u64)i * N);
    free(coef);
    return st;
}

/* ------------------------------------------------------------------ */
/* extended-basis (Q_l u P) helpers for double-hoisted rotations        */
/* ------------------------------------------------------------------ */
/* Rotation kept in the extended basis (no ModDown): out [2][k+np][N] =
 * (P*sigma_g(c0) + u0, u1) with u = sum_j sigma_g(ModUp(D_j(c1))) * rk_{g,j} (C8);
 * P*sigma_g(c0) is 0 on the P limbs.  g = 1: the lifted input (P*c0, P*c1). */
void orc_rotate_ext(const orc_ctx *c, const u64 *ct, int lvl, const u64 *rk, u64 g, u64 *out) {
    int k = lvl + 1, E = k + c->np, beta = (k + c->alpha - 1) / c->alpha;
    u64 N = c->N;
    if (g == 1) {  /* lift: (P c0, P c1) */
        for (int p = 0; p < 2; p++)
            for (int m = 0; m < E; m++) {
                u64 *o = out + ((u64)p * E + m) * N;
                if (m >= k) { memset(o, 0, N * sizeof(u64)); continue; }
                u64 q = c->mod[m], Pm = 1;
                for (int t = 0; t < c->np; t++) Pm = mulmod(Pm, c->mod[c->K + t] % q, q);
                for (u64 x = 0; x < N; x++) o[x] = mulmod(ct[((u64)p * k + m) * N + x], Pm, q);
            }
        return;
    }
    u64 *ext = (u64 *)malloc((u64)beta * E * N * sizeof(u64));
    orc_modup(c, ct + (u64)k * N, lvl, ext);
    orc_ks_inner(c, ext, lvl, rk, g, out);
    u64 *sc0 = (u64 *)malloc((u64)k * N * sizeof(u64));
    orc_automorphism_ntt(c, ct, sc0, g, k);
    for (int m = 0; m < k; m++) {
        u64 q = c->mod[m], Pm = 1;
        for (int t = 0; t < c->np; t++) Pm = mulmod(Pm, c->mod[c->K + t] % q, q);
        for (u64 x = 0; x < N; x++) out[(u64)m * N + x] = addmod(out[(u64)m * N + x], mulmod(sc0[(u64)m * N + x], Pm, q), q);
    }
    free(ext); free(sc0);
}

/* pointwise ops over an explicit prime list: a, out [n_polys][n_limbs][N]; pt [n_limbs][N] */
void orc_mul_pt_idx(const orc_ctx *c, const u64 *a, const u64 *pt, const int *pidx, int n_limbs, int n_polys, u64 *out) {
    u64 N = c->N;
    for (int p = 0; p < n_polys; p++)
        for (int l = 0; l < n_limbs; l++) {
            u64 q = c->mod[pidx[l]];
            for (u64 x = 0; x < N; x++)
                out[((u64)p * n_limbs + l) * N + x] = mulmod(a[((u64)p * n_limbs + l) * N + x], pt[(u64)l * N + x], q);
        }
}
void orc_add_idx(const orc_ctx *c, const u64 *a, const u64 *b, const int *pidx, int n_limbs, int n_polys, u64 *out) {
    u64 N = c->N;
    for (int p = 0; p < n_polys; p++)
        for (int l = 0; l < n_limbs; l++) {
            u64 q = c->mod[pidx[l]];
            for (u64 x = 0; x < N; x++)
                out[((u64)p * n_limbs + l) * N + x] = addmod(a[((u64)p * n_limbs + l) * N + x], b[((u64)p * n_limbs + l) * N + x], q);
        }
}
/* encode at level lvl over the extended basis Q_lvl u P: out [lvl+1+np][N] */
int orc_encode_ext(const orc_ctx *c, const double *z, double scale, int lvl, u64 *out) {
    u64 N = c->N;
    int k = lvl + 1, E = k + c->np;
    i64 *coef = (i64 *)malloc(N * sizeof(i64));
    int st = orc_encode_coeffs(c, z, scale, coef);
    for (int m = 0; m < E; m++) small_to_ntt(c, coef, m < k ? m : c->K + (m - k), out + (u64)m * N);
    free(coef);
    return st;
}

/* ------------------------------------------------------------------ */
/* ModDown fused with rescale (reading C17): one exact rounding         */
/* ------------------------------------------------------------------ */
/* in [2][k+np][N] NTT over Q_lvl u P (k = lvl+1) -> out [2][lvl][N] NTT over Q_{lvl-1}:
 *   y = round(X / M),  M = q_lvl * p_0 ... p_{np-1} (odd, so no ties),
 * computed as y = (X + h - r) / M with h = (M-1)/2 and r = (X + h) mod M, where r is
 * rebuilt exactly from the residues of X + h at the M-moduli (Garner's mixed radix:
 * r = d_0 + m_0 (d_1 + m_1 (d_2 + ...)), d_t < m_t).  The quotient is the same integer
 * mod Q_{lvl-1} whichever representative of X mod Q_lvl P is taken (it shifts by
 * multiples of Q_lvl P / M = Q_{lvl-1}). */
void orc_moddown_rescale(const orc_ctx *c, const u64 *in, int lvl, u64 *out) {
    int k = lvl + 1, np = c->np, E = k + np, nd = 1 + np;
    u64 N = c->N;
    u64 m[ORC_MAXP]; int mi[ORC_MAXP];
    m[0] = c->mod[lvl]; mi[0] = lvl;
    for (int t = 0; t < np; t++) { m[1 + t] = c->mod[c->K + t]; mi[1 + t] = c->K + t; }
    u64 *drop = (u64 *)malloc((u64)nd * N * sizeof(u64));
    u64 *w = (u64 *)malloc((u64)lvl * N * sizeof(u64));
    for (int p = 0; p < 2; p++) {
        const u64 *x = in + (u64)p * E * N;
        for (int t = 0; t < nd; t++) {
            memcpy(drop + (u64)t * N, x + (u64)(lvl + t) * N, N * sizeof(u64));  /* limbs lvl, k.. are q_lvl, P */
            intt_limb(c, drop + (u64)t * N, mi[t]);
        }
        /* per-(s, t) inverses m_s^{-1} mod m_t and per-limb (M - 1)/2 mod q_i: constants of the loop */
        u64 minv[ORC_MAXP][ORC_MAXP], hq[ORC_MAXP];
        for (int t = 0; t < nd; t++)
            for (int s = 0; s < t; s++) minv[t][s] = invmod(m[s] % m[t], m[t]);
        for (int i = 0; i < lvl; i++) {
            u64 q = c->mod[i], Mq = 1;
            for (int t = 0; t < nd; t++) Mq = mulmod(Mq, m[t] % q, q);
            hq[i] = mulmod(submod(Mq, 1, q), invmod(2, q), q);   /* (M - 1) / 2 mod q_i */
        }
#pragma omp parallel for
        for (u64 j = 0; j < N; j++) {
            u64 d[ORC_MAXP];
            for (int t = 0; t < nd; t++) {
                u64 v = addmod(drop[(u64)t * N + j], (m[t] - 1) / 2, m[t]);  /* h = -1/2 mod m_t */
                for (int s = 0; s < t; s++) v = mulmod(submod(v, d[s] % m[t], m[t]), minv[t][s], m[t]);
                d[t] = v;
            }
            for (int i = 0; i < lvl; i++) {
                u64 q = c->mod[i], r = 0;
                for (int t = nd - 1; t >= 0; t--) r = addmod(mulmod(r, m[t] % q, q), d[t] % q, q);
                w[(u64)i * N + j] = submod(hq[i], r, q);
            }
        }
        for (int i = 0; i < lvl; i++) {
            u64 q = c->mod[i], Mq = 1;
            for (int t = 0; t < nd; t++) Mq = mulmod(Mq, m[t] % q, q);
            u64 Minv = invmod(Mq, q);
            ntt_limb(c, w + (u64)i * N, i);
            for (u64 j = 0; j < N; j++)
                out[((u64)p * lvl + i) * N + j] = mulmod(addmod(x[(u64)i * N + j], w[(u64)i * N + j], q), Minv, q);
        }
    }
    free(drop); free(w);
}

/* Relinearisation kept in Q_l u P (reading C17): d = (d0, d1, d2) [3][k][N] ->
 * out [2][k+np][N] = (P d0 + u0, P d1 + u1), u = sum_j ModUp(D_j(d2)) * rlk_j (C7, C9);
 * a following ModDown + rescale is then one exact rounding (orc_moddown_rescale). */
void orc_relinearize_ext(const orc_ctx *c, const u64 *d, int lvl, const u64 *rlk, u64 *out) {
    int k = lvl + 1, E = k + c->np, beta = (k + c->alpha - 1) / c->alpha;
    u64 N = c->N;
    u64 *ext = (u64 *)malloc((u64)beta * E * N * sizeof(u64));
    orc_modup(c, d + 2ull * k * N, lvl, ext);
    orc_ks_inner(c, ext, lvl, rlk, 1, out);
    for (int p = 0; p < 2; p++)
        for (int i = 0; i < k; i++) {
            u64 q = c->mod[i], Pm = 1;
            for (int t = 0; t < c->np; t++) Pm = mulmod(Pm, c->mod[c->K + t] % q, q);
            for (u64 x = 0; x < N; x++) {
                u64 *o = out + ((u64)p * E + i) * N + x;
                *o = addmod(*o, mulmod(d[((u64)p * k + i) * N + x], Pm, q), q);
            }
        }
    free(ext);
}

/* ------------------------------------------------------------------ */
/* f3: MPC -> CKKS ingest (Alg. 2 line 4; ring-to-field eq. P:1222-1232) */
/* ------------------------------------------------------------------ */
/* A share x in Z_{2^w} (w <= 64, x < 2^w) mapped to the field: x mod q_i (P0's share) or
 * x - 2^w mod q_i (P1's share, sub = 1), per limb i <= lvl, then NTT (C2): out [lvl+1][N]. */
void orc_share_to_rns(const orc_ctx *c, const u64 *x, int w, int sub, int lvl, u64 *out) {
    u64 N = c->N;
    for (int i = 0; i <= lvl; i++) {
        u64 q = c->mod[i];
        u64 two_w = (u64)(((u128)1 << w) % q);
        u64 *o = out + (u64)i * N;
        for (u64 j = 0; j < N; j++) {
            u64 v = x[j] % q;
            o[j] = sub ? submod(v, two_w, q) : v;
        }
        ntt_limb(c, o, i);
    }
}

/* The same for a share in Z_{2^w} with w <= 128 (x: [N][2] u64 little-endian words, x < 2^w): the
 * paper's ring-to-field runs on Z_{2^{l+40}}, l = 43, wider than one word. */
void orc_share_to_rns128(const orc_ctx *c, const u64 *x, int w, int sub, int lvl, u64 *out) {
    u64 N = c->N;
    for (int i = 0; i <= lvl; i++) {
        u64 q = c->mod[i];
        u64 r64 = (u64)(((u128)1 << 64) % q);
        u64 two_w = w < 128 ? (u64)(((u128)1 << w) % q) : mulmod(r64, r64, q);
        u64 *o = out + (u64)i * N;
        for (u64 j = 0; j < N; j++) {
            u64 v = (u64)((((u128)x[2 * j + 1] << 64) | x[2 * j]) % q);
            o[j] = sub ? submod(v, two_w, q) : v;
        }
        ntt_limb(c, o, i);
    }
}

/* ------------------------------------------------------------------ */
/* f3: local fixed-point Decode of a share over Z_{2^128}               */
/* ("O(N log N) FFT ... extend the shares to a larger ring and  */
/* conduct local truncations"; App. C.4 P:1246-1262 extend-then-truncate) */
/* ------------------------------------------------------------------ */
typedef __int128 i128;
/* arithmetic right shift of a ring element read as a signed 128-bit integer (SecureML-style local
 * truncation, App. C.4: [m']_b = [m]_b >>_a s) */
static inline u128 ashr128(u128 v, int s) { return (u128)(((i128)v) >> s); }
/* x: [N][2] u64 = little-endian u128 share of the coefficient vector; y: [N/2][2] share of the
 * real slots.  Cooley-Tukey network over Z_{2^128}[i] (stage m = 1, 2, .., N/2, block i, twiddle
 * W = round(2^ft zeta^{brv(m+i)}), zeta = e^{i pi / N}): V = (Y * W) >>_a ft (each component),
 * X' = X + V, Y' = X - V, so position k ends with sum_j x_j zeta^{(2 brv(k)+1) j} (C2 / C3
 * ordering); slot j (zeta^{5^j}) sits at k with 2 brv(k) + 1 = 5^j mod 2N; y_j = Re >>_a s_out. */
void orc_share_decode(const orc_ctx *c, const u64 *x, int ft, int s_out, u64 *y) {
    u64 N = c->N, twoN = 2 * N;
    int logN = c->logN;
    u128 *re = (u128 *)malloc(N * sizeof(u128)), *im = (u128 *)malloc(N * sizeof(u128));
    for (u64 k = 0; k < N; k++) { re[k] = (u128)x[2 * k] | ((u128)x[2 * k + 1] << 64); im[k] = 0; }
    __float128 sc = ldexpq(1.0Q, ft);
    for (u64 m = 1; m < N; m <<= 1) {
        u64 t = N / (2 * m);
        for (u64 i = 0; i < m; i++) {
            __float128 ang = M_PIq * (__float128)brv(m + i, logN) / (__float128)N;
            long long wr = (long long)roundq(sc * cosq(ang)), wi = (long long)roundq(sc * sinq(ang));
            u128 Wr = (u128)(i128)wr, Wi = (u128)(i128)wi;
            for (u64 j = 2 * i * t; j < 2 * i * t + t; j++) {
                u128 yr = re[j + t], yi = im[j + t];
                u128 vr = ashr128(yr * Wr - yi * Wi, ft), vi = ashr128(yr * Wi + yi * Wr, ft);
                u128 xr = re[j], xi = im[j];
                re[j] = xr + vr; im[j] = xi + vi;
                re[j + t] = xr - vr; im[j + t] = xi - vi;
            }
        }
    }
    u64 e = 1;  /* 5^j mod 2N */
    for (u64 j = 0; j < N / 2; j++) {
        u64 k = brv((e - 1) / 2, logN);
        u128 v = ashr128(re[k], s_out);
        y[2 * j] = (u64)v; y[2 * j + 1] = (u64)(v >> 64);
        e = (e * 5) % twoN;
    }
    free(re); free(im);
}

/* ------------------------------------------------------------------ */
/* f3: local fixed-point Encode of a share over Z_{2^128}               */
/* (Alg. 2 line 1: "P_b locally evaluates the CKKS encoding";      */
/* P:684-685 O(N log N) FFT with local truncations on the extended ring;  */
/* App. C.4 P:1246-1262 SecureML truncation >>_a; reading C20)            */
/* ------------------------------------------------------------------ */
/* y: [N/2][2] u64 = little-endian u128 share of the real slot vector (fixed point).  The CKKS
 * encode pi^{-1} (C3): the slot value is placed at the evaluation points zeta^{5^j} and its
 * conjugate zeta^{-5^j} (real slots, footnote P:540), then the inverse transform
 * m_k = (1/N) sum_e a_e zeta^{-e k} as the Gentleman-Sande network over Z_{2^128}[i]
 * (stage m = N/2, .., 2, 1, block i, twiddle conj(W), W = round(2^ft zeta^{brv(m+i)})):
 * X' = X + Y, Y' = ((X - Y) * conj(W)) >>_a ft (each component); then coefficient
 * x_k = Re_k >>_a s_out (s_out folds the 1/N = 2^-logN and the scale change of the fixed point).
 * x: [N][2] u64 share of the integer coefficient vector. */
void orc_share_encode(const orc_ctx *c, const u64 *y, int ft, int s_out, u64 *x) {
    u64 N = c->N, twoN = 2 * N;
    int logN = c->logN;
    u128 *re = (u128 *)calloc(N, sizeof(u128)), *im = (u128 *)calloc(N, sizeof(u128));
    u64 e = 1;  /* 5^j mod 2N */
    for (u64 j = 0; j < N / 2; j++) {
        u64 k = brv((e - 1) / 2, logN);               /* position of zeta^{5^j}: 2 brv(k) + 1 = 5^j */
        u64 kc = brv((twoN - e - 1) / 2, logN);       /* position of zeta^{-5^j} = conj */
        u128 v = (u128)y[2 * j] | ((u128)y[2 * j + 1] << 64);
        re[k] = v; re[kc] = v;
        e = (e * 5) % twoN;
    }
    __float128 sc = ldexpq(1.0Q, ft);
    for (u64 m = N / 2; m >= 1; m >>= 1) {
        u64 t = N / (2 * m);
        for (u64 i = 0; i < m; i++) {
            __float128 ang = M_PIq * (__float128)brv(m + i, logN) / (__float128)N;
            long long wr = (long long)roundq(sc * cosq(ang)), wi = (long long)roundq(sc * sinq(ang));
            u128 Wr = (u128)(i128)wr, Wi = (u128)(i128)(-wi);   /* conj(W) */
            for (u64 j = 2 * i * t; j < 2 * i * t + t; j++) {
                u128 xr = re[j], xi = im[j], yr = re[j + t], yi = im[j + t];
                u128 dr = xr - yr, di = xi - yi;
                re[j] = xr + yr; im[j] = xi + yi;
                re[j + t] = ashr128(dr * Wr - di * Wi, ft);
                im[j + t] = ashr128(dr * Wi + di * Wr, ft);
            }
        }
        if (m == 1) break;
    }
    for (u64 k = 0; k < N; k++) {
        u128 v = ashr128(re[k], s_out);
        x[2 * k] = (u64)v; x[2 * k + 1] = (u64)(v >> 64);
    }
    free(re); free(im);
}
