#include <algorithm>
// kernels.cu -- RNS pointwise kernels of the B200 BLB library:
//   ChaCha20 samplers (C4), key generation (C5), encrypt / decrypt (C6),
//   FastBConv ModUp / ModDown and the key-switch inner product with the
//   NTT-domain automorphism folded into its loads (C7, C8; rows a2 / a4),
//   rescale (C10; row a5) and the CKKS->MPC mask (C14; row a8).
// All kernels are coefficient-parallel: thread x handles residue x of a row,
// so every global access is coalesced along the limb-major layout.
#include "blb_internal.cuh"

namespace {
constexpr int kTB = 256;

// ---------------------------------------------------------------- ChaCha20
__device__ __forceinline__ uint32_t rotl32(uint32_t x, int r) { return __funnelshift_l(x, x, r); }
#define QR(a, b, c, d)                                                      \
    a += b; d ^= a; d = rotl32(d, 16); c += d; b ^= c; b = rotl32(b, 12); \
    a += b; d ^= a; d = rotl32(d, 8);  c += d; b ^= c; b = rotl32(b, 7);

__device__ __forceinline__ void chacha_block(const ChachaKey &key, uint32_t counter, uint32_t n0, uint32_t n1,
                                             uint32_t n2, uint32_t o[16]) {
    uint32_t s[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u, key.k[0], key.k[1], key.k[2], key.k[3],
                      key.k[4],    key.k[5],    key.k[6],    key.k[7],    counter,  n0,       n1,       n2};
#pragma unroll
    for (int i = 0; i < 16; i++) o[i] = s[i];
#pragma unroll
    for (int r = 0; r < 10; r++) {
        QR(o[0], o[4], o[8], o[12]); QR(o[1], o[5], o[9], o[13]);
        QR(o[2], o[6], o[10], o[14]); QR(o[3], o[7], o[11], o[15]);
        QR(o[0], o[5], o[10], o[15]); QR(o[1], o[6], o[11], o[12]);
        QR(o[2], o[7], o[8], o[13]); QR(o[3], o[4], o[9], o[14]);
    }
#pragma unroll
    for (int i = 0; i < 16; i++) o[i] += s[i];
}
// C4 layout: nonce = LE32(tag) || LE64(objid); block b = coefficients 4b..4b+3,
// draw d = (w_{2d}, w_{2d+1}) with w_i the little-endian u64 words.
__device__ __forceinline__ void draw_block(const ChachaKey &key, uint32_t tag, u64 objid, uint32_t blk, u64 lo[4],
                                           u64 hi[4]) {
    uint32_t o[16];
    chacha_block(key, blk, tag, (uint32_t)objid, (uint32_t)(objid >> 32), o);
#pragma unroll
    for (int d = 0; d < 4; d++) {
        lo[d] = (u64)o[4 * d] | ((u64)o[4 * d + 1] << 32);
        hi[d] = (u64)o[4 * d + 2] | ((u64)o[4 * d + 3] << 32);
    }
}

struct LimbList {
    int n;
    int prime[BLB_MAXP];   // modulus index per row
    int nonce[BLB_MAXP];   // limb index entering the ChaCha object id
};

// uniform mod q rows (NTT-domain "a" polynomials): out[r][x], objid = (id << 8) | nonce[r]
__global__ void k_sample_uniform(u64 *out, long long row_stride, LimbList ll, Primes pr, ChachaKey key, uint32_t tag,
                                 u64 id, int N) {
    const int blk = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y;
    if (blk >= N / 4) return;
    u64 lo[4], hi[4];
    draw_block(key, tag, (id << 8) | (u64)ll.nonce[r], blk, lo, hi);
    const ModConst &mc = pr.m[ll.prime[r]];
    u64 *o = out + r * row_stride;
#pragma unroll
    for (int d = 0; d < 4; d++) o[4 * blk + d] = reduce128(hi[d], lo[d], mc);
}

// small coefficient polynomial (ternary secret: mode 0; CBD eta=21: mode 1)
// from draws with objid = id << 8, written as residues into every listed row
__global__ void k_sample_small(u64 *out, long long row_stride, LimbList ll, Primes pr, ChachaKey key, uint32_t tag,
                               u64 id, int mode, int N) {
    const int blk = blockIdx.x * blockDim.x + threadIdx.x;
    if (blk >= N / 4) return;
    u64 lo[4], hi[4];
    draw_block(key, tag, id << 8, blk, lo, hi);
    long long v[4];
#pragma unroll
    for (int d = 0; d < 4; d++) {
        if (mode == 0) v[d] = (long long)(lo[d] % 3ull) - 1;
        else {
            const u64 m = (1ull << 21) - 1;
            v[d] = (long long)__popcll(lo[d] & m) - (long long)__popcll((lo[d] >> 21) & m);
        }
    }
    for (int r = 0; r < ll.n; r++) {
        const u64 q = pr.m[ll.prime[r]].q;
        u64 *o = out + r * row_stride;
#pragma unroll
        for (int d = 0; d < 4; d++) o[4 * blk + d] = v[d] >= 0 ? (u64)v[d] : q - (u64)(-v[d]);
    }
}

// switching key rows: b = e - a*s + gadget*s'   (s' = sigma_g(s) or s^2)
__global__ void k_keygen_combine(u64 *b, const u64 *a, const u64 *s, long long stride, LimbList ll, Primes pr,
                                 uint32_t galois, int relin, const u64 *gadget, int logN) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y;
    const int N = 1 << logN;
    if (x >= N) return;
    const int pi = ll.prime[r];
    const ModConst &mc = pr.m[pi];
    const u64 *sr = s + (long long)pi * N;
    const u64 sx = sr[x];
    const u64 as = mulmod(a[r * stride + x], sx, mc);
    u64 v = submod(b[r * stride + x], as, mc.q);
    const u64 g = gadget[pi];
    if (g) {
        u64 sp = relin ? mulmod(sx, sx, mc) : sr[galois_perm(x, galois, logN)];
        v = addmod(v, mulmod(g, sp, mc), mc.q);
    }
    b[r * stride + x] = v;
}

// c0 = e - a*s + pt  (c0 holds NTT(e) on entry)
__global__ void k_encrypt_combine(u64 *c0, const u64 *c1, const u64 *s, const u64 *pt, Primes pr, int N) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y;
    if (x >= N) return;
    const ModConst &mc = pr.m[i];
    const long long o = (long long)i * N + x;
    u64 v = submod(c0[o], mulmod(c1[o], s[o], mc), mc.q);
    c0[o] = addmod(v, pt[o], mc.q);
}

__global__ void k_decrypt(const u64 *c0, const u64 *c1, const u64 *s, u64 *out, Primes pr, int N) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y;
    if (x >= N) return;
    const ModConst &mc = pr.m[i];
    const long long o = (long long)i * N + x;
    out[o] = addmod(c0[o], mulmod(c1[o], s[o], mc), mc.q);
}

__global__ void k_mul_pt(const u64 *in, const u64 *pt, u64 *out, Primes pr, int k, int N) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y, p = blockIdx.z;
    if (x >= N) return;
    const ModConst &mc = pr.m[i];
    const long long o = ((long long)p * k + i) * N + x;
    out[o] = mulmod(in[o], pt[(long long)i * N + x], mc);
}

__global__ void k_add(const u64 *a, const u64 *b, u64 *out, Primes pr, int k, int N) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y, p = blockIdx.z;
    if (x >= N) return;
    const long long o = ((long long)p * k + i) * N + x;
    out[o] = addmod(a[o], b[o], pr.m[i].q);
}
__global__ void k_sub(const u64 *a, const u64 *b, u64 *out, Primes pr, int k, int N) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y, p = blockIdx.z;
    if (x >= N) return;
    const long long o = ((long long)p * k + i) * N + x;
    out[o] = submod(a[o], b[o], pr.m[i].q);
}

// ------------------------------------------------------------ ModUp (C7)
struct PtrList {
    const u64 *p[kMaxJobs];
};

// S13 flooding noise (reading C22): e0[x] = (lo64(draw x) mod 2^(f+1)) - 2^f as a residue mod q_0,
// rows t of n_ct conversions (object id (id0 + t) << 8), coefficient domain
__global__ void k_sample_flood(u64 *out, Primes pr, ChachaKey key, u64 id0, int flood_bits, int N) {
    const int blk = blockIdx.x * blockDim.x + threadIdx.x;
    const int t = blockIdx.y;
    if (blk >= N / 4) return;
    u64 lo[4], hi[4];
    draw_block(key, TAG_RR_E0, (id0 + (u64)t) << 8, blk, lo, hi);
    const u64 q = pr.m[0].q, m = (2ull << flood_bits) - 1, h = 1ull << flood_bits;
#pragma unroll
    for (int d = 0; d < 4; d++) {
        const u64 u = lo[d] & m;
        out[(long long)t * N + 4 * blk + d] = u >= h ? u - h : q - (h - u);
    }
}
// c0 += v b0 + e0, c1 += v a0 + e1 (mod q_0, NTT): rows [t][3][N] = (v, e0, e1); pk [2][kpk][N]
__global__ void k_rr_combine(PtrList cts, const u64 *vee, const u64 *pk, long long kpkN, Primes pr, int N) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int t = blockIdx.y;
    if (x >= N) return;
    const ModConst &mc = pr.m[0];
    u64 *c = const_cast<u64 *>(cts.p[t]);
    const u64 v = vee[((long long)t * 3 + 0) * N + x], e0 = vee[((long long)t * 3 + 1) * N + x],
              e1 = vee[((long long)t * 3 + 2) * N + x];
    c[x] = addmod(addmod(c[x], mulmod(v, pk[x], mc), mc.q), e0, mc.q);
    c[N + x] = addmod(addmod(c[N + x], mulmod(v, pk[kpkN + x], mc), mc.q), e1, mc.q);
}


// coef[t][i][x] = c1[t][i][x] for i < k (copy before the INTT)
__global__ void k_gather_rows(PtrList src, u64 *dst, int k, int N) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y, t = blockIdx.z;
    if (x >= N) return;
    dst[((long long)t * k + i) * N + x] = src.p[t][(long long)i * N + x];
}

// ext[t][j][m][x]: digit j's own limbs copy the NTT-domain input; the others are
// FastBConv_{D_j -> m}(coef) = sum_i [coef_i * dhat_i^{-1}]_{d_i} * dhat_i  mod m.
// Table at tab + bconv_modup_off(level, j): inv[nd], inv_sh[nd], chat[nd][E].
struct Offs {
    long long o[BLB_MAXP];
};
__global__ void k_bconv_modup(PtrList c1_ntt, const u64 *coef, u64 *ext, const u64 *tab, Offs tab_off, Primes pr,
                              int k, int np, int K, int alpha, int beta, int N) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int m = blockIdx.y;               // ext limb
    const int t = blockIdx.z / beta, j = blockIdx.z % beta;
    if (x >= N) return;
    const int E = k + np;
    const int lo = j * alpha, hi = min((j + 1) * alpha, k), nd = hi - lo;
    u64 *o = ext + (((long long)t * beta + j) * E + m) * N + x;
    if (m >= lo && m < hi) {
        *o = c1_ntt.p[t][(long long)m * N + x];
        return;
    }
    const int pm = m < k ? m : K + (m - k);
    const ModConst &mc = pr.m[pm];
    if (nd == 1) {  // alpha = 1: dhat = 1, dhat^{-1} = 1 -> FastBConv(x) = x mod m
        *o = mod64(coef[((long long)t * k + lo) * N + x], mc);
        return;
    }
    const u64 *tb = tab + tab_off.o[j];
    Acc128 acc;
    acc.zero();
    for (int d = 0; d < nd; d++) {
        const int pi = lo + d;
        const u64 v = coef[((long long)t * k + pi) * N + x];
        const u64 y = shoup(v, tb[d], tb[nd + d], pr.m[pi].q);
        acc.mac(y, tb[2 * nd + d * E + m]);
    }
    *o = acc.reduce(mc);
}

// ------------------------------------------------------- key switch (C7, C8)

// u[t][b][m][x] = sum_j sigma_g(ext_j)[m][x] * key_j[b][pm][x]
// Jobs sharing one switching key (same Galois element) form a group of <= 4:
// every key word is loaded once per group and re-used from registers (the key
// stream is the dominant HBM traffic of a key switch).
#ifndef BLB_KS_GROUP
#define BLB_KS_GROUP 4
#endif
constexpr int kKsGroup = BLB_KS_GROUP;  // jobs sharing one key per CTA (compile-time A/B)
struct KsGroups {
    int n;
    int start[kMaxJobs + 1];
};
// BETA > 0: digit count known at compile time (all loads of a thread are issued
// before the first multiply); BETA = 0: runtime beta.
// EXT: write the extended-basis result (P sigma_g(c0) + u0, u1) over Q_l u P straight to
// jobs.j[t].out ([2][E][N]) -- the double-hoisted rotation (no ModDown).
// SMALL (prime < 2^41): both products of a digit run on the FP64 pipe (AccG, no per-product
// reduction); 60-bit rows take ks_inner_body60 (Acc60, one job at a time) when beta is a compile-time
// constant <= 7, else Acc128 here.
// Digit source: DigG loads job t's extended digit j straight from global memory.
struct DigG {
    const KsJobs *jobs;
    long long off;  // m * N + x
    long long EN;   // E * N
    __device__ __forceinline__ u64 operator()(int t, int, int j) const { return jobs->j[t].ext[j * EN + off]; }
};

template <int BETA, bool EXT, bool SMALL, class DS>
__device__ __forceinline__ void ks_inner_body(const KsJobs &jobs, const KsGroups &grp, u64 *u, const Primes &pr, int k,
                                              int np, int K, int beta_rt, int logN, const PinvTab &pq, int x, int m,
                                              int gi, const DS &ds) {
    const int N = 1 << logN;
    const int beta = BETA > 0 ? BETA : beta_rt;
    const int t0 = grp.start[gi], cnt = grp.start[gi + 1] - t0;
    const int E = k + np, Lk = K + np;
    const int pm = m < k ? m : K + (m - k);
    const KsJob &J0 = jobs.j[t0];
    // rotation keys are stored pre-permuted (k'[y] = k[perm_{g^-1}(y)], blb_keys): every load is
    // contiguous and only the two outputs are scattered, to x = perm_{g^-1}(y)
    const uint32_t dst = J0.galois == 1 ? (uint32_t)x : galois_perm(x, J0.galois_inv, logN);
    const ModConst &mc = pr.m[pm];
    using A1 = typename std::conditional<SMALL, AccG, Acc128>::type;
    using A0 = A1;
    const double qd = (double)mc.q, qinv = 1.0 / qd;
    A0 a0[kKsGroup];
    A1 a1[kKsGroup];
#pragma unroll
    for (int q = 0; q < kKsGroup; q++) { a0[q].zero(); a1[q].zero(); }
    if (BETA > 0) {
        u64 kb[BETA > 0 ? BETA : 1], ka[BETA > 0 ? BETA : 1];
#pragma unroll
        for (int j = 0; j < BETA; j++) {
            kb[j] = J0.key[(((long long)j * 2 + 0) * Lk + pm) * N + x];
            ka[j] = J0.key[(((long long)j * 2 + 1) * Lk + pm) * N + x];
        }
#pragma unroll
        for (int q = 0; q < kKsGroup; q++) {
            if (q < cnt) {
                u64 e[BETA > 0 ? BETA : 1];
#pragma unroll
                for (int j = 0; j < BETA; j++) e[j] = ds(t0 + q, q, j);
#pragma unroll
                for (int j = 0; j < BETA; j++) {
                    accm(a0[q], e[j], kb[j], qd, qinv);
                    accm(a1[q], e[j], ka[j], qd, qinv);
                }
            }
        }
    } else {
        for (int j = 0; j < beta; j++) {
            const u64 kb = J0.key[(((long long)j * 2 + 0) * Lk + pm) * N + x];
            const u64 ka = J0.key[(((long long)j * 2 + 1) * Lk + pm) * N + x];
#pragma unroll
            for (int q = 0; q < kKsGroup; q++) {
                if (q < cnt) {
                    const u64 e = ds(t0 + q, q, j);
                    accm(a0[q], e, kb, qd, qinv);
                    accm(a1[q], e, ka, qd, qinv);
                }
            }
        }
    }
    auto a1r = [&](int q) -> u64 { return accr(a1[q], mc, qd, qinv); };
    // The additive terms: EXT adds P c0 (and P c1_add) over the Q limbs of the extended result.  The
    // ModDown path folds the rotation's sigma_g(c0) (add_mode 1) or the relinearisation's (c0, c1)
    // (add_mode 2) in the same way: ModDown(u + P c) = ModDown(u) + c exactly (P P^{-1} = 1 mod q_i;
    // the P limbs, P c = 0 mod p, are unchanged), and at output position dst = perm_{g^-1}(x)
    // sigma_g(c0) is c0[x] -- a contiguous read instead of a gather in the ModDown epilogue.
    // All loads of the group are issued before its first store (the stores may alias as far as the
    // compiler knows): one exposed latency instead of one per job.
    u64 c0v[kKsGroup], c1v[kKsGroup];
#pragma unroll
    for (int q = 0; q < kKsGroup; q++) {
        c0v[q] = 0; c1v[q] = 0;
        if (q < cnt && m < k) {
            const KsJob &J = jobs.j[t0 + q];
            if (EXT || J.add_mode != 0) c0v[q] = J.c0[(long long)m * N + x];
            if (J.c1_add && (EXT || J.add_mode == 2)) c1v[q] = J.c1_add[(long long)m * N + x];
        }
    }
    // P c added as one more product in the accumulators (P mod q_m < q_m; one product more than
    // beta stays inside every accumulator's bound) instead of a Shoup multiply + modular add
    if (m < k) {
#pragma unroll
        for (int q = 0; q < kKsGroup; q++) {
            if (q < cnt) {
                accm(a0[q], c0v[q], pq.v[m], qd, qinv);
                accm(a1[q], c1v[q], pq.v[m], qd, qinv);
            }
        }
    }
#pragma unroll
    for (int q = 0; q < kKsGroup; q++) {
        if (q < cnt) {
            const int t = t0 + q;
            const KsJob &J = jobs.j[t];
            const u64 r0 = accr(a0[q], mc, qd, qinv), r1 = a1r(q);
            if (EXT) {
                const bool f = SMALL && J.out_f64;
                J.out[(long long)m * N + dst] = f ? (u64)__double_as_longlong((double)r0) : r0;
                J.out[((long long)E + m) * N + dst] = f ? (u64)__double_as_longlong((double)r1) : r1;
            } else {
                u[(((long long)t * 2 + 0) * E + m) * N + dst] = r0;
                u[(((long long)t * 2 + 1) * E + m) * N + dst] = r1;
            }
        }
    }
}

// grid (tiles * groups, E) with the group index fastest: the CTAs in flight cover every group of a
// few (limb, tile) slices, so groups that share a key (or an input's hoisted digits) read each tile
// from DRAM once and from L2 after that
#ifndef BLB_KS_MINB
#define BLB_KS_MINB 0   // 0: no launch bound (the compiler picks 64 registers); else CTAs per SM
#endif
template <int BETA, bool EXT = false>
__global__ void
#if BLB_KS_MINB > 0
__launch_bounds__(256, BLB_KS_MINB)
#endif
k_ks_inner(KsJobs jobs, KsGroups grp, u64 *u, Primes pr, int k, int np, int K, int beta_rt,
                           int logN, PinvTab pq) {
    const int gi = blockIdx.x % grp.n;
    const int x = (blockIdx.x / grp.n) * blockDim.x + threadIdx.x;
    const int m = blockIdx.y;
    if (x >= (1 << logN)) return;
    const int pm = m < k ? m : K + (m - k);
    const DigG ds{&jobs, (long long)m * (1 << logN) + x, (long long)(k + np) << logN};
    if (pr.m[pm].q < (1ull << 41)) ks_inner_body<BETA, EXT, true>(jobs, grp, u, pr, k, np, K, beta_rt, logN, pq, x, m, gi, ds);
    else ks_inner_body<BETA, EXT, false>(jobs, grp, u, pr, k, np, K, beta_rt, logN, pq, x, m, gi, ds);
}

// Bulk-staged key-switch inner product (the default for 1 <= beta <= 8).  A CTA owns a tile of
// kKsTile coefficients x of limb m for the jobs of one key group.  Thread 0 issues every input the
// tile needs -- the 2 beta key rows, the group's beta digit rows per job, the jobs' c0 / c1 rows -- as
// 1 KB cp.async.bulk copies into shared memory on one mbarrier, so a CTA keeps all of its ~38 KB in
// flight at once (the per-thread load version was bound by the loads its 64 registers could hold:
// long-scoreboard stalls first, 0.3 of HBM).  The products then run from shared memory one job at a
// time: AccG (FP64 pipe) on primes < 2^41, Acc60 on the 60-bit ones; same sums, additive P c term
// and scattered stores as ks_inner_body.
#ifndef BLB_KS_TILE
#define BLB_KS_TILE 128
#endif
constexpr int kKsTile = BLB_KS_TILE;  // coefficients per CTA
template <int BETA>
__host__ __device__ constexpr int ks_bulk_words(int T) { return (2 * BETA + kKsGroup * BETA + 2 * kKsGroup) * T; }
template <int BETA, bool EXT>
__global__ void __launch_bounds__(kKsTile) k_ks_bulk(KsJobs jobs, KsGroups grp, u64 *u, Primes pr, int k, int np,
                                                     int K, int logN, PinvTab pq) {
    extern __shared__ __align__(16) u64 ksm[];
    __shared__ uint64_t bar[kKsGroup];  // bar[q]: job q's rows (and, for q = 0, the key rows)
    const int N = 1 << logN, T = blockDim.x;
    const int gi = blockIdx.x % grp.n;
    const int x0 = (blockIdx.x / grp.n) * T;
    const int m = blockIdx.y;
    const int t0 = grp.start[gi], cnt = grp.start[gi + 1] - t0;
    const int E = k + np, Lk = K + np;
    const int pm = m < k ? m : K + (m - k);
    u64 *skey = ksm;                          // [2 BETA][T]: (j, b) -> 2 j + b
    u64 *sdig = ksm + 2 * BETA * T;           // [kKsGroup][BETA][T]
    u64 *sc = sdig + kKsGroup * BETA * T;     // [kKsGroup][2][T]: c0, c1
    const KsJob &J0 = jobs.j[t0];
    if (threadIdx.x == 0) {
        for (int q = 0; q < kKsGroup; q++) mbar_init(&bar[q], 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        // warp 0 issues the copies, one per lane at a time (lane 0 first registers the byte count)
        const unsigned tb = (unsigned)T * 8u;
        const int lane = threadIdx.x;
        const int nk = 2 * BETA, nd = cnt * BETA;
        int nc = 0;  // c0 / c1 rows present, in job order
        uint32_t cmask = 0;
        for (int q = 0; q < cnt; q++) {
            const KsJob &J = jobs.j[t0 + q];
            if (m < k && (EXT || J.add_mode != 0)) { cmask |= 1u << (2 * q); nc++; }
            if (m < k && J.c1_add && (EXT || J.add_mode == 2)) { cmask |= 1u << (2 * q + 1); nc++; }
        }
        if (lane < cnt) {  // lane q registers job q's bytes (job 0 also carries the keys)
            const int q = lane;
            const int ncq = ((cmask >> (2 * q)) & 1) + ((cmask >> (2 * q + 1)) & 1);
            mbar_expect_tx(&bar[q], (unsigned)((q == 0 ? nk : 0) + BETA + ncq) * tb);
        }
        __syncwarp();
        // job-major copy order (keys, then each job's digit and c rows), so job 0 lands first
        for (int c = lane; c < nk + nd + nc; c += 32) {
            if (c < nk) {
                const int j = c >> 1, b = c & 1;
                bulk_g2s(skey + c * T, J0.key + (((long long)j * 2 + b) * Lk + pm) * N + x0, tb, &bar[0]);
                continue;
            }
            int r = c - nk, q = 0;
            for (;; q++) {
                const int nq = BETA + ((cmask >> (2 * q)) & 1) + ((cmask >> (2 * q + 1)) & 1);
                if (r < nq) break;
                r -= nq;
            }
            const KsJob &J = jobs.j[t0 + q];
            if (r < BETA) {
                bulk_g2s(sdig + (q * BETA + r) * T, J.ext + ((long long)r * E + m) * N + x0, tb, &bar[q]);
            } else {
                const int slot = (r == BETA && ((cmask >> (2 * q)) & 1)) ? 2 * q : 2 * q + 1;
                bulk_g2s(sc + slot * T, ((slot & 1) ? J.c1_add : J.c0) + (long long)m * N + x0, tb, &bar[q]);
            }
        }
    }
    const int x = x0 + threadIdx.x;
    const uint32_t dst = J0.galois == 1 ? (uint32_t)x : galois_perm(x, J0.galois_inv, logN);
    const ModConst &mc = pr.m[pm];
    const bool small = mc.q < (1ull << 41);
    mbar_wait(&bar[0], 0);  // keys + job 0
    auto store = [&](int q, u64 r0, u64 r1) {
        const int t = t0 + q;
        if (EXT) {
            const KsJob &J = jobs.j[t];
            if (small && J.out_f64) {  // the ct-ct mask MACs read these limbs as doubles
                r0 = (u64)__double_as_longlong(AccF64::u2d(r0));
                r1 = (u64)__double_as_longlong(AccF64::u2d(r1));
            }
            J.out[(long long)m * N + dst] = r0;
            J.out[((long long)E + m) * N + dst] = r1;
        } else {
            u[(((long long)t * 2 + 0) * E + m) * N + dst] = r0;
            u[(((long long)t * 2 + 1) * E + m) * N + dst] = r1;
        }
    };
    // an absent c0 / c1 row contributes 0 (its slot was not filled)
    auto cval = [&](int q, int b) -> u64 {
        const KsJob &J = jobs.j[t0 + q];
        const bool has = b == 0 ? (EXT || J.add_mode != 0) : (J.c1_add && (EXT || J.add_mode == 2));
        return has ? sc[(2 * q + b) * T + threadIdx.x] : 0ull;
    };
    if (small) {
        const double qd = (double)mc.q, qinv = 1.0 / qd;
        double kb[BETA], ka[BETA];
#pragma unroll
        for (int j = 0; j < BETA; j++) {
            kb[j] = AccF64::u2d(skey[(2 * j) * T + threadIdx.x]);
            ka[j] = AccF64::u2d(skey[(2 * j + 1) * T + threadIdx.x]);
        }
        const double pc = m < k ? AccF64::u2d(pq.v[m]) : 0.0;
#pragma unroll 1
        for (int q = 0; q < cnt; q++) {
            if (q > 0) mbar_wait(&bar[q], 0);
            AccG a0, a1;
            a0.zero();
            a1.zero();
#pragma unroll
            for (int j = 0; j < BETA; j++) {
                const double e = AccF64::u2d(sdig[(q * BETA + j) * T + threadIdx.x]);
                a0.macd(e, kb[j]);
                a1.macd(e, ka[j]);
            }
            if (m < k) {
                a0.macd(AccF64::u2d(cval(q, 0)), pc);
                a1.macd(AccF64::u2d(cval(q, 1)), pc);
            }
            store(q, a0.reduce(qd, qinv), a1.reduce(qd, qinv));
        }
    } else {
        u64 kb[BETA], ka[BETA];
#pragma unroll
        for (int j = 0; j < BETA; j++) {
            kb[j] = skey[(2 * j) * T + threadIdx.x];
            ka[j] = skey[(2 * j + 1) * T + threadIdx.x];
        }
        // Acc60 holds <= 7 products (BETA <= 6 plus the P c term), Acc128 any number up to 64
        using A60 = typename std::conditional<(BETA <= 6), Acc60, Acc128>::type;
#pragma unroll 1
        for (int q = 0; q < cnt; q++) {
            if (q > 0) mbar_wait(&bar[q], 0);
            A60 a0, a1;
            a0.zero();
            a1.zero();
#pragma unroll
            for (int j = 0; j < BETA; j++) {
                const u64 e = sdig[(q * BETA + j) * T + threadIdx.x];
                a0.mac(e, kb[j]);
                a1.mac(e, ka[j]);
            }
            if (m < k) {
                a0.mac(cval(q, 0), pq.v[m]);
                a1.mac(cval(q, 1), pq.v[m]);
            }
            store(q, a0.reduce(mc), a1.reduce(mc));
        }
    }
}

// conv[t][b][i][x] = FastBConv_{P -> q_i}(INTT(u_P))   (u P-rows already INTT'd)
__global__ void k_bconv_moddown(const u64 *u, u64 *conv, const u64 *tb, Primes pr, int k, int np, int K, int N) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y, tb2 = blockIdx.z;  // tb2 = t*2 + b
    if (x >= N) return;
    const int E = k + np;
    if (np == 1) {  // single special prime: FastBConv_{P -> q_i}(y) = y mod q_i
        conv[((long long)tb2 * k + i) * N + x] = mod64(u[((long long)tb2 * E + k) * N + x], pr.m[i]);
        return;
    }
    Acc128 acc;
    acc.zero();
    for (int d = 0; d < np; d++) {
        const u64 v = u[((long long)tb2 * E + k + d) * N + x];
        const u64 y = shoup(v, tb[d], tb[np + d], pr.m[K + d].q);
        acc.mac(y, tb[2 * np + d * k + i]);
    }
    conv[((long long)tb2 * k + i) * N + x] = acc.reduce(pr.m[i]);
}

// out = (u_Q - conv) * P^{-1}  (+ sigma_g(c0) on poly 0 for rotations, + (c0, c1) for relin)
__global__ void k_ks_combine(KsJobs jobs, const u64 *u, const u64 *conv, PinvTab pinv, Primes pr, int k, int np,
                             int logN) {
    const int N = 1 << logN;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y;
    const int t = blockIdx.z >> 1, b = blockIdx.z & 1;
    if (x >= N) return;
    const KsJob &J = jobs.j[t];
    const int E = k + np;
    const u64 q = pr.m[i].q;
    const u64 uv = u[(((long long)t * 2 + b) * E + i) * N + x];
    const u64 cv = conv[(((long long)t * 2 + b) * k + i) * N + x];
    u64 r = shoup(uv + q - cv, pinv.v[i], pinv.sh[i], q);
    if (J.add_mode == 1 && b == 0) {
        const uint32_t src = J.galois == 1 ? (uint32_t)x : galois_perm(x, J.galois, logN);
        r = addmod(r, J.c0[(long long)i * N + src], q);
    } else if (J.add_mode == 2) {
        const u64 *c = b == 0 ? J.c0 : J.c1_add;
        r = addmod(r, c[(long long)i * N + x], q);
    }
    if (J.out_f64 && q < (1ull << 41)) r = (u64)__double_as_longlong((double)r);
    J.out[((long long)b * k + i) * N + x] = r;
}

// ------------------------------------------------------------- rescale (C10)
// last[p][x] = in[p][level][x]
__global__ void k_copy_limb(const u64 *in, u64 *out, int k, int limb, int N) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int p = blockIdx.y;
    if (x >= N) return;
    out[(long long)p * N + x] = in[((long long)p * k + limb) * N + x];
}
// r[p][i][x] = centred(last[p][x]) mod q_i, i < level
__global__ void k_rescale_lift(const u64 *last, u64 *r, Primes pr, int level, int N) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y, p = blockIdx.z;
    if (x >= N) return;
    const u64 ql = pr.m[level].q;
    const u64 v = last[(long long)p * N + x];
    const ModConst &mc = pr.m[i];
    u64 out;
    if (v <= (ql - 1) / 2) out = mod64(v, mc);
    else {
        const u64 neg = mod64(ql - v, mc);
        out = neg ? mc.q - neg : 0;
    }
    r[((long long)p * level + i) * N + x] = out;
}
// out[p][i][x] = (in[p][i][x] - r) * q_l^{-1} mod q_i
__global__ void k_rescale_combine(const u64 *in, const u64 *r, u64 *out, PinvTab qlinv, Primes pr, int level, int N) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y, p = blockIdx.z;
    if (x >= N) return;
    const u64 q = pr.m[i].q;
    const u64 a = in[((long long)p * (level + 1) + i) * N + x];
    const u64 b = r[((long long)p * level + i) * N + x];
    out[((long long)p * level + i) * N + x] = shoup(a + q - b, qlinv.v[i], qlinv.sh[i], q);
}

// ---------------------------------------------------------------- mask (C14)
// masked[t][0] += r, share[t] = -r mod q0 with r = ChaCha(MASK, (id0 + t) << 8) mod q0
__global__ void k_mask(u64 *masked, u64 *share, Primes pr, ChachaKey key, u64 id0, int N) {
    const int blk = blockIdx.x * blockDim.x + threadIdx.x;
    const int t = blockIdx.y;
    if (blk >= N / 4) return;
    u64 lo[4], hi[4];
    draw_block(key, TAG_MASK, (id0 + (u64)t) << 8, blk, lo, hi);
    const ModConst &mc = pr.m[0];
    u64 *m0 = masked + (long long)t * 2 * N;
    u64 *sh = share + (long long)t * N;
#pragma unroll
    for (int d = 0; d < 4; d++) {
        const u64 r = reduce128(hi[d], lo[d], mc);
        const int x = 4 * blk + d;
        m0[x] = addmod(m0[x], r, mc.q);
        sh[x] = r ? mc.q - r : 0;
    }
}
// masked[t][b][x] = in_t[b][0][x]   (drop to q_0)
__global__ void k_drop_q0(PtrList in, u64 *masked, int k, int N) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int t = blockIdx.y, b = blockIdx.z;
    if (x >= N) return;
    masked[((long long)t * 2 + b) * N + x] = in.p[t][(long long)b * k * N + x];
}

// ct (x) ct tensor (C9): d = (a0 b0, a0 b1 + a1 b0, a1 b1)
__global__ void k_tensor(const u64 *a, const u64 *b, u64 *d, Primes pr, int k, int N) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int l = blockIdx.y;
    if (x >= N) return;
    const long long kN = (long long)k * N, lx = (long long)l * N + x;
    const u64 a0 = a[lx], a1 = a[kN + lx], b0 = b[lx], b1 = b[kN + lx];
    const ModConst &mc = pr.m[l];
    Acc128 s;
    s.zero();
    s.mac(a0, b1);
    s.mac(a1, b0);
    d[lx] = mulmod(a0, b0, mc);
    d[kN + lx] = s.reduce(mc);
    d[2 * kN + lx] = mulmod(a1, b1, mc);
}

// n tensors (C9) in one launch: d[t] = (a0 b0, a0 b1 + a1 b0, a1 b1) of the pair (a[t], b[t]), [n][3][k][N]
__global__ void k_tensor_n(PtrList a, PtrList b, u64 *d, Primes pr, int k, int N) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int l = blockIdx.y, t = blockIdx.z;
    if (x >= N) return;
    const long long kN = (long long)k * N, lx = (long long)l * N + x;
    const u64 a0 = a.p[t][lx], a1 = a.p[t][kN + lx], b0 = b.p[t][lx], b1 = b.p[t][kN + lx];
    const ModConst &mc = pr.m[l];
    Acc128 s;
    s.zero();
    s.mac(a0, b1);
    s.mac(a1, b0);
    u64 *o = d + (long long)t * 3 * kN + lx;
    o[0] = mulmod(a0, b0, mc);
    o[kN] = s.reduce(mc);
    o[2 * kN] = mulmod(a1, b1, mc);
}

inline dim3 grid_x(int N, int y = 1, int z = 1) { return dim3((N + kTB - 1) / kTB, y, z); }
}  // namespace

// n ct x pt products in one launch: out[t] = (c0 * pt[t], c1 * pt[t]) into [n][2][k][N]
__global__ void k_mul_pt_n(PtrList in, PtrList pt, u64 *out, Primes pr, int k, int N) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y, t = blockIdx.z;
    if (x >= N) return;
    const ModConst &mc = pr.m[i];
    const long long kN = (long long)k * N, lx = (long long)i * N + x;
    const u64 p = pt.p[t][lx];
    u64 *o = out + (long long)t * 2 * kN + lx;
    o[0] = mulmod(in.p[t][lx], p, mc);
    o[kN] = mulmod(in.p[t][kN + lx], p, mc);
}
blb_status blb_launch_mul_pt_n(const blb_params *P, const u64 *const *in, const u64 *const *pt, int n, u64 *out, int k,
                               cudaStream_t st) {
    if (n <= 0) return BLB_OK;
    if (n > kMaxJobs) return BLB_E_INVALID_ARG;
    PtrList a{}, b{};
    for (int t = 0; t < n; t++) { a.p[t] = in[t]; b.p[t] = pt[t]; }
    k_mul_pt_n<<<grid_x(P->N, k, n), kTB, 0, st>>>(a, b, out, P->pr, k, P->N);
    BLB_COUNT_LAUNCH(1);
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}
blb_status blb_launch_tensor_n(const blb_params *P, const u64 *const *a, const u64 *const *b, int n, u64 *d, int k,
                               cudaStream_t st) {
    if (n <= 0) return BLB_OK;
    if (n > kMaxJobs) return BLB_E_INVALID_ARG;
    PtrList pa{}, pb{};
    for (int t = 0; t < n; t++) { pa.p[t] = a[t]; pb.p[t] = b[t]; }
    k_tensor_n<<<grid_x(P->N, k, n), kTB, 0, st>>>(pa, pb, d, P->pr, k, P->N);
    BLB_COUNT_LAUNCH(1);
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}

blb_status blb_launch_tensor(const blb_params *P, const u64 *a, const u64 *b, u64 *d, int k, cudaStream_t st) {
    k_tensor<<<grid_x(P->N, k), kTB, 0, st>>>(a, b, d, P->pr, k, P->N);
    BLB_COUNT_LAUNCH(1);
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}

// ============================================================ launchers
extern "C" u64 blbh_shoup(u64 w, u64 q);
extern "C" u64 blbh_mulmod(u64 a, u64 b, u64 q);
extern "C" u64 blbh_invmod(u64 a, u64 q);
static u64 blbh_shoup_dev_table(const blb_params *P, int i) { return blbh_shoup(P->P_mod_q[i], P->mod[i]); }

ChachaKey chacha_key_from_bytes(const uint8_t seed[32]) {
    ChachaKey k;
    for (int i = 0; i < 8; i++)
        k.k[i] = (uint32_t)seed[4 * i] | ((uint32_t)seed[4 * i + 1] << 8) | ((uint32_t)seed[4 * i + 2] << 16) |
                 ((uint32_t)seed[4 * i + 3] << 24);
    return k;
}

blb_status launch_modup(const blb_params *P, int level, const u64 *const *c1_ntt, int n, u64 *ext, u64 *coef,
                        cudaStream_t st) {
    if (n <= 0) return BLB_OK;
    if (n > kMaxJobs) {
        blb_set_error("launch_modup: n > %d", kMaxJobs);
        return BLB_E_INVALID_ARG;
    }
    const int N = P->N, k = level + 1, E = k + P->np, beta = blb_beta(P, level);
    PtrList src{};
    for (int t = 0; t < n; t++) src.p[t] = c1_ntt[t];
    RowBatch rb{};
    rb.base = coef; rb.poly_stride = (long long)k * N; rb.n_polys = n; rb.limbs = k; rb.limb0 = 0;
    for (int i = 0; i < k; i++) rb.prime[i] = i;
    if ((P->logN == 16 || P->logN == 15) && P->alpha == 1) {
        // fused: the INTT's first pass reads the c1 rows in place (no gather copy); in the forward
        // NTT's first pass the own rows are copied and the others converted (x mod q_m)
        NttFuse gz{};
        gz.pro = 2;
        for (int t = 0; t < n; t++) gz.srcp.p[t] = c1_ntt[t];
        BLB_TRY(launch_ntt_fused(P, rb, true, gz, st));
        RowBatch eb{};
        eb.base = ext; eb.poly_stride = (long long)E * N; eb.n_polys = n * beta; eb.limbs = E; eb.limb0 = 0;
        for (int m = 0; m < E; m++) eb.prime[m] = m < k ? m : P->K + (m - k);
        eb.skip_alpha = 1; eb.skip_beta = beta; eb.skip_kmax = k;
        NttFuse fz{};
        fz.pro = 1;
        fz.src = coef;
        fz.src_div = beta;
        fz.src_nq = beta;  // alpha = 1: digit j holds residues mod q_j
        for (int j = 0; j < beta && j < 8; j++) fz.src_q[j] = P->mod[j];
        fz.src_hi = (long long)k * N;
        fz.src_lo = N;
        fz.copy_own = 1;
        for (int t = 0; t < n; t++) fz.srcp.p[t] = c1_ntt[t];
        return launch_ntt_fused(P, eb, false, fz, st);
    }
    k_gather_rows<<<grid_x(N, k, n), kTB, 0, st>>>(src, coef, k, N);
    BLB_COUNT_LAUNCH(1);
    BLB_TRY(launch_ntt(P, rb, true, st));
    Offs offs{};
    for (int j = 0; j < beta; j++) offs.o[j] = (long long)bconv_modup_off(P, level, j);
    k_bconv_modup<<<grid_x(N, E, n * beta), kTB, 0, st>>>(src, coef, ext, P->d_bconv, offs, P->pr, k, P->np, P->K,
                                                          P->alpha, beta, N);
    BLB_COUNT_LAUNCH(1);
    BLB_CHECK_LAUNCH();
    RowBatch eb{};
    eb.base = ext; eb.poly_stride = (long long)E * N; eb.n_polys = n * beta; eb.limbs = E; eb.limb0 = 0;
    for (int m = 0; m < E; m++) eb.prime[m] = m < k ? m : P->K + (m - k);
    eb.skip_alpha = P->alpha; eb.skip_beta = beta; eb.skip_kmax = k;
    return launch_ntt(P, eb, false, st);
}

size_t keyswitch_scratch_elems(const blb_params *P, int level, int n_jobs) {
    const int k = level + 1, E = k + P->np;
    return (size_t)n_jobs * 2 * ((size_t)E + k) * P->N;
}

// group jobs that share a key (stable order by key), <= kKsGroup per group
// g^{-1} mod 2N (g odd): g^(N-1), the group (Z/2N)^* having exponent dividing N
static uint32_t galois_inverse(uint32_t g, int logN) {
    const u64 m = 2ull << logN;
    u64 r = 1, b = g % m, e = (1ull << logN) - 1;
    while (e) {
        if (e & 1) r = r * b % m;
        b = b * b % m;
        e >>= 1;
    }
    return (uint32_t)r;
}
static void group_jobs(const KsJob *jobs, int n, KsJobs &J, KsGroups &G, int logN) {
    bool used[kMaxJobs] = {false};
    int t = 0;
    G.n = 0;
    for (int a = 0; a < n; a++) {
        if (used[a]) continue;
        G.start[G.n++] = t;
        int cnt = 0;
        for (int b = a; b < n && cnt < kKsGroup; b++)
            if (!used[b] && jobs[b].key == jobs[a].key && jobs[b].galois == jobs[a].galois) {
                used[b] = true;
                J.j[t] = jobs[b];
                J.j[t].galois_inv = galois_inverse(jobs[b].galois, logN);
                t++;
                cnt++;
            }
    }
    G.start[G.n] = t;
}

template <bool EXT>
static blb_status ks_inner_launch(const blb_params *P, int level, const KsJobs &J, const KsGroups &G, u64 *u,
                                  cudaStream_t st) {
    const int N = P->N, k = level + 1, np = P->np, E = k + np, beta = blb_beta(P, level);
    PinvTab pq{};
    for (int i = 0; i < k; i++) {
        pq.v[i] = P->P_mod_q[i];
        pq.sh[i] = blbh_shoup_dev_table(P, i);
    }
    cudaEvent_t t0 = blb_timing_begin(st);
    const int T = N < kKsTile ? N : kKsTile;
    const dim3 gb((unsigned)((N / T) * G.n), E);
    switch (beta) {
#define KSB(B)                                                                                               \
    case B: {                                                                                                \
        const size_t sm = (size_t)ks_bulk_words<B>(T) * 8;                                                    \
        if (sm > 48 * 1024) blb_smem_optin(k_ks_bulk<B, EXT>, sm);                                            \
        k_ks_bulk<B, EXT><<<gb, T, sm, st>>>(J, G, u, P->pr, k, np, P->K, P->logN, pq);                       \
        break;                                                                                               \
    }
        KSB(1) KSB(2) KSB(3) KSB(4) KSB(5) KSB(6) KSB(7) KSB(8)
#undef KSB
        default: {  // beta > 8: the per-thread kernel with a runtime digit count
            const dim3 gks((unsigned)(((N + kTB - 1) / kTB) * G.n), E);
            k_ks_inner<0, EXT><<<gks, kTB, 0, st>>>(J, G, u, P->pr, k, np, P->K, beta, P->logN, pq);
        }
    }
    BLB_COUNT_LAUNCH(1);
    // algorithmic bytes: each distinct key once (groups sharing a key read it through L2)
    int n_keys = 0;
    for (int g = 0; g < G.n; g++) {
        bool seen = false;
        for (int h = 0; h < g && !seen; h++) seen = J.j[G.start[h]].key == J.j[G.start[g]].key;
        n_keys += !seen;
    }
    blb_timing_end(2, t0, st, (double)n_keys * 2.0 * beta * E * N * 8.0);
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}

// ModDown of u[t] ([2][E][N], extended basis) into J.j[t].out with the job's add mode
static blb_status moddown_launch(const blb_params *P, int level, const KsJobs &J, int n, u64 *u, u64 *conv,
                                 cudaStream_t st) {
    const int N = P->N, k = level + 1, np = P->np, E = k + np;
    RowBatch rb{};
    rb.base = u; rb.poly_stride = (long long)E * N; rb.n_polys = 2 * n; rb.limbs = np; rb.limb0 = k;
    for (int d = 0; d < np; d++) rb.prime[d] = P->K + d;
    BLB_TRY(launch_ntt(P, rb, true, st));
    if ((P->logN == 16 || P->logN == 15) && np == 1) {
        // fused ModDown: conv = NTT(u_P mod q_i) with the reduction in the first pass and
        // (u_i - conv) * P^{-1} (+ sigma(c0) / (c0, c1)) in the last pass
        RowBatch cb{};
        cb.base = conv; cb.poly_stride = (long long)k * N; cb.n_polys = 2 * n; cb.limbs = k; cb.limb0 = 0;
        for (int i = 0; i < k; i++) cb.prime[i] = i;
        NttFuse fz{};
        fz.pro = 1;
        fz.src = u + (long long)k * N;
        fz.src_div = 1;
        fz.src_nq = 1;  // residues mod the special prime
        fz.src_q[0] = P->mod[P->K];
        fz.src_hi = (long long)E * N;
        fz.epi = 1;
        fz.u = u;
        fz.E = E;
        fz.k = k;
        for (int i = 0; i < k; i++) { fz.pinv.v[i] = P->Pinv[i]; fz.pinv.sh[i] = P->Pinv_sh[i]; }
        fz.jobs = J;
        return launch_ntt_fused(P, cb, false, fz, st);
    }
    k_bconv_moddown<<<grid_x(N, k, 2 * n), kTB, 0, st>>>(u, conv, P->d_bconv + bconv_moddown_off(P, level), P->pr, k,
                                                         np, P->K, N);
    BLB_COUNT_LAUNCH(1);
    BLB_CHECK_LAUNCH();
    RowBatch cb{};
    cb.base = conv; cb.poly_stride = (long long)k * N; cb.n_polys = 2 * n; cb.limbs = k; cb.limb0 = 0;
    for (int i = 0; i < k; i++) cb.prime[i] = i;
    BLB_TRY(launch_ntt(P, cb, false, st));
    PinvTab pt{};
    for (int i = 0; i < k; i++) { pt.v[i] = P->Pinv[i]; pt.sh[i] = P->Pinv_sh[i]; }
    k_ks_combine<<<grid_x(N, k, 2 * n), kTB, 0, st>>>(J, u, conv, pt, P->pr, k, np, P->logN);
    BLB_COUNT_LAUNCH(1);
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}

blb_status launch_keyswitch(const blb_params *P, int level, const KsJob *jobs, int n, u64 *u, u64 *conv,
                            cudaStream_t st) {
    if (n <= 0) return BLB_OK;
    if (n > kMaxJobs) {
        blb_set_error("launch_keyswitch: n > %d", kMaxJobs);
        return BLB_E_INVALID_ARG;
    }
    KsJobs J{};
    KsGroups G{};
    group_jobs(jobs, n, J, G, P->logN);
    BLB_TRY(ks_inner_launch<false>(P, level, J, G, u, st));
    // sigma_g(c0) / (c0, c1) were folded into u as P * c by the inner product: plain ModDown
    for (int t = 0; t < n; t++) J.j[t].add_mode = 0;
    BLB_TRY(moddown_launch(P, level, J, n, u, conv, st));
    BLB_COUNT(1, n);
    return BLB_OK;
}

blb_status launch_keyswitch_ext(const blb_params *P, int level, const KsJob *jobs, int n, cudaStream_t st) {
    if (n <= 0) return BLB_OK;
    if (n > kMaxJobs) return BLB_E_INVALID_ARG;
    KsJobs J{};
    KsGroups G{};
    group_jobs(jobs, n, J, G, P->logN);
    BLB_TRY(ks_inner_launch<true>(P, level, J, G, nullptr, st));
    BLB_COUNT(1, n);
    return BLB_OK;
}

blb_status launch_moddown(const blb_params *P, int level, u64 *u, int n, u64 *out, u64 *conv, cudaStream_t st) {
    const int N = P->N, k = level + 1, E = k + P->np;
    for (int t0 = 0; t0 < n; t0 += kMaxJobs) {
        const int cnt = n - t0 < kMaxJobs ? n - t0 : kMaxJobs;
        KsJobs J{};
        for (int t = 0; t < cnt; t++) {
            J.j[t].out = out + (size_t)(t0 + t) * 2 * k * N;
            J.j[t].add_mode = 0;
            J.j[t].galois = 1;
        }
        BLB_TRY(moddown_launch(P, level, J, cnt, u + (size_t)t0 * 2 * E * N, conv, st));
    }
    return BLB_OK;
}

// ---------------------------------------------------------------------------
// ModDown fused with rescale (reading C17): y = round(X / M), M = q_l * p_0 ... (odd: no ties),
// y = (X + h - r) / M with h = (M - 1) / 2 and r = (X + h) mod M rebuilt exactly from the
// residues at the M-moduli by Garner's mixed radix (digits d_t < m_t), reduced mod q_i by Horner.
// ---------------------------------------------------------------------------
constexpr int kMdrMax = 5;  // q_l + up to 4 special primes (dnum = 1 at k = 5, reading C23)
struct MdrTab {
    int nd;
    ModConst md[kMdrMax];                          // m_0 = q_l, m_1.. = p_0..
    u64 hd[kMdrMax];                               // h mod m_t = (m_t - 1) / 2
    u64 gi[kMdrMax][kMdrMax], gish[kMdrMax][kMdrMax];  // m_s^{-1} mod m_t (s < t), Shoup
    u64 mq[kMdrMax][BLB_MAXP], mqsh[kMdrMax][BLB_MAXP];  // m_t mod q_i, Shoup
    u64 hq[BLB_MAXP];                              // h mod q_i
};
// u: [2n][E][N], limbs k-1 .. E-1 (q_l, P) already INTT'd in place;  conv [2n][level][N] = (r - h) mod q_i
__global__ void k_mdr_lift(const u64 *u, u64 *conv, MdrTab T, Primes pr, int k, int E, int N) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int pp = blockIdx.z;
    if (x >= N) return;
    const int level = k - 1;
    const u64 *base = u + ((long long)pp * E + level) * N + x;
    u64 d[kMdrMax], in[kMdrMax];
#pragma unroll
    for (int t = 0; t < kMdrMax; t++) in[t] = t < T.nd ? base[(long long)t * N] : 0;  // loads issued together
#pragma unroll
    for (int t = 0; t < kMdrMax; t++) {
        if (t >= T.nd) break;
        const u64 mt = T.md[t].q;
        u64 v = in[t] + T.hd[t];
        if (v >= mt) v -= mt;
#pragma unroll
        for (int s2 = 0; s2 < kMdrMax; s2++) {
            if (s2 >= t) break;
            v = submod(v, mod64(d[s2], T.md[t]), mt);
            v = shoup(v, T.gi[s2][t], T.gish[s2][t], mt);
        }
        d[t] = v;
    }
    if (T.nd == 2) {
        // one special prime: r = d1 m0 + d0 mod q_i.  The Shoup product takes d1 < 2^64 directly (no
        // reduction of d1 first), and d0 < m0 = q_l is below 2 q_i for the chain's same-size primes
        // (one conditional subtraction; the general reduction only if it is not)
        for (int i = 0; i < level; i++) {
            const ModConst &mc = pr.m[i];
            u64 d0 = d[0];
            if (d0 >= mc.q) d0 -= mc.q;
            if (d0 >= mc.q) d0 = mod64(d0, mc);
            const u64 r = addmod(shoup(d[1], T.mq[0][i], T.mqsh[0][i], mc.q), d0, mc.q);
            conv[((long long)pp * level + i) * N + x] = submod(r, T.hq[i], mc.q);
        }
        return;
    }
    for (int i = 0; i < level; i++) {
        const ModConst &mc = pr.m[i];
        u64 r = mod64(d[T.nd - 1], mc);
        for (int t = T.nd - 2; t >= 0; t--) r = addmod(shoup(r, T.mq[t][i], T.mqsh[t][i], mc.q), mod64(d[t], mc), mc.q);
        conv[((long long)pp * level + i) * N + x] = submod(r, T.hq[i], mc.q);
    }
}
// out_i = (u_i - NTT(conv)_i) * M^{-1}  (generic-N path; N = 2^16 fuses this into the NTT epilogue)
__global__ void k_mdr_combine(const u64 *u, const u64 *conv, KsJobs J, PinvTab mi, Primes pr, int level, int E,
                              int N) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int l = blockIdx.y, pp = blockIdx.z;
    if (x >= N) return;
    const u64 q = pr.m[l].q;
    const u64 v = submod(u[((long long)pp * E + l) * N + x], conv[((long long)pp * level + l) * N + x], q);
    J.j[pp >> 1].out[((long long)(pp & 1) * level + l) * N + x] = shoup(v, mi.v[l], mi.sh[l], q);
}

// u [n][2][E][N] (modified: its q_l and P limbs are INTT'd in place) -> outs[t] [2][level][N]
blb_status launch_moddown_rescale(const blb_params *P, int level, u64 *u, int n, u64 *const *outs, u64 *conv,
                                  cudaStream_t st) {
    if (n <= 0) return BLB_OK;
    const int N = P->N, k = level + 1, np = P->np, E = k + np, nd = 1 + np;
    if (level < 1 || nd > kMdrMax) {
        blb_set_error("moddown_rescale: level %d / %d special primes unsupported", level, np);
        return BLB_E_INVALID_ARG;
    }
    MdrTab T{};
    T.nd = nd;
    u64 m[kMdrMax];
    for (int t = 0; t < nd; t++) {
        m[t] = t == 0 ? P->mod[level] : P->mod[P->K + t - 1];
        T.md[t] = P->pr.m[t == 0 ? level : P->K + t - 1];
        T.hd[t] = (m[t] - 1) / 2;
    }
    for (int t = 0; t < nd; t++)
        for (int s2 = 0; s2 < t; s2++) {
            T.gi[s2][t] = blbh_invmod(m[s2] % m[t], m[t]);
            T.gish[s2][t] = blbh_shoup(T.gi[s2][t], m[t]);
        }
    PinvTab mi{};
    for (int i = 0; i < level; i++) {
        const u64 qi = P->mod[i];
        u64 Mq = 1;
        for (int t = 0; t < nd; t++) {
            T.mq[t][i] = m[t] % qi;
            T.mqsh[t][i] = blbh_shoup(T.mq[t][i], qi);
            Mq = blbh_mulmod(Mq, T.mq[t][i], qi);
        }
        T.hq[i] = blbh_mulmod((Mq + qi - 1) % qi, blbh_invmod(2, qi), qi);
        mi.v[i] = blbh_invmod(Mq, qi);
        mi.sh[i] = blbh_shoup(mi.v[i], qi);
    }
    for (int t0 = 0; t0 < n; t0 += kMaxJobs) {
        const int cnt = n - t0 < kMaxJobs ? n - t0 : kMaxJobs;
        u64 *ub = u + (size_t)t0 * 2 * E * N;
        RowBatch rb{};
        rb.base = ub; rb.poly_stride = (long long)E * N; rb.n_polys = 2 * cnt; rb.limbs = nd; rb.limb0 = level;
        for (int t = 0; t < nd; t++) rb.prime[t] = t == 0 ? level : P->K + t - 1;
        BLB_TRY(launch_ntt(P, rb, true, st));
        k_mdr_lift<<<grid_x(N, 1, 2 * cnt), kTB, 0, st>>>(ub, conv, T, P->pr, k, E, N);
        BLB_COUNT_LAUNCH(1);
        BLB_CHECK_LAUNCH();
        KsJobs J{};
        for (int t = 0; t < cnt; t++) {
            J.j[t].out = outs[t0 + t];
            J.j[t].add_mode = 0;
            J.j[t].galois = 1;
        }
        RowBatch cb{};
        cb.base = conv; cb.poly_stride = (long long)level * N; cb.n_polys = 2 * cnt; cb.limbs = level; cb.limb0 = 0;
        for (int i = 0; i < level; i++) cb.prime[i] = i;
        if (P->logN == 16 || P->logN == 15) {
            NttFuse fz{};
            fz.epi = 1;
            fz.u = ub;
            fz.E = E;
            fz.k = level;
            fz.pinv = mi;
            fz.jobs = J;
            BLB_TRY(launch_ntt_fused(P, cb, false, fz, st));
        } else {
            BLB_TRY(launch_ntt(P, cb, false, st));
            k_mdr_combine<<<grid_x(N, level, 2 * cnt), kTB, 0, st>>>(ub, conv, J, mi, P->pr, level, E, N);
            BLB_COUNT_LAUNCH(1);
            BLB_CHECK_LAUNCH();
        }
    }
    BLB_COUNT(4, n);
    return BLB_OK;
}
blb_status launch_moddown_rescale(const blb_params *P, int level, u64 *u, int n, u64 *out, u64 *conv,
                                  cudaStream_t st) {
    std::vector<u64 *> o(n);
    for (int t = 0; t < n; t++) o[t] = out + (size_t)t * 2 * level * P->N;
    return launch_moddown_rescale(P, level, u, n, o.data(), conv, st);
}
// ModDown of n extended ciphertexts into separate outputs
blb_status launch_moddown(const blb_params *P, int level, u64 *u, int n, u64 *const *outs, u64 *conv,
                          cudaStream_t st) {
    const int N = P->N, k = level + 1, E = k + P->np;
    for (int t0 = 0; t0 < n; t0 += kMaxJobs) {
        const int cnt = n - t0 < kMaxJobs ? n - t0 : kMaxJobs;
        KsJobs J{};
        for (int t = 0; t < cnt; t++) {
            J.j[t].out = outs[t0 + t];
            J.j[t].add_mode = 0;
            J.j[t].galois = 1;
        }
        BLB_TRY(moddown_launch(P, level, J, cnt, u + (size_t)t0 * 2 * E * N, conv, st));
    }
    return BLB_OK;
}

// lift a Q_l ciphertext to Q_l u P: (P c0, P c1) on the q limbs, 0 on the p limbs
__global__ void k_lift_ext(const u64 *in, u64 *out, PinvTab pq, Primes pr, int k, int np, int N, int f64) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int m = blockIdx.y, p = blockIdx.z;
    if (x >= N) return;
    const int E = k + np;
    u64 v = 0;
    if (m < k) {
        v = shoup(in[((long long)p * k + m) * N + x], pq.v[m], pq.sh[m], pr.m[m].q);
        if (f64 && pr.m[m].q < (1ull << 41)) v = (u64)__double_as_longlong((double)v);
    }
    out[((long long)p * E + m) * N + x] = v;  // P limbs: 0 (also as a double)
}
blb_status launch_lift_ext(const blb_params *P, int level, const u64 *in, u64 *out, cudaStream_t st, bool f64) {
    const int k = level + 1;
    PinvTab pq{};
    for (int i = 0; i < k; i++) { pq.v[i] = P->P_mod_q[i]; pq.sh[i] = blbh_shoup_dev_table(P, i); }
    k_lift_ext<<<grid_x(P->N, k + P->np, 2), kTB, 0, st>>>(in, out, pq, P->pr, k, P->np, P->N, f64 ? 1 : 0);
    BLB_COUNT_LAUNCH(1);
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}

extern "C" u64 blbh_shoup(u64 w, u64 q);
extern "C" u64 blbh_invmod(u64 a, u64 q);

blb_status launch_rescale(const blb_params *P, const u64 *in, int level, int n_polys, u64 *out, u64 *scratch,
                          cudaStream_t st) {
    const int N = P->N, k = level + 1;
    u64 *last = scratch, *r = scratch + (size_t)n_polys * N;
    k_copy_limb<<<grid_x(N, n_polys), kTB, 0, st>>>(in, last, k, level, N);
    BLB_COUNT_LAUNCH(1);
    RowBatch lb{};
    lb.base = last; lb.poly_stride = N; lb.n_polys = n_polys; lb.limbs = 1; lb.limb0 = 0; lb.prime[0] = level;
    BLB_TRY(launch_ntt(P, lb, true, st));
    k_rescale_lift<<<grid_x(N, level, n_polys), kTB, 0, st>>>(last, r, P->pr, level, N);
    BLB_COUNT_LAUNCH(1);
    RowBatch rb{};
    rb.base = r; rb.poly_stride = (long long)level * N; rb.n_polys = n_polys; rb.limbs = level; rb.limb0 = 0;
    for (int i = 0; i < level; i++) rb.prime[i] = i;
    BLB_TRY(launch_ntt(P, rb, false, st));
    PinvTab qi{};
    const u64 ql = P->mod[level];
    for (int i = 0; i < level; i++) {
        qi.v[i] = blbh_invmod(ql % P->mod[i], P->mod[i]);
        qi.sh[i] = blbh_shoup(qi.v[i], P->mod[i]);
    }
    k_rescale_combine<<<grid_x(N, level, n_polys), kTB, 0, st>>>(in, r, out, qi, P->pr, level, N);
    BLB_COUNT_LAUNCH(1);
    BLB_COUNT(4, n_polys / 2);
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}

// ------------------------------------------------ exported through api.cu
blb_status blb_launch_sample_uniform(const blb_params *P, u64 *out, long long row_stride, int n_rows,
                                     const int *prime, const int *nonce, const uint8_t seed[32], uint32_t tag, u64 id,
                                     cudaStream_t st) {
    LimbList ll{};
    ll.n = n_rows;
    for (int r = 0; r < n_rows; r++) { ll.prime[r] = prime[r]; ll.nonce[r] = nonce[r]; }
    k_sample_uniform<<<dim3((P->N / 4 + kTB - 1) / kTB, n_rows), kTB, 0, st>>>(out, row_stride, ll, P->pr,
                                                                              chacha_key_from_bytes(seed), tag, id, P->N);
    BLB_COUNT_LAUNCH(1);
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}
blb_status blb_launch_sample_small(const blb_params *P, u64 *out, long long row_stride, int n_rows, const int *prime,
                                   const uint8_t seed[32], uint32_t tag, u64 id, int mode, cudaStream_t st) {
    LimbList ll{};
    ll.n = n_rows;
    for (int r = 0; r < n_rows; r++) ll.prime[r] = prime[r];
    k_sample_small<<<(P->N / 4 + kTB - 1) / kTB, kTB, 0, st>>>(out, row_stride, ll, P->pr, chacha_key_from_bytes(seed),
                                                               tag, id, mode, P->N);
    BLB_COUNT_LAUNCH(1);
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}
blb_status blb_launch_keygen_combine(const blb_params *P, u64 *b, const u64 *a, const u64 *s, long long stride,
                                     int n_rows, const int *prime, uint32_t galois, int relin, const u64 *gadget_dev,
                                     cudaStream_t st) {
    LimbList ll{};
    ll.n = n_rows;
    for (int r = 0; r < n_rows; r++) ll.prime[r] = prime[r];
    k_keygen_combine<<<grid_x(P->N, n_rows), kTB, 0, st>>>(b, a, s, stride, ll, P->pr, galois, relin, gadget_dev,
                                                           P->logN);
    BLB_COUNT_LAUNCH(1);
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}
blb_status blb_launch_encrypt_combine(const blb_params *P, u64 *c0, const u64 *c1, const u64 *s, const u64 *pt, int k,
                                      cudaStream_t st) {
    k_encrypt_combine<<<grid_x(P->N, k), kTB, 0, st>>>(c0, c1, s, pt, P->pr, P->N);
    BLB_COUNT_LAUNCH(1);
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}
blb_status blb_launch_decrypt(const blb_params *P, const u64 *c0, const u64 *c1, const u64 *s, u64 *out, int k,
                              cudaStream_t st) {
    k_decrypt<<<grid_x(P->N, k), kTB, 0, st>>>(c0, c1, s, out, P->pr, P->N);
    BLB_COUNT_LAUNCH(1);
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}
blb_status blb_launch_mul_pt(const blb_params *P, const u64 *in, const u64 *pt, u64 *out, int k, cudaStream_t st) {
    k_mul_pt<<<grid_x(P->N, k, 2), kTB, 0, st>>>(in, pt, out, P->pr, k, P->N);
    BLB_COUNT_LAUNCH(1);
    BLB_COUNT(3, 1);
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}
blb_status blb_launch_add(const blb_params *P, const u64 *a, const u64 *b, u64 *out, int k, int npoly,
                          cudaStream_t st) {
    k_add<<<grid_x(P->N, k, npoly), kTB, 0, st>>>(a, b, out, P->pr, k, P->N);
    BLB_COUNT_LAUNCH(1);
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}
blb_status blb_launch_sub(const blb_params *P, const u64 *a, const u64 *b, u64 *out, int k, int npoly,
                          cudaStream_t st) {
    k_sub<<<grid_x(P->N, k, npoly), kTB, 0, st>>>(a, b, out, P->pr, k, P->N);
    BLB_COUNT_LAUNCH(1);
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}
// S13 re-randomisation of n level-0 ciphertexts rr[t] ([2][N], NTT, modified in place) with the public
// key pk ([2][kpk][N]); vee: scratch [n][3][N]
blb_status blb_launch_rerand(const blb_params *P, u64 *const *rr, int n, const u64 *pk, int kpk, const uint8_t seed[32],
                             u64 id0, int flood_bits, u64 *vee, cudaStream_t st) {
    const int N = P->N;
    const ChachaKey key = chacha_key_from_bytes(seed);
    LimbList ll{};
    ll.n = 1;
    ll.prime[0] = 0;
    for (int t = 0; t < n; t++) {
        u64 *r = vee + (size_t)t * 3 * N;
        k_sample_small<<<(N / 4 + kTB - 1) / kTB, kTB, 0, st>>>(r, N, ll, P->pr, key, TAG_RR_V, id0 + t, 0, N);
        k_sample_small<<<(N / 4 + kTB - 1) / kTB, kTB, 0, st>>>(r + 2 * (size_t)N, N, ll, P->pr, key, TAG_RR_E1, id0 + t, 1, N);
        if (flood_bits == 0)
            k_sample_small<<<(N / 4 + kTB - 1) / kTB, kTB, 0, st>>>(r + N, N, ll, P->pr, key, TAG_RR_E0, id0 + t, 1, N);
        BLB_COUNT_LAUNCH(flood_bits == 0 ? 3 : 2);
    }
    if (flood_bits > 0) {
        // e0 rows of all conversions: row t of a [n][N] view with stride 3N -> write per conversion
        for (int t = 0; t < n; t++) {
            k_sample_flood<<<dim3((N / 4 + kTB - 1) / kTB, 1), kTB, 0, st>>>(vee + ((size_t)t * 3 + 1) * N, P->pr, key,
                                                                            id0 + t, flood_bits, N);
            BLB_COUNT_LAUNCH(1);
        }
    }
    BLB_CHECK_LAUNCH();
    RowBatch rb{};
    rb.base = vee; rb.poly_stride = N; rb.n_polys = 3 * n; rb.limbs = 1; rb.limb0 = 0; rb.prime[0] = 0;
    BLB_TRY(launch_ntt(P, rb, false, st));
    for (int t0 = 0; t0 < n; t0 += kMaxJobs) {
        const int cnt = std::min(kMaxJobs, n - t0);
        PtrList pl{};
        for (int t = 0; t < cnt; t++) pl.p[t] = rr[t0 + t];
        k_rr_combine<<<grid_x(N, cnt), kTB, 0, st>>>(pl, vee + (size_t)t0 * 3 * N, pk, (long long)kpk * N, P->pr, N);
        BLB_COUNT_LAUNCH(1);
    }
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}
blb_status blb_launch_mask(const blb_params *P, const u64 *const *in, int n, int level, const uint8_t key[32],
                           u64 id0, u64 *masked, u64 *share, cudaStream_t st) {
    const int N = P->N;
    for (int t0 = 0; t0 < n; t0 += kMaxJobs) {
        const int cnt = (n - t0) < kMaxJobs ? (n - t0) : kMaxJobs;
        PtrList pl{};
        for (int t = 0; t < cnt; t++) pl.p[t] = in[t0 + t];
        k_drop_q0<<<grid_x(N, cnt, 2), kTB, 0, st>>>(pl, masked + (size_t)t0 * 2 * N, level + 1, N);
        BLB_COUNT_LAUNCH(1);
    }
    RowBatch rb{};
    rb.base = masked; rb.poly_stride = N; rb.n_polys = 2 * n; rb.limbs = 1; rb.limb0 = 0; rb.prime[0] = 0;
    BLB_TRY(launch_ntt(P, rb, true, st));
    k_mask<<<dim3((N / 4 + kTB - 1) / kTB, n), kTB, 0, st>>>(masked, share, P->pr, chacha_key_from_bytes(key), id0, N);
    BLB_COUNT_LAUNCH(1);
    BLB_COUNT(5, n);
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}
