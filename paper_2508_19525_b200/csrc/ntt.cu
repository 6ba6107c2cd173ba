#include <algorithm>
// ntt.cu -- limb-batched negacyclic NTT / INTT for sm_100a (row a1; C2).
//
// NTT(a)[k] = a(psi^{2 brv(k) + 1}) mod q: the in-place Cooley-Tukey network
// (natural order in, bit-reversed order out) with twiddles psi^{brv(m+i)};
// INTT = the Gentleman-Sande network with psi^{-brv(m+i)}, then N^{-1}.
//
// Design: the log N stages are split into two
// shared-memory passes of 2^S1 and 2^S2 points (N = 2^16: 256 x 256).  Pass 1
// transforms strided columns (elements mid*T + lo, T = N/2^S1) for 16
// consecutive lo per CTA, so every global access is a 128-byte coalesced row
// segment; pass 2 transforms 16 contiguous 2^S2-point blocks per CTA.  Each
// CTA keeps 4096 residues (32 KB) in shared memory across its S stages.
// Butterflies are Harvey-lazy with Shoup twiddles: values stay in [0, 4q)
// (forward) / [0, 2q) (inverse) and are made canonical in the last pass.
// N <= 2^12 runs in a single pass (one row per CTA).
#include "blb_internal.cuh"

namespace {

constexpr int kThreads = 256;

template <bool INV>
__global__ void __launch_bounds__(kThreads) ntt_pass(RowBatch rb, const u64 *__restrict__ tw_all, Primes pr, int logN,
                                                     int s0, int logM, int logT, int logC, int last) {
    extern __shared__ u64 sm[];
    const int M = 1 << logM, C = 1 << logC;
    const int N = 1 << logN;
    const int row = blockIdx.y;
    const int p = row / rb.limbs, l = row - p * rb.limbs;
    u64 *a = rb.base + (long long)p * rb.poly_stride + (long long)(rb.limb0 + l) * N;
    if (rb.skip_alpha) {
        const int dig = p % rb.skip_beta;
        if (l < rb.skip_kmax && l >= dig * rb.skip_alpha && l < (dig + 1) * rb.skip_alpha) return;
    }
    const int pi = rb.prime[l];
    const u64 q = pr.m[pi].q, q2 = 2 * q;
    const ulonglong2 *twp = reinterpret_cast<const ulonglong2 *>(tw_all + (size_t)pi * 4 * N + (INV ? 2 * N : 0));
    const int colg0 = blockIdx.x * C;
    const bool strided = logT > 0;
    const int TM = C * M;

    // load: smem index == linear index within the tile
    for (int idx = threadIdx.x; idx < TM; idx += kThreads) {
        int col, mid;
        if (strided) { mid = idx >> logC; col = idx & (C - 1); }
        else { col = idx >> logM; mid = idx & (M - 1); }
        const int colg = colg0 + col;
        const size_t addr = ((size_t)(colg >> logT) << (logM + logT)) + ((size_t)mid << logT) + (colg & ((1 << logT) - 1));
        sm[idx] = a[addr];
    }

    for (int rr = 0; rr < logM; rr++) {
        const int r = INV ? (logM - 1 - rr) : rr;
        const int logtl = logM - r - 1;
        const int tl = 1 << logtl;
        const int s = s0 + r;
        __syncthreads();
        for (int pidx = threadIdx.x; pidx < TM / 2; pidx += kThreads) {
            int col, qq;
            if (strided) { col = pidx & (C - 1); qq = pidx >> logC; }
            else { col = pidx >> (logM - 1); qq = pidx & ((M >> 1) - 1); }
            const int mid = ((qq >> logtl) << (logtl + 1)) + (qq & (tl - 1));
            const int h = (colg0 + col) >> logT;
            const int widx = (1 << s) + (h << r) + (qq >> logtl);
            const ulonglong2 tv = twp[widx];
            const u64 w = tv.x, wsh = tv.y;
            const int i0 = strided ? (mid * C + col) : (col * M + mid);
            const int i1 = i0 + (strided ? (tl << logC) : tl);
            u64 X = sm[i0], Y = sm[i1];
            if (!INV) {
                if (X >= q2) X -= q2;
                const u64 t = shoup_lazy(Y, w, wsh, q);
                sm[i0] = X + t;
                sm[i1] = X - t + q2;
            } else {
                u64 sum = X + Y;
                if (sum >= q2) sum -= q2;
                sm[i0] = sum;
                sm[i1] = shoup_lazy(X - Y + q2, w, wsh, q);
            }
        }
    }
    __syncthreads();
    const ModConst &mc = pr.m[pi];
    for (int idx = threadIdx.x; idx < TM; idx += kThreads) {
        int col, mid;
        if (strided) { mid = idx >> logC; col = idx & (C - 1); }
        else { col = idx >> logM; mid = idx & (M - 1); }
        const int colg = colg0 + col;
        const size_t addr = ((size_t)(colg >> logT) << (logM + logT)) + ((size_t)mid << logT) + (colg & ((1 << logT) - 1));
        u64 v = sm[idx];
        if (last) {
            if (!INV) {
                if (v >= q2) v -= q2;
                if (v >= q) v -= q;
            } else {
                v = shoup_lazy(v, mc.ninv, mc.ninv_sh, q);
                if (v >= q) v -= q;
            }
        }
        a[addr] = v;
    }
}

// ---------------------------------------------------------------------------
// N = 2^16 fast path: each pass is a 256-point sub-transform of 16 columns per
// CTA, but instead of one shared-memory round trip per stage every thread keeps
// 16 residues in registers and runs 4 radix-2 stages in registers ("round A":
// the 16 residues mid = tc + 16 m of its column, pairs 16*dist apart; "round B":
// mid = 16 tc + m, pairs dist apart), with two swizzled shared-memory exchanges
// per pass (A -> B, B -> A) so that global loads and stores both use the
// coalesced A mapping.  Twiddle index of stage s = s0 + r (generic formula):
// (1 << s) + (h << r) + mid / (2 t_l).
__device__ __forceinline__ int swz(int col, int mid) { return (col << 8) | (mid & 0xF0) | ((mid ^ (mid >> 4) ^ col) & 15); }

// Integer butterflies with the truncated-quotient Shoup product (shoup_lazy4, result in [0, 4q)):
// forward values stay in [0, 8q) (X is brought below 4q, X + t < 8q, X - t + 4q in (0, 8q)),
// inverse values in [0, 4q); 8q < 2^64 for every prime < 2^61.
// LZ forward (primes < 2^60, so 16q <= 2^64): X is corrected only on every other stage, by 8q:
// a stage adds < 4q to the bound, so inputs < 12q -> outputs < 16q -> (corrected X < 8q) -> < 12q.
// MODE: 0 = no correction, 1 = X >= 8q -> X - 8q, 2 = X >= 4q -> X - 4q.
template <bool INV, int MODE = 2>
__device__ __forceinline__ void bfly(u64 &X, u64 &Y, u64 w, u64 wsh, u64 q, u64 q4) {
    if (!INV) {
        if constexpr (MODE == 2) {
            if (X >= q4) X -= q4;
        } else if constexpr (MODE == 1) {
            if (X >= 2 * q4) X -= 2 * q4;
        }
        const u64 t = shoup_lazy4(Y, w, wsh, q);
        Y = X - t + q4;
        X = X + t;
    } else {
        u64 s = X + Y;
        if (s >= q4) s -= q4;
        const u64 d = X - Y + q4;
        X = s;
        Y = shoup_lazy4(d, w, wsh, q);
    }
}
// [0, 8q) -> [0, q)
__device__ __forceinline__ u64 canon8(u64 x, u64 q) {
    if (x >= 4 * q) x -= 4 * q;
    if (x >= 2 * q) x -= 2 * q;
    if (x >= q) x -= q;
    return x;
}
// [0, 16q) -> [0, q)
__device__ __forceinline__ u64 canon16(u64 x, u64 q) {
    if (x >= 8 * q) x -= 8 * q;
    return canon8(x, q);
}

// ---------------------------------------------------------------------------
// FP64 butterflies for the primes < 2^41 (4 of the 5 BERT chain primes).  The B200 FP64 pipe
// (64 DFMA/clk/SM) is separate from the fma-heavy pipe that the 64-bit integer multiplies of
// the Shoup butterfly saturate, and residues < 2^41 with their lazy growth stay exact integers
// in a double.  y * w mod q = (p - c q) + e with p = fl(y w), e = y w - p (exact, one fma),
// c = round(fl(y w) / q) (one fma against 1.5 * 2^52): |c - y w / q| < 5/8, so the remainder
// lies in (-5q/8, 5q/8) and every step is exact (twiddles are plain doubles: 8-byte loads).  Values are signed and unreduced: forward
// |x| grows by < q per stage (< 13 q after 16 stages), inverse sums double per stage and are
// re-centred between the two passes, so all inputs stay below 2^50.
// ---------------------------------------------------------------------------
constexpr double kTwo52 = 4503599627370496.0, kMagic = 6755399441055744.0;  // 2^52, 1.5 * 2^52
__device__ __forceinline__ double u2d(u64 x) {  // x < 2^52
    return __dsub_rn(__hiloint2double(0x43300000 | (int)(x >> 32), (int)(uint32_t)x), kTwo52);
}
#ifndef BLB_NTT_RND
#define BLB_NTT_RND 0
#endif
__device__ __forceinline__ double mulr(double y, double w, double q, double qinv) {
    const double p = __dmul_rn(y, w);
    const double e = __fma_rn(y, w, -p);
#if BLB_NTT_RND
    // round(p / q) as fl(p * qinv) + 1.5 2^52 - 1.5 2^52: three FP64 ops but no register copies of
    // the uniform qinv (DFMA cannot take a uniform-register B operand together with an immediate C)
    const double c = __dsub_rn(__dadd_rn(__dmul_rn(p, qinv), kMagic), kMagic);
#else
    const double c = __dsub_rn(__fma_rn(p, qinv, kMagic), kMagic);  // round(p / q): |c - y w / q| < 5/8
#endif
    return __dadd_rn(__fma_rn(-c, q, p), e);
}
__device__ __forceinline__ double centre(double x, double q, double qinv) {  // x - round(x / q) q
    const double c = __dsub_rn(__fma_rn(x, qinv, kMagic), kMagic);
    return __fma_rn(-c, q, x);
}
__device__ __forceinline__ u64 canon(double x, double q, double qinv) {  // x mod q in [0, q)
    double r = centre(x, q, qinv);
    if (r < 0.0) r = __dadd_rn(r, q);
    if (r >= q) r = __dsub_rn(r, q);
    return (u64)__double_as_longlong(__dadd_rn(r, kTwo52)) & 0x000FFFFFFFFFFFFFull;
}
template <bool INV>
__device__ __forceinline__ void bfly_f64(double &X, double &Y, double w, double q, double qinv) {
    if (!INV) {
        const double r = mulr(Y, w, q, qinv), x = X;
        X = __dadd_rn(x, r);
        Y = __dsub_rn(x, r);
    } else {
        const double s = __dadd_rn(X, Y), d = __dsub_rn(X, Y);
        X = s;
        Y = mulr(d, w, q, qinv);
    }
}

#ifndef BLB_NTT_MINB
#define BLB_NTT_MINB 3
#endif
// FP64 contiguous pass: the CTA's 16 x 255 twiddles of stages 8..15 are staged in shared memory by 8
// bulk copies at the start (twd_s[16 (2^r - 1) + (h - c0) 2^r + j] = twd[2^(8+r) + h 2^r + j]), so the
// rounds read them from shared memory instead of waiting on dependent L2 loads
constexpr int kTwsWords = 16 * 255;
template <bool INV, bool SMALL, int PRO>
__device__ __forceinline__ void ntt15_strided(u64 *sm, const RowBatch &rb, const u64 *__restrict__ tw_all,
                                              const double *__restrict__ twd_all, const Primes &pr, const NttFuse &fz,
                                              int p, int l);
template <bool INV, bool STRIDED, int PRO, int EPI, bool SMALL, bool LZ = false, int LOGN = 16>
__device__ __forceinline__ void ntt16_body(u64 *sm, const RowBatch &rb, const u64 *__restrict__ tw_all,
                                           const double *__restrict__ twd_all, const Primes &pr, int, int,
                                           const NttFuse &fz, int p, int l, double *tws = nullptr,
                                           uint64_t *twbar = nullptr) {
    if constexpr (LOGN == 15 && STRIDED) {  // N = 2^15: 128-point strided columns (ntt15_strided)
        ntt15_strided<INV, SMALL, PRO>(sm, rb, tw_all, twd_all, pr, fz, p, l);
        return;
    }
    constexpr int logN = LOGN, N = 1 << logN;
    // the strided pass runs stages [0, 8), the contiguous one [logN - 8, logN) (256-point blocks); the
    // last pass of a transform is the contiguous one forward and the strided one inverse (compile-time:
    // no dead epilogue selects)
    constexpr int s0 = STRIDED ? 0 : logN - 8;
    constexpr bool last = INV == STRIDED;
    u64 *a = rb.base + (long long)p * rb.poly_stride + (long long)(rb.limb0 + l) * N;
    const int pi = rb.prime[l];
    const u64 q = pr.m[pi].q, q4 = 4 * q;
    // interleaved (w, w') pairs: one 16-byte load per butterfly
    const ulonglong2 *twp = reinterpret_cast<const ulonglong2 *>(tw_all + (size_t)pi * 4 * N + (INV ? 2 * N : 0));
    const double *twd = twd_all + (size_t)pi * 2 * N + (INV ? N : 0);
    const int t = threadIdx.x;
    const int c0 = blockIdx.x * 16;  // first column of the tile (lo0 for STRIDED, h0 otherwise)
    // A mapping (coalesced global access)
    const int colA = STRIDED ? (t & 15) : (t >> 4);
    const int tcA = STRIDED ? (t >> 4) : (t & 15);
    // B mapping
    const int colB = t >> 4, tcB = t & 15;
    const int hA = STRIDED ? 0 : (c0 + colA);
    const int hB = STRIDED ? 0 : (c0 + colB);
    // (the integer kernel's 16-byte (w, w') pairs staged the same way need 96 KB per CTA: measured no faster)
    constexpr bool TWS = SMALL && !STRIDED;
    if constexpr (TWS) {  // stage the twiddles (bulk copies, completion on twbar), waited for before round 1
        if (t == 0) {
            const double *src = twd_all + (size_t)pi * 2 * N + (INV ? N : 0);
            mbar_expect_tx(twbar, kTwsWords * 8u);
#pragma unroll
            for (int r = 0; r < 8; r++)
                bulk_g2s(tws + 16 * ((1 << r) - 1), src + (1 << (s0 + r)) + (c0 << r), (16u << r) * 8u, twbar);
        }
    }
    // SMALL (q < 2^41): values are doubles; between the two passes they are stored as double bits
    using V = typename std::conditional<SMALL, double, u64>::type;
    const double qd = (double)q, qinv = 1.0 / qd;
    V v[16];
    auto from_u64 = [&](u64 x) -> V {
        if constexpr (SMALL) return u2d(x);
        else return x;
    };
    auto to_bits = [&](V x) -> u64 {
        if constexpr (SMALL) return (u64)__double_as_longlong(x);
        else return x;
    };
    auto from_bits = [&](u64 x) -> V {
        if constexpr (SMALL) return __longlong_as_double((long long)x);
        else return x;
    };
    if (PRO == 2) {
        const u64 *src = fz.srcp.p[p] + (long long)(rb.limb0 + l) * N;
#pragma unroll
        for (int m = 0; m < 16; m++) {
            const int mid = tcA + 16 * m;
            const size_t addr = STRIDED ? (((size_t)mid << 8) + c0 + colA) : (((size_t)(c0 + colA) << 8) + mid);
            v[m] = from_u64(src[addr]);
        }
    } else if (PRO == 3) {  // compact 5-byte signed coefficients -> residues mod the row's prime
        const unsigned char *cb = fz.coef + (long long)p * 5 * N;
        const ModConst &mt = pr.m[pi];
#pragma unroll
        for (int m = 0; m < 16; m++) {
            const int mid = tcA + 16 * m;
            const uint32_t kx = STRIDED ? (((uint32_t)mid << 8) + c0 + colA) : (((uint32_t)(c0 + colA) << 8) + mid);
            const unsigned long long ub =
                (unsigned long long)reinterpret_cast<const uint32_t *>(cb)[kx] | ((unsigned long long)cb[4 * N + kx] << 32);
            const long long c = (long long)(ub << 24) >> 24;
            u64 a = c < 0 ? (u64)(-c) : (u64)c;
            if (a >= mt.q) a = mod64(a, mt);
            v[m] = from_u64(c < 0 && a ? mt.q - a : a);
        }
    } else if (PRO == 1) {
        const u64 *src = fz.src + (long long)(p / fz.src_div) * fz.src_hi + (long long)(p % fz.src_div) * fz.src_lo;
        const ModConst &mt = pr.m[pi];
        const int dj = p % fz.src_div;
        if ((fz.red0 >> dj) & 1) {  // digit already below the target prime
#pragma unroll
            for (int m = 0; m < 16; m++) {
                const int mid = tcA + 16 * m;
                const size_t addr = STRIDED ? (((size_t)mid << 8) + c0 + colA) : (((size_t)(c0 + colA) << 8) + mid);
                v[m] = from_u64(src[addr]);
            }
        } else if ((fz.red1 >> dj) & 1) {  // below twice the target prime
#pragma unroll
            for (int m = 0; m < 16; m++) {
                const int mid = tcA + 16 * m;
                const size_t addr = STRIDED ? (((size_t)mid << 8) + c0 + colA) : (((size_t)(c0 + colA) << 8) + mid);
                const u64 x = src[addr];
                v[m] = from_u64(x >= mt.q ? x - mt.q : x);
            }
        } else {
#pragma unroll
            for (int m = 0; m < 16; m++) {
                const int mid = tcA + 16 * m;
                const size_t addr = STRIDED ? (((size_t)mid << 8) + c0 + colA) : (((size_t)(c0 + colA) << 8) + mid);
                v[m] = from_u64(mod64(src[addr], mt));
            }
        }
    } else {
#pragma unroll
        for (int m = 0; m < 16; m++) {
            const int mid = tcA + 16 * m;
            const size_t addr = STRIDED ? (((size_t)mid << 8) + c0 + colA) : (((size_t)(c0 + colA) << 8) + mid);
            v[m] = last ? from_bits(a[addr]) : from_u64(a[addr]);  // second pass: the first pass's format
        }
    }
    auto roundA = [&](int r) {
        const int dist = 8 >> r;
        const int s = s0 + r;
#pragma unroll
        for (int m = 0; m < 16; m++) {
            if (m & dist) continue;
            const int widx = (1 << s) + (hA << r) + (m >> (4 - r));
            if constexpr (TWS) {
                bfly_f64<INV>(v[m], v[m + dist], tws[16 * ((1 << r) - 1) + (colA << r) + (m >> (4 - r))], qd, qinv);
            } else if constexpr (SMALL) {
                bfly_f64<INV>(v[m], v[m + dist], twd[widx], qd, qinv);
            } else {
                const ulonglong2 tv = twp[widx];
                if (LZ && !INV) {
                    if (r & 1) bfly<INV, 1>(v[m], v[m + dist], tv.x, tv.y, q, q4);
                    else bfly<INV, 0>(v[m], v[m + dist], tv.x, tv.y, q, q4);
                } else {
                    bfly<INV>(v[m], v[m + dist], tv.x, tv.y, q, q4);
                }
            }
        }
    };
    auto roundB = [&](int r) {
        const int dist = 8 >> (r - 4);
        const int s = s0 + r;
#pragma unroll
        for (int m = 0; m < 16; m++) {
            if (m & dist) continue;
            const int widx = (1 << s) + (hB << r) + ((16 * tcB + m) >> (8 - r));
            if constexpr (TWS) {
                bfly_f64<INV>(v[m], v[m + dist], tws[16 * ((1 << r) - 1) + (colB << r) + ((16 * tcB + m) >> (8 - r))],
                              qd, qinv);
            } else if constexpr (SMALL) {
                bfly_f64<INV>(v[m], v[m + dist], twd[widx], qd, qinv);
            } else {
                const ulonglong2 tv = twp[widx];
                if (LZ && !INV) {
                    if (r & 1) bfly<INV, 1>(v[m], v[m + dist], tv.x, tv.y, q, q4);
                    else bfly<INV, 0>(v[m], v[m + dist], tv.x, tv.y, q, q4);
                } else {
                    bfly<INV>(v[m], v[m + dist], tv.x, tv.y, q, q4);
                }
            }
        }
    };
    if constexpr (TWS) mbar_wait(twbar, 0);
    if (!INV) {
#pragma unroll
        for (int r = 0; r < 4; r++) roundA(r);
    }
#pragma unroll
    for (int m = 0; m < 16; m++) sm[swz(colA, tcA + 16 * m)] = to_bits(v[m]);
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 16; m++) v[m] = from_bits(sm[swz(colB, 16 * tcB + m)]);
    if (!INV) {
#pragma unroll
        for (int r = 4; r < 8; r++) roundB(r);
    } else {
#pragma unroll
        for (int r = 7; r >= 4; r--) roundB(r);
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 16; m++) sm[swz(colB, 16 * tcB + m)] = to_bits(v[m]);
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 16; m++) v[m] = from_bits(sm[swz(colA, tcA + 16 * m)]);
    if (INV) {
#pragma unroll
        for (int r = 3; r >= 0; r--) roundA(r);
    }
    const ModConst &mc = pr.m[pi];
    if constexpr (EPI == 1) {  // ModDown combine (forward, contiguous last pass)
        const int tj = p >> 1, b = p & 1;
        const KsJob &J = fz.jobs.j[tj];
        const u64 *ui = fz.u + ((long long)p * fz.E + l) * N;
        u64 *out = J.out + ((long long)b * fz.k + l) * N;
        const u64 pv = fz.pinv.v[l], psh = fz.pinv.sh[l];
        // all 16 u_i loads are issued before the first store to out (which may alias as far as the
        // compiler knows): one exposed DRAM latency per thread instead of 16
        u64 uv[16];
#pragma unroll
        for (int m = 0; m < 16; m++) uv[m] = ui[(uint32_t)((c0 + colA) << 8) + tcA + 16 * m];
#pragma unroll
        for (int m = 0; m < 16; m++) {
            u64 x;
            if constexpr (SMALL) x = canon(v[m], qd, qinv);
            else x = LZ ? canon16(v[m], q) : canon8(v[m], q);
            const int mid = tcA + 16 * m;
            const uint32_t gx = (uint32_t)((c0 + colA) << 8) + mid;
            u64 r = shoup(uv[m] + q - x, pv, psh, q);
            if (J.add_mode == 1 && b == 0) {
                const uint32_t src = J.galois == 1 ? gx : galois_perm(gx, J.galois, logN);
                r = addmod(r, J.c0[(long long)l * N + src], q);
            } else if (J.add_mode == 2) {
                const u64 *c = b == 0 ? J.c0 : J.c1_add;
                r = addmod(r, c[(long long)l * N + gx], q);
            }
            if constexpr (SMALL) {
                if (J.out_f64) r = (u64)__double_as_longlong(u2d(r));
            }
            out[gx] = r;
        }
    } else if constexpr (EPI == 2) {  // blocked width-packed MAC layout (blb_matmul_coeffs_to_pts)
        const int e = fz.pk_e0 + p;
        const int o = fz.pk_ent_o[e];
        const int e_lo = fz.pk_ent_start[o], n_e = fz.pk_ent_start[o + 1] - e_lo;
        const int w = fz.pk_w[l];
        const uint32_t g0 = (uint32_t)(c0 + colA) << 8;  // the thread's 16 coefficients lie in one 512-tile
        unsigned char *tile = fz.pk_dst + (long long)(e_lo - fz.pk_ebase) * fz.pk_bpp + (long long)n_e * fz.pk_loff[l] +
                              ((long long)(g0 >> 9) * n_e + (e - e_lo)) * 512 * w;
#pragma unroll
        for (int m = 0; m < 16; m++) {
            u64 x;
            if constexpr (SMALL) x = canon(v[m], qd, qinv);
            else x = LZ ? canon16(v[m], q) : canon8(v[m], q);
            const uint32_t pos = (g0 + tcA + 16 * m) & 511;
            if (w == 5) {
                reinterpret_cast<uint32_t *>(tile)[pos] = (uint32_t)x;
                tile[2048 + pos] = (unsigned char)(x >> 32);
            } else {
                reinterpret_cast<u64 *>(tile)[pos] = x;
            }
        }
    } else {
#pragma unroll
        for (int m = 0; m < 16; m++) {
            u64 x;
            if constexpr (SMALL) {
                if (last) x = canon(INV ? mulr(v[m], (double)mc.ninv, qd, qinv) : v[m], qd, qinv);
                else x = to_bits(INV ? centre(v[m], qd, qinv) : v[m]);  // inverse sums re-centred for pass 2
            } else {
                x = v[m];
                if (last) {
                    if (!INV) {
                        x = LZ ? canon16(x, q) : canon8(x, q);
                    } else {
                        x = shoup_lazy(x, mc.ninv, mc.ninv_sh, q);
                        if (x >= q) x -= q;
                    }
                }
            }
            const int mid = tcA + 16 * m;
            const size_t addr = STRIDED ? (((size_t)mid << 8) + c0 + colA) : (((size_t)(c0 + colA) << 8) + mid);
            a[addr] = x;
        }
    }
}

// N = 2^15 = 128 x 256: the strided pass transforms 128-point columns (stages 0..6, element
// j = mid * 256 + lo) for 32 consecutive lo per CTA: round A (stages 0..3) on mid = tc + 8 m, round B
// (stages 4..6) on mid = 16 tc + m, shared-memory tile [mid][32 columns] with the column index XORed
// by 2 ((mid >> 4) & 7) (conflict-free for both mappings); the contiguous pass is ntt16_body's with
// s0 = 7.  PRO = 1 (forward): the ModUp / ModDown prologue of ntt16_body (row read from fz.src and
// reduced mod the row's prime).
template <bool INV, bool SMALL, int PRO>
__device__ __forceinline__ void ntt15_strided(u64 *sm, const RowBatch &rb, const u64 *__restrict__ tw_all,
                                              const double *__restrict__ twd_all, const Primes &pr, const NttFuse &fz,
                                              int p, int l) {
    constexpr int N = 1 << 15;
    u64 *a = rb.base + (long long)p * rb.poly_stride + (long long)(rb.limb0 + l) * N;
    const int pi = rb.prime[l];
    const u64 q = pr.m[pi].q, q4 = 4 * q;
    const ulonglong2 *twp = reinterpret_cast<const ulonglong2 *>(tw_all + (size_t)pi * 4 * N + (INV ? 2 * N : 0));
    const double *twd = twd_all + (size_t)pi * 2 * N + (INV ? N : 0);
    const int t = threadIdx.x;
    const int c0 = blockIdx.x * 32;
    const int colA = t & 31, tcA = t >> 5;  // A: mid = tcA + 8 m (a warp: 32 consecutive lo)
    const int colB = t >> 3, tcB = t & 7;   // B: mid = 16 tcB + m
    auto ph = [](int mid, int col) { return mid * 32 + (col ^ (((mid >> 4) & 7) << 1)); };
    using V = typename std::conditional<SMALL, double, u64>::type;
    const double qd = (double)q, qinv = 1.0 / qd;
    V v[16];
    auto to_bits = [&](V x) -> u64 {
        if constexpr (SMALL) return (u64)__double_as_longlong(x);
        else return x;
    };
    auto from_bits = [&](u64 x) -> V {
        if constexpr (SMALL) return __longlong_as_double((long long)x);
        else return x;
    };
    auto bf = [&](int m, int dist, int widx) {
        if constexpr (SMALL) {
            bfly_f64<INV>(v[m], v[m + dist], twd[widx], qd, qinv);
        } else {
            const ulonglong2 tv = twp[widx];
            bfly<INV>(v[m], v[m + dist], tv.x, tv.y, q, q4);
        }
    };
    auto roundA = [&](int s) {  // stages 0..3: mid distance 64 >> s = 8 (8 >> s)
        const int dist = 8 >> s;
#pragma unroll
        for (int m = 0; m < 16; m++)
            if (!(m & dist)) bf(m, dist, (1 << s) + (m >> (4 - s)));
    };
    auto roundB = [&](int s) {  // stages 4..6: mid distance 4 >> (s - 4)
        const int dist = 4 >> (s - 4);
#pragma unroll
        for (int m = 0; m < 16; m++)
            if (!(m & dist)) bf(m, dist, (1 << s) + ((16 * tcB + m) >> (7 - s)));
    };
    auto from_u64 = [&](u64 x) -> V {
        if constexpr (SMALL) return u2d(x);
        else return x;
    };
    if constexpr (PRO == 1) {
        const u64 *src = fz.src + (long long)(p / fz.src_div) * fz.src_hi + (long long)(p % fz.src_div) * fz.src_lo;
        const ModConst &mt = pr.m[pi];
        const int dj = p % fz.src_div;
        const int mode = ((fz.red0 >> dj) & 1) ? 0 : (((fz.red1 >> dj) & 1) ? 1 : 2);
#pragma unroll
        for (int m = 0; m < 16; m++) {
            u64 x = src[((tcA + 8 * m) << 8) + c0 + colA];
            if (mode == 1) x = x >= mt.q ? x - mt.q : x;
            else if (mode == 2) x = mod64(x, mt);
            v[m] = from_u64(x);
        }
    } else {
        // inverse: the second pass reads the first (contiguous) pass's format (FP64 rows: double bits)
#pragma unroll
        for (int m = 0; m < 16; m++) {
            const u64 x = a[((tcA + 8 * m) << 8) + c0 + colA];
            if constexpr (SMALL) v[m] = INV ? from_bits(x) : u2d(x);
            else v[m] = x;
        }
    }
    if (!INV) {
#pragma unroll
        for (int s = 0; s < 4; s++) roundA(s);
    }
#pragma unroll
    for (int m = 0; m < 16; m++) sm[ph(tcA + 8 * m, colA)] = to_bits(v[m]);
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 16; m++) v[m] = from_bits(sm[ph(16 * tcB + m, colB)]);
    if (!INV) {
#pragma unroll
        for (int s = 4; s < 7; s++) roundB(s);
    } else {
#pragma unroll
        for (int s = 6; s >= 4; s--) roundB(s);
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 16; m++) sm[ph(16 * tcB + m, colB)] = to_bits(v[m]);
    __syncthreads();
#pragma unroll
    for (int m = 0; m < 16; m++) v[m] = from_bits(sm[ph(tcA + 8 * m, colA)]);
    const ModConst &mc = pr.m[pi];
    if (INV) {
#pragma unroll
        for (int s = 3; s >= 0; s--) roundA(s);
    }
#pragma unroll
    for (int m = 0; m < 16; m++) {
        u64 x;
        if constexpr (SMALL) {
            x = INV ? canon(mulr(v[m], (double)mc.ninv, qd, qinv), qd, qinv) : to_bits(v[m]);
        } else {
            x = v[m];
            if (INV) {
                x = shoup_lazy(x, mc.ninv, mc.ninv_sh, q);
                if (x >= q) x -= q;
            }
        }
        a[((tcA + 8 * m) << 8) + c0 + colA] = x;
    }
}

__device__ __forceinline__ bool ntt16_row(const RowBatch &rb, int &p, int &l) {
    const int row = blockIdx.y;
    if (rb.nsel > 0) {
        p = row / rb.nsel;
        l = rb.sel[row - p * rb.nsel];
    } else {
        p = row / rb.limbs;
        l = row - p * rb.limbs;
    }
    if (rb.skip_alpha) {
        const int dig = p % rb.skip_beta;
        if (l < rb.skip_kmax && l >= dig * rb.skip_alpha && l < (dig + 1) * rb.skip_alpha) return false;
    }
    return true;
}
// a skipped (own-digit) row of a ModUp batch: copy this CTA's 16 columns of the NTT-form input row
template <int LOGN = 16>
__device__ __forceinline__ void copy_own_tile(const RowBatch &rb, const NttFuse &fz, int p, int l) {
    if (!fz.copy_own) return;
    constexpr int N = 1 << LOGN;
    const u64 *src = fz.srcp.p[p / fz.src_div] + (long long)l * N;
    u64 *a = rb.base + (long long)p * rb.poly_stride + (long long)(rb.limb0 + l) * N;
    const int t = threadIdx.x;
    // this CTA's strided tile: 16 columns x 256 (2^16) or 32 columns x 128 (2^15) of j = mid * 256 + lo
    constexpr int C = LOGN == 16 ? 16 : 32;
    const int c0 = blockIdx.x * C;
#pragma unroll
    for (int m = 0; m < 16; m++) {
        const size_t addr = ((size_t)(t / C + (256 / C) * m) << 8) + c0 + (t % C);
        a[addr] = src[addr];
    }
}
#ifndef BLB_NTT_F64_MINB
#define BLB_NTT_F64_MINB 3
#endif
// integer (Shoup) kernel for the primes >= 2^41, FP64 kernel for the others; a launch covers
// rows of one kind (launch_ntt splits a mixed batch with RowBatch::sel)
template <bool INV, bool STRIDED, int PRO = 0, int EPI = 0, bool LZ = false, int LOGN = 16>
__global__ void __launch_bounds__(256, BLB_NTT_MINB) ntt16_int(RowBatch rb, const u64 *__restrict__ tw_all,
                                                                const double *__restrict__ twd, Primes pr, int s0,
                                                                int last, const NttFuse fz) {
    __shared__ u64 sm[16 * 256];
    int p, l;
    if (!ntt16_row(rb, p, l)) {
        if (PRO == 1 && STRIDED) copy_own_tile<LOGN>(rb, fz, p, l);
        return;
    }
    ntt16_body<INV, STRIDED, PRO, EPI, false, LZ, LOGN>(sm, rb, tw_all, twd, pr, s0, last, fz, p, l);
}
// dynamic shared memory: 4096 residues, then (contiguous pass) the staged twiddles and their mbarrier
template <bool STRIDED>
constexpr size_t ntt16_f64_smem() { return STRIDED ? 4096 * 8 : 4096 * 8 + kTwsWords * 8 + 16; }
template <bool INV, bool STRIDED, int PRO = 0, int EPI = 0, int LOGN = 16>
__global__ void __launch_bounds__(256, BLB_NTT_F64_MINB) ntt16_f64(RowBatch rb, const u64 *__restrict__ tw_all,
                                                                    const double *__restrict__ twd, Primes pr, int s0,
                                                                    int last, const NttFuse fz) {
    extern __shared__ __align__(16) u64 dsm[];
    int p, l;
    if (!ntt16_row(rb, p, l)) {
        if (PRO == 1 && STRIDED) copy_own_tile<LOGN>(rb, fz, p, l);
        return;
    }
    if constexpr (STRIDED) {
        ntt16_body<INV, STRIDED, PRO, EPI, true, false, LOGN>(dsm, rb, tw_all, twd, pr, s0, last, fz, p, l);
    } else {
        double *tws = reinterpret_cast<double *>(dsm + 4096);
        uint64_t *bar = reinterpret_cast<uint64_t *>(dsm + 4096 + kTwsWords);
        if (threadIdx.x == 0) {
            mbar_init(bar, 1);
            mbar_fence_init();
        }
        __syncthreads();
        ntt16_body<INV, STRIDED, PRO, EPI, true, false, LOGN>(dsm, rb, tw_all, twd, pr, s0, last, fz, p, l, tws, bar);
    }
}

template <bool INV, bool STRIDED, int PRO = 0, int EPI = 0, int LOGN = 16>
static void launch_f64(const blb_params *P, const RowBatch &r, dim3 g, cudaStream_t st, int s0, int last,
                       const NttFuse &fz) {
    constexpr size_t smem = ntt16_f64_smem<STRIDED>();
    if (smem > 48 * 1024) blb_smem_optin(ntt16_f64<INV, STRIDED, PRO, EPI, LOGN>, smem);
    ntt16_f64<INV, STRIDED, PRO, EPI, LOGN><<<g, 256, smem, st>>>(r, P->d_tw, P->d_twd, P->pr, s0, last, fz);
}
// integer-kernel launch: forward rows whose primes are all < 2^60 take the LZ butterflies
static bool rb_below60(const blb_params *P, const RowBatch &r) {
    const int nl = r.nsel ? r.nsel : r.limbs;
    for (int i = 0; i < nl; i++)
        if (P->mod[r.prime[r.nsel ? r.sel[i] : i]] >= (1ull << 60)) return false;
    return true;
}
template <bool INV, bool STRIDED, int PRO = 0, int EPI = 0, int LOGN = 16>
static void launch_int(const blb_params *P, const RowBatch &r, dim3 g, cudaStream_t st, int s0, int last,
                       const NttFuse &fz) {
    if constexpr (LOGN != 16) {  // N = 2^15: no LZ (pass 1 has 7 stages; the LZ bound needs whole rounds)
        ntt16_int<INV, STRIDED, PRO, EPI, false, LOGN><<<g, 256, 0, st>>>(r, P->d_tw, P->d_twd, P->pr, s0, last, fz);
        return;
    }
#ifndef BLB_NTT_LZ
#define BLB_NTT_LZ 1
#endif
    if constexpr (!INV) {
        if (BLB_NTT_LZ && rb_below60(P, r)) {
            ntt16_int<INV, STRIDED, PRO, EPI, true><<<g, 256, 0, st>>>(r, P->d_tw, P->d_twd, P->pr, s0, last, fz);
            return;
        }
    }
    ntt16_int<INV, STRIDED, PRO, EPI, false><<<g, 256, 0, st>>>(r, P->d_tw, P->d_twd, P->pr, s0, last, fz);
}

// split the limbs of a batch by prime size: out[0] = FP64 rows (q < 2^41), out[1] = integer rows
static int split_rows(const blb_params *P, const RowBatch &rb, RowBatch out[2]) {
    RowBatch f = rb, g = rb;
    f.nsel = 0; g.nsel = 0;
    for (int l = 0; l < rb.limbs; l++) {
        if (P->mod[rb.prime[l]] < (1ull << 41)) f.sel[f.nsel++] = l;
        else g.sel[g.nsel++] = l;
    }
    int n = 0;
    if (f.nsel) { if (f.nsel == rb.limbs) f.nsel = 0; out[n++] = f; }
    if (g.nsel) { if (g.nsel == rb.limbs) g.nsel = 0; out[n++] = g; }
    return n;
}
// rows of a batch on primes >= 2^41 (the integer NTT kernel): counter [6]
static long long rb_int_rows(const blb_params *P, const RowBatch &r) {
    int n = 0;
    const int nl = r.nsel ? r.nsel : r.limbs;
    for (int i = 0; i < nl; i++) n += P->mod[r.prime[r.nsel ? r.sel[i] : i]] >= (1ull << 41);
    return (long long)n * r.n_polys;
}
static inline bool rb_small(const blb_params *P, const RowBatch &r) {
    return P->mod[r.prime[r.nsel ? r.sel[0] : 0]] < (1ull << 41);
}
static inline int rb_rows(const RowBatch &r) { return r.n_polys * (r.nsel ? r.nsel : r.limbs); }

// Two-stream NTT: the integer-kernel rows of a mixed batch run on the auxiliary
// stream while the FP64-kernel rows run on the caller's stream -- the two kernels load different
// pipes (fma-heavy vs FP64), so CTAs of both can share an SM.  fork() before the launches, join()
// after; the stream of part h is part_stream(h).
struct NttStreams {
    const blb_params *P;
    cudaStream_t st;
    bool two;
    NttStreams(const blb_params *P_, cudaStream_t st_, int np2) : P(P_), st(st_), two(np2 == 2 && P_->aux) {
        if (two) {
            cudaEvent_t e = P->ev[P->ev_next];
            P->ev_next = (P->ev_next + 1) % 64;
            cudaEventRecord(e, st);
            cudaStreamWaitEvent(P->aux, e, 0);
        }
    }
    cudaStream_t part_stream(int h) const { return two && h == 1 ? P->aux : st; }
    void join() const {
        if (!two) return;
        cudaEvent_t e = P->ev[P->ev_next];
        P->ev_next = (P->ev_next + 1) % 64;
        cudaEventRecord(e, P->aux);
        cudaStreamWaitEvent(st, e, 0);
    }
};

}  // namespace

blb_status launch_ntt(const blb_params *P, const RowBatch &rb, bool inverse, cudaStream_t st) {
    const cudaStream_t st0 = st;
    const int rows = rb.n_polys * rb.limbs;
    if (rows == 0) return BLB_OK;
    const int logN = P->logN;
    if (rows > 65535) {
        // split by polys to respect gridDim.y
        int per = 65535 / rb.limbs;
        for (int p0 = 0; p0 < rb.n_polys; p0 += per) {
            RowBatch sub = rb;
            sub.base = rb.base + (long long)p0 * rb.poly_stride;
            sub.n_polys = (rb.n_polys - p0) < per ? (rb.n_polys - p0) : per;
            BLB_TRY(launch_ntt(P, sub, inverse, st));
        }
        return BLB_OK;
    }
    BLB_COUNT(2, rows);
    BLB_COUNT(6, rb_int_rows(P, rb));
    cudaEvent_t t0 = blb_timing_begin(st);
    const double alg = (double)rows * 2.0 * 8.0 * (double)(1 << logN);
    if (logN <= 12) {
        const size_t smem = (size_t)8 << logN;
        dim3 grid(1, rows);
        if (!inverse) ntt_pass<false><<<grid, kThreads, smem, st>>>(rb, P->d_tw, P->pr, logN, 0, logN, 0, 0, 1);
        else ntt_pass<true><<<grid, kThreads, smem, st>>>(rb, P->d_tw, P->pr, logN, 0, logN, 0, 0, 1);
        BLB_COUNT_LAUNCH(1);
        blb_timing_end(1, t0, st, alg);
        BLB_CHECK_LAUNCH();
        return BLB_OK;
    }
    if (logN == 15) {  // 128-point strided columns (32 per CTA) + 256-point contiguous blocks (16 per CTA)
        const NttFuse fz{};
        RowBatch parts[2];
        const int np2 = split_rows(P, rb, parts);
        const NttStreams ss(P, st0, np2);
        for (int h = 0; h < np2; h++) {
            const cudaStream_t st = ss.part_stream(h);
            const RowBatch &r = parts[h];
            const dim3 g(8, rb_rows(r));
            if (rb_small(P, r)) {
                if (!inverse) {
                    launch_f64<false, true, 0, 0, 15>(P, r, g, st, 0, 0, fz);
                    launch_f64<false, false, 0, 0, 15>(P, r, g, st, 7, 1, fz);
                } else {
                    launch_f64<true, false, 0, 0, 15>(P, r, g, st, 7, 0, fz);
                    launch_f64<true, true, 0, 0, 15>(P, r, g, st, 0, 1, fz);
                }
            } else {
                if (!inverse) {
                    launch_int<false, true, 0, 0, 15>(P, r, g, st, 0, 0, fz);
                    launch_int<false, false, 0, 0, 15>(P, r, g, st, 7, 1, fz);
                } else {
                    launch_int<true, false, 0, 0, 15>(P, r, g, st, 7, 0, fz);
                    launch_int<true, true, 0, 0, 15>(P, r, g, st, 0, 1, fz);
                }
            }
        }
        ss.join();
        BLB_COUNT_LAUNCH(2 * np2);
        blb_timing_end(1, t0, st0, alg);
        BLB_CHECK_LAUNCH();
        return BLB_OK;
    }
    if (logN == 16) {
        const NttFuse fz{};
        RowBatch parts[2];
        const int np2 = split_rows(P, rb, parts);
        const NttStreams ss(P, st0, np2);
        for (int h = 0; h < np2; h++) {
            const cudaStream_t st = ss.part_stream(h);
            const RowBatch &r = parts[h];
            const dim3 g(16, rb_rows(r));
            if (rb_small(P, r)) {
                if (!inverse) {
                    launch_f64<false, true>(P, r, g, st, 0, 0, fz);
                    launch_f64<false, false>(P, r, g, st, 8, 1, fz);
                } else {
                    launch_f64<true, false>(P, r, g, st, 8, 0, fz);
                    launch_f64<true, true>(P, r, g, st, 0, 1, fz);
                }
            } else {
                if (!inverse) {
                    launch_int<false, true>(P, r, g, st, 0, 0, fz);
                    launch_int<false, false>(P, r, g, st, 8, 1, fz);
                } else {
                    launch_int<true, false>(P, r, g, st, 8, 0, fz);
                    launch_int<true, true>(P, r, g, st, 0, 1, fz);
                }
            }
        }
        ss.join();
        BLB_COUNT_LAUNCH(2 * np2);
        blb_timing_end(1, t0, st0, alg);
        BLB_CHECK_LAUNCH();
        return BLB_OK;
    }
    const int S1 = logN / 2, S2 = logN - S1;
    const int logTile = 12;  // 4096 residues per CTA
    const size_t smem = (size_t)8 << logTile;
    // pass over the strided columns: stages [0, S1), M = 2^S1, T = 2^S2
    const int logC1 = logTile - S1;
    dim3 g1((1 << S2) >> logC1, rows);
    // pass over contiguous blocks: stages [S1, logN), M = 2^S2, T = 1
    const int logC2 = logTile - S2;
    dim3 g2((1 << S1) >> logC2, rows);
    if (!inverse) {
        ntt_pass<false><<<g1, kThreads, smem, st>>>(rb, P->d_tw, P->pr, logN, 0, S1, S2, logC1, 0);
        ntt_pass<false><<<g2, kThreads, smem, st>>>(rb, P->d_tw, P->pr, logN, S1, S2, 0, logC2, 1);
    } else {
        ntt_pass<true><<<g2, kThreads, smem, st>>>(rb, P->d_tw, P->pr, logN, S1, S2, 0, logC2, 0);
        ntt_pass<true><<<g1, kThreads, smem, st>>>(rb, P->d_tw, P->pr, logN, 0, S1, S2, logC1, 1);
    }
    BLB_COUNT_LAUNCH(2);
    blb_timing_end(1, t0, st, alg);
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}

// Forward N = 2^16 NTT with a fused prologue (pro = 1) and / or ModDown epilogue (epi = 1).
// the fused launch pair of one part (prime kind) of a batch at N = 2^LOGN (15 or 16)
template <int LOGN>
static void fused_pair(const blb_params *P, const RowBatch &r, cudaStream_t st, bool inverse, const NttFuse &fz,
                       const NttFuse &fzp) {
    constexpr int S2 = LOGN - 8;                      // first stage of the contiguous pass
    const dim3 g(LOGN == 16 ? 16 : 8, rb_rows(r));
    const bool small = rb_small(P, r);
    if (inverse) {  // pro = 2: first (contiguous) pass loads from the pointer table
        if (small) {
            launch_f64<true, false, 2, 0, LOGN>(P, r, g, st, S2, 0, fz);
            launch_f64<true, true, 0, 0, LOGN>(P, r, g, st, 0, 1, fz);
        } else {
            launch_int<true, false, 2, 0, LOGN>(P, r, g, st, S2, 0, fz);
            launch_int<true, true, 0, 0, LOGN>(P, r, g, st, 0, 1, fz);
        }
        return;
    }
    if constexpr (LOGN == 16) {
        if (fz.pro == 3) {  // compact coefficients -> packed plaintexts (blb_matmul_coeffs_to_pts)
            if (small) {
                launch_f64<false, true, 3, 0>(P, r, g, st, 0, 0, fz);
                launch_f64<false, false, 0, 2>(P, r, g, st, 8, 1, fz);
            } else {
                launch_int<false, true, 3, 0>(P, r, g, st, 0, 0, fz);
                launch_int<false, false, 0, 2>(P, r, g, st, 8, 1, fz);
            }
            return;
        }
    }
    if (small) {
        if (fz.pro == 1) launch_f64<false, true, 1, 0, LOGN>(P, r, g, st, 0, 0, fzp);
        else launch_f64<false, true, 0, 0, LOGN>(P, r, g, st, 0, 0, fz);
        if (fz.epi == 1) launch_f64<false, false, 0, 1, LOGN>(P, r, g, st, S2, 1, fz);
        else launch_f64<false, false, 0, 0, LOGN>(P, r, g, st, S2, 1, fz);
    } else {
        if (fz.pro == 1) launch_int<false, true, 1, 0, LOGN>(P, r, g, st, 0, 0, fzp);
        else launch_int<false, true, 0, 0, LOGN>(P, r, g, st, 0, 0, fz);
        if (fz.epi == 1) launch_int<false, false, 0, 1, LOGN>(P, r, g, st, S2, 1, fz);
        else launch_int<false, false, 0, 0, LOGN>(P, r, g, st, S2, 1, fz);
    }
}

blb_status launch_ntt_fused(const blb_params *P, const RowBatch &rb, bool inverse, const NttFuse &fz,
                            cudaStream_t st0) {
    const cudaStream_t st = st0;
    const int rows = rb.n_polys * rb.limbs;
    if (rows == 0) return BLB_OK;
    if ((P->logN != 16 && P->logN != 15) || rows > 65535 || (inverse && (fz.pro != 2 || fz.epi)) ||
        (!inverse && fz.pro == 2) || ((fz.pro == 3 || fz.epi == 2) && (fz.pro != 3 || fz.epi != 2 || P->logN != 16))) {
        blb_set_error("launch_ntt_fused: N = 2^15 / 2^16 forward batches (or inverse with pro = 2) only");
        return BLB_E_INVALID_ARG;
    }
    BLB_COUNT(2, rows);
    BLB_COUNT(6, rb_int_rows(P, rb));
    cudaEvent_t t0 = blb_timing_begin(st);
    RowBatch parts[2];
    const int np2 = split_rows(P, rb, parts);
    const NttStreams ss(P, st0, np2);
    for (int h = 0; h < np2; h++) {
        const RowBatch &rp = parts[h];
        const cudaStream_t st = ss.part_stream(h);
        NttFuse fzp = fz;  // this part's reduction masks (pro = 1)
        fzp.red0 = fzp.red1 = 0;
        if (!inverse && fz.pro == 1 && fz.src_nq > 0 && fz.src_nq <= 8) {
            u64 minq = ~0ull;
            const int nl = rp.nsel ? rp.nsel : rp.limbs;
            for (int i = 0; i < nl; i++) minq = std::min<u64>(minq, P->mod[rp.prime[rp.nsel ? rp.sel[i] : i]]);
            for (int j = 0; j < fz.src_nq; j++) {
                if (fz.src_q[j] == 0) continue;
                if (fz.src_q[j] <= minq) fzp.red0 |= 1u << j;
                else if (fz.src_q[j] / 2 < minq) fzp.red1 |= 1u << j;  // q_j <= 2 minq - 1 (odd primes)
            }
        }
        if (P->logN == 16) fused_pair<16>(P, rp, st, inverse, fz, fzp);
        else fused_pair<15>(P, rp, st, inverse, fz, fzp);
    }
    ss.join();
    BLB_COUNT_LAUNCH(2 * np2);
    blb_timing_end(1, t0, st0, (double)rows * 16.0 * (double)(1 << P->logN));
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}
