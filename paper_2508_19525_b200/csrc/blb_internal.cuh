// blb_internal.cuh -- internal types and device arithmetic of the B200 BLB
// CKKS library (product code; shares nothing with oracle/).
//
// 64-bit RNS residues, primes < 2^61.  Device modular arithmetic:
//   * Shoup multiplication for constant multiplicands (twiddles, P^{-1}, ...):
//     w' = floor(w * 2^64 / q),  x*w mod q in [0, 2q) for any 64-bit x.
//   * 128-bit lazy accumulation of products of canonical residues, reduced
//     once by reduce128 (hi < 2^63 required, i.e. <= 2^(127 - 2*61) = 32
//     products of 61-bit residues; the MAC uses <= 96 products of < 2^60
//     operands for q_0).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <vector>
#include <string>
#include "../../include/blb.h"

typedef uint64_t u64;
typedef unsigned __int128 u128;

#define BLB_MAXP BLB_MAX_PRIMES

// ---------------------------------------------------------------------------
// per-prime constants (passed by value to kernels)
// ---------------------------------------------------------------------------
struct ModConst {
    u64 q;
    u64 ninv, ninv_sh;   // N^{-1} mod q and its Shoup companion
    u64 r64, r64_sh;     // 2^64 mod q and Shoup
    u64 mu;              // floor((2^64 - 1) / q)  (Barrett for 64-bit values)
};
struct Primes {
    ModConst m[BLB_MAXP];
};

__host__ __device__ __forceinline__ u64 umulhi64(u64 a, u64 b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (u64)(((u128)a * b) >> 64);
#endif
}

// x mod q for any 64-bit x (Barrett, floor error <= 2)
__device__ __forceinline__ u64 mod64(u64 x, const ModConst &c) {
    u64 qh = umulhi64(x, c.mu);
    u64 r = x - qh * c.q;
    if (r >= c.q) r -= c.q;
    if (r >= c.q) r -= c.q;
    return r;
}
// Shoup: x * w mod q in [0, 2q)
__device__ __forceinline__ u64 shoup_lazy(u64 x, u64 w, u64 wsh, u64 q) {
    return x * w - umulhi64(x, wsh) * q;
}
__device__ __forceinline__ u64 shoup(u64 x, u64 w, u64 wsh, u64 q) {
    u64 r = shoup_lazy(x, w, wsh, q);
    return r >= q ? r - q : r;
}
// Shoup with a truncated quotient: Q' = xh sh + hi32(xh sl) + hi32(xl sh) drops the xl sl partial
// product and the carries of the two cross terms (x s / 2^64 - Q' < 3, so Q' >= floor(x s / 2^64) - 2):
// x * w mod q in [0, 4q) for any 64-bit x, with one 32x32->64 and two 32x32->hi32 multiplies
// instead of the four wide multiplies of __umul64hi (the fma pipe is what bounds the 64-bit NTT).
__device__ __forceinline__ u64 shoup_lazy4(u64 x, u64 w, u64 wsh, u64 q) {
    const uint32_t xl = (uint32_t)x, xh = (uint32_t)(x >> 32);
    const uint32_t sl = (uint32_t)wsh, sh = (uint32_t)(wsh >> 32);
    const u64 Q = (u64)xh * sh + (u64)__umulhi(xh, sl) + (u64)__umulhi(xl, sh);
    return x * w - Q * q;
}
// (hi * 2^64 + lo) mod q, hi < 2^64
__device__ __forceinline__ u64 reduce128(u64 hi, u64 lo, const ModConst &c) {
    u64 h = mod64(hi, c);
    u64 t = shoup(h, c.r64, c.r64_sh, c.q);
    u64 l = mod64(lo, c);
    u64 r = t + l;
    return r >= c.q ? r - c.q : r;
}
// a*b mod q, a, b < 2^64
__device__ __forceinline__ u64 mulmod(u64 a, u64 b, const ModConst &c) {
    return reduce128(umulhi64(a, b), a * b, c);
}
__device__ __forceinline__ u64 addmod(u64 a, u64 b, u64 q) {
    u64 r = a + b;
    return r >= q ? r - q : r;
}
__device__ __forceinline__ u64 submod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }

// 128-bit accumulator
struct Acc128 {
    u64 lo, hi;
    __device__ __forceinline__ void zero() { lo = 0; hi = 0; }
    __device__ __forceinline__ void mac(u64 a, u64 b) {
        u64 pl = a * b, ph = umulhi64(a, b);
        u64 nl = lo + pl;
        hi += ph + (nl < lo ? 1 : 0);
        lo = nl;
    }
    __device__ __forceinline__ u64 reduce(const ModConst &c) const { return reduce128(hi, lo, c); }
    // keep the sum exact beyond 2^127 / q^2 products: replace it by its residue
    __device__ __forceinline__ void fold(const ModConst &c) {
        lo = reduce(c);
        hi = 0;
    }
};

// Accumulator for products of residues < 2^41 (the 40-bit chain primes), with
// 32-bit partial products: a = a1 2^32 + a0, a1 < 2^9.  lo (96 bits, 3 words)
// += a0 b0; mid (64 bits) += a1 b0 + a0 b1 (< 2^42 each); hi (32 bits) += a1 b1
// (< 2^18 each): 6 IMAD-class instructions per product instead of the ~13 of
// a 64x64->128 multiply + 128-bit add.  Valid for < 2^14 products.
struct Acc41 {
    uint32_t l0, l1, l2, hi;
    u64 mid;
    __device__ __forceinline__ void zero() { l0 = l1 = l2 = hi = 0; mid = 0; }
    __device__ __forceinline__ void mac(u64 a, u64 b) {
        const uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32), b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
        asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
            "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
            "addc.u32 %2, %2, 0;"
            : "+r"(l0), "+r"(l1), "+r"(l2)
            : "r"(a0), "r"(b0));
        mid += (u64)a1 * b0 + (u64)a0 * b1;
        hi += a1 * b1;
    }
    __device__ __forceinline__ u64 reduce(const ModConst &c) const {
        // total = (l2:l1:l0) + mid * 2^32 + hi * 2^64
        const u64 lo = ((u64)l1 << 32) | l0;
        const u64 m_lo = mid << 32, m_hi = mid >> 32;
        const u64 s = lo + m_lo;
        const u64 H = (u64)l2 + hi + m_hi + (s < lo ? 1 : 0);
        return reduce128(H, s, c);
    }
    __device__ __forceinline__ void fold(const ModConst &) {}  // exact for < 2^14 products
};

// Accumulator for up to 7 products of residues < 2^60 (the 60-bit chain / special primes) with
// 32-bit partial products: a = a1 2^32 + a0 (a1 < 2^28).  lo (96 bits) += a0 b0; mid (64 bits) +=
// a1 b0 + a0 b1 (< 2^60 each, 14 terms < 2^64); hi (64 bits) += a1 b1: 6 IMAD-class instructions per
// product instead of the ~11 of Acc128's 64x64->128 multiply + 128-bit add.
struct Acc60 {
    uint32_t l0, l1, l2;
    u64 mid, hi;
    __device__ __forceinline__ void zero() { l0 = l1 = l2 = 0; mid = 0; hi = 0; }
    __device__ __forceinline__ void mac(u64 a, u64 b) {
        const uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32), b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
        asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
            "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
            "addc.u32 %2, %2, 0;"
            : "+r"(l0), "+r"(l1), "+r"(l2)
            : "r"(a0), "r"(b0));
        mid += (u64)a1 * b0 + (u64)a0 * b1;
        hi += (u64)a1 * b1;
    }
    __device__ __forceinline__ u64 reduce(const ModConst &c) const {
        // total = (l2:l1:l0) + mid 2^32 + hi 2^64
        const u64 lo = ((u64)l1 << 32) | l0;
        const u64 m_lo = mid << 32, m_hi = mid >> 32;
        const u64 s = lo + m_lo;
        const u64 H = (u64)l2 + hi + m_hi + (s < lo ? 1 : 0);
        return reduce128(H, s, c);
    }
};

// Carry-save accumulator for many products of residues < 2^60 (the weight MAC's q0 limb): a = a1 2^32 +
// a0 (a1 < 2^28); L (96 bits, carry chain) += a0 b0, M (96 bits) += a0 b1 + a1 b0, H (64 bits) += a1 b1
// (< 2^56): 10 instructions per product, no compare / select.  total = L + M 2^32 + H 2^64 < P 2^120
// stays below 2^128 for P < 256 products (fold every 128).
struct Acc60W {
    uint32_t l0, l1, l2, m0, m1, m2;
    u64 h;
    __device__ __forceinline__ void zero() { l0 = l1 = l2 = m0 = m1 = m2 = 0; h = 0; }
    __device__ __forceinline__ void mac(u64 a, u64 b) {
        const uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32), b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
        asm("mad.lo.cc.u32 %0, %6, %8, %0;\n\t"
            "madc.hi.cc.u32 %1, %6, %8, %1;\n\t"
            "addc.u32 %2, %2, 0;\n\t"
            "mad.lo.cc.u32 %3, %6, %9, %3;\n\t"
            "madc.hi.cc.u32 %4, %6, %9, %4;\n\t"
            "addc.u32 %5, %5, 0;\n\t"
            "mad.lo.cc.u32 %3, %7, %8, %3;\n\t"
            "madc.hi.cc.u32 %4, %7, %8, %4;\n\t"
            "addc.u32 %5, %5, 0;"
            : "+r"(l0), "+r"(l1), "+r"(l2), "+r"(m0), "+r"(m1), "+r"(m2)
            : "r"(a0), "r"(a1), "r"(b0), "r"(b1));
        h += (u64)a1 * b1;
    }
    __device__ __forceinline__ u64 reduce(const ModConst &c) const {
        const u64 lo = ((u64)l1 << 32) | l0;
        const u64 s = lo + ((u64)m0 << 32);
        const u64 H = (u64)l2 + (((u64)m2 << 32) | m1) + h + (s < lo ? 1 : 0);
        return reduce128(H, s, c);
    }
    __device__ __forceinline__ void fold(const ModConst &c) {
        const u64 r = reduce(c);
        zero();
        l0 = (uint32_t)r;
        l1 = (uint32_t)(r >> 32);
    }
};

// Exact FP64-pipe accumulator for products of residues < 2^41 (offloads the fma-heavy pipe that
// the integer accumulators saturate; the B200 FP64 pipe runs 64 DFMA/clk/SM beside it):
// a b = p + e with p = fl(a b) and e = fma(a, b, -p) exact; c = round(p / q) by one fma against
// 1.5 * 2^52 (|error| < 2^-11, so p - c q lies in (-q, q) and is exact); sums of the remainders
// and of the e's stay exact integers below 2^51 for < 2^10 products.
struct AccF64 {
    double r;  // sum of the exact remainders (p - c q) + e
    __device__ __forceinline__ void zero() { r = 0.0; }
    __device__ __forceinline__ static double u2d(u64 x) {  // x < 2^52
        return __dsub_rn(__hiloint2double(0x43300000 | (int)(x >> 32), (int)(uint32_t)x), 4503599627370496.0);
    }
    __device__ __forceinline__ void mac(u64 a, u64 b, double qd, double qinv) {
        const double A = u2d(a), B = u2d(b);
        const double p = __dmul_rn(A, B);
        const double e = __fma_rn(A, B, -p);
        const double c = __dsub_rn(__fma_rn(p, qinv, 6755399441055744.0), 6755399441055744.0);
        r = __dadd_rn(r, __dadd_rn(__fma_rn(-c, qd, p), e));  // |p - c q + e| < q + 2^30: exact
    }
    __device__ __forceinline__ void fold(double qd, double qinv) {  // back to |r| <= q/2
        const double c = __dsub_rn(__fma_rn(r, qinv, 6755399441055744.0), 6755399441055744.0);
        r = __fma_rn(-c, qd, r);
    }
    __device__ __forceinline__ u64 reduce(double qd, double qinv) const {
        const double c = __dsub_rn(__fma_rn(r, qinv, 6755399441055744.0), 6755399441055744.0);
        double v = __fma_rn(-c, qd, r);
        if (v < 0.0) v = __dadd_rn(v, qd);
        if (v >= qd) v = __dsub_rn(v, qd);
        return (u64)__double_as_longlong(__dadd_rn(v, 4503599627370496.0)) & 0x000FFFFFFFFFFFFFull;
    }
};

// Grid-split FP64 accumulator for residues < 2^41: no reduction per product.  The running sum
// s = M + H 2^40 (M = 1.5 * 2^92) stays in [2^92, 2^93), where the double grid is 2^40: each product
// is added with one fma, s' = fl(s + A B), and its rounding error A B + s - s' (|.| <= 2^39, exact:
// s - s' is an exact multiple of 2^40) is recovered with a second fma and summed in l.  Per product:
// 2 fma + 2 add on the FP64 pipe, nothing else (AccF64: 6 FP64 ops).  Exact for <= 512 products of
// residues < 2^41 between folds (s < M + 2^91 = 2^93, l < 2^48); the value is (s - M) + l.
struct AccG {
    double s, l;
    static constexpr double kM = 0x1.8p+92;  // 1.5 * 2^92
    __device__ __forceinline__ void zero() { s = kM; l = 0.0; }
    __device__ __forceinline__ void mac(u64 a, u64 b) { macd(AccF64::u2d(a), AccF64::u2d(b)); }
    __device__ __forceinline__ void macd(double A, double B) {  // A, B: integers < 2^41
        const double sn = __fma_rn(A, B, s);
        l = __dadd_rn(l, __fma_rn(A, B, __dsub_rn(s, sn)));
        s = sn;
    }
    // (s - M) + l mod q as a double with |value| < q + 2^49 (exact)
    __device__ __forceinline__ double rem(double qd, double qinv) const {
        const double magic = 6755399441055744.0;
        const double Hd = __dmul_rn(__dsub_rn(s, kM), 0x1p-40);  // H < 2^51, exact
        const double Hm = __fma_rn(-__dsub_rn(__fma_rn(Hd, qinv, magic), magic), qd, Hd);  // |Hm| <= q/2 + 1
        const double two40 = 1099511627776.0;
        const double c40 = __fma_rn(-__dsub_rn(__fma_rn(two40, qinv, magic), magic), qd, two40);  // 2^40 mod q, centred
        const double p = __dmul_rn(Hm, c40);
        const double e = __fma_rn(Hm, c40, -p);
        const double c = __dsub_rn(__fma_rn(p, qinv, magic), magic);
        return __dadd_rn(__dadd_rn(__fma_rn(-c, qd, p), e), l);
    }
    // back to s = M and |l| <= q/2 + 1: rem() keeps the old l unreduced, so l is re-centred here
    // (|rem| < q + 2^49 < 2^53: c = round(l / q) by one fma against 1.5 * 2^52 and l - c q by one
    // exact fma), which keeps every period's bound l < 2^48 + q for any number of folds
    __device__ __forceinline__ void fold(double qd, double qinv) {
        const double r = rem(qd, qinv);
        const double c = __dsub_rn(__fma_rn(r, qinv, 6755399441055744.0), 6755399441055744.0);
        l = __fma_rn(-c, qd, r);
        s = kM;
    }
    __device__ __forceinline__ u64 reduce(double qd, double qinv) const {
        AccF64 f;
        f.r = rem(qd, qinv);
        return f.reduce(qd, qinv);
    }
};

// accumulator helpers with one call signature (Acc41 / Acc128 ignore the FP64 constants)
__device__ __forceinline__ void accm(Acc41 &a, u64 x, u64 y, double, double) { a.mac(x, y); }
__device__ __forceinline__ void accm(Acc128 &a, u64 x, u64 y, double, double) { a.mac(x, y); }
__device__ __forceinline__ void accm(Acc60 &a, u64 x, u64 y, double, double) { a.mac(x, y); }
__device__ __forceinline__ u64 accr(const Acc60 &a, const ModConst &mc, double, double) { return a.reduce(mc); }
__device__ __forceinline__ void accm(AccF64 &a, u64 x, u64 y, double qd, double qinv) { a.mac(x, y, qd, qinv); }
__device__ __forceinline__ u64 accr(const Acc41 &a, const ModConst &mc, double, double) { return a.reduce(mc); }
__device__ __forceinline__ u64 accr(const Acc128 &a, const ModConst &mc, double, double) { return a.reduce(mc); }
__device__ __forceinline__ u64 accr(const AccF64 &a, const ModConst &, double qd, double qinv) { return a.reduce(qd, qinv); }
__device__ __forceinline__ void accf(Acc41 &, const ModConst &, double, double) {}  // exact for < 2^14 products
__device__ __forceinline__ void accf(Acc128 &a, const ModConst &mc, double, double) { a.fold(mc); }
__device__ __forceinline__ void accf(AccF64 &a, const ModConst &, double qd, double qinv) { a.fold(qd, qinv); }
__device__ __forceinline__ void accm(AccG &a, u64 x, u64 y, double, double) { a.mac(x, y); }
__device__ __forceinline__ u64 accr(const AccG &a, const ModConst &, double qd, double qinv) { return a.reduce(qd, qinv); }
__device__ __forceinline__ void accf(AccG &a, const ModConst &, double qd, double qinv) { a.fold(qd, qinv); }

// ---------------------------------------------------------------------------
// mbarrier + bulk-copy (TMA engine, cp.async.bulk) helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// the same on a precomputed shared-window address (no generic-to-shared conversion in a hot loop)
__device__ __forceinline__ void mbar_arrive_sa(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_sa(unsigned bar, unsigned phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
// generic-proxy reads of a ring slot (the consumers, ordered by the empty mbarrier) before the
// async-proxy (cp.async.bulk) writes that refill it
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// the same with an L2 cache policy (createpolicy): streamed-once data (the weight plaintexts) marked
// evict_first so it does not push the re-read operands (the baby-step rotations R) out of L2
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void *dst, const void *src, unsigned bytes, uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// Opt a kernel in to > 48 KB of dynamic shared memory on the CURRENT device, once per (kernel,
// device): the attribute is per device context, so a process driving several GPUs sets it on each.
bool blb_smem_optin_needed(const void *kernel, size_t bytes);  // api.cu: registry keyed by (kernel, device)
template <class Kern>
inline void blb_smem_optin(Kern kernel, size_t bytes) {
    if (blb_smem_optin_needed((const void *)kernel, bytes))
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// NTT-domain automorphism index: out[k] = in[perm(k)],
// perm(k) = brv(((g * (2 brv(k) + 1)) mod 2N - 1) / 2)
__device__ __forceinline__ uint32_t galois_perm(uint32_t k, uint32_t g, int logN) {
    uint32_t e = 2u * (__brev(k) >> (32 - logN)) + 1u;
    uint32_t e2 = (uint32_t)(((u64)g * e) & ((2ull << logN) - 1));
    return __brev((e2 - 1u) >> 1) >> (32 - logN);
}

// ---------------------------------------------------------------------------
// host-side objects
// ---------------------------------------------------------------------------
struct BconvTable;  // fwd

struct blb_params {
    int logN, N, K, np, dnum, alpha, device;
    int num_sms = 148;
    // auxiliary stream: the integer-kernel (60-bit prime) rows of a mixed N = 2^16 NTT batch run on it
    // beside the FP64-kernel rows on the caller's stream (ntt.cu)
    cudaStream_t aux = nullptr;
    cudaEvent_t ev[64] = {};
    mutable int ev_next = 0;
    u64 mod[BLB_MAXP];
    u64 psi[BLB_MAXP];
    Primes pr;                    // by-value copy for kernel args
    u64 *d_tw = nullptr;          // [K+np][2][N][2]: (fwd, fwd Shoup), (inv, inv Shoup) pairs, bit-reversed order
    double *d_twd = nullptr;      // [K+np][2][N] twiddles as doubles (fwd, inv) for the primes < 2^41 (FP64 NTT)
    double *d_zeta = nullptr;     // [N][4]: zeta^{brv(i)} as (re_hi, re_lo, im_hi, im_lo)
    int32_t *d_slot_pos = nullptr; // [N/2]: NTT-domain position k of slot j (brv(k) = (5^j - 1)/2)
    // FastBConv tables, see bconv_* in kernels.cu
    u64 *d_bconv = nullptr;
    std::vector<size_t> bconv_off;   // offset of table (level, digit) / moddown(level)
    u64 P_mod_q[BLB_MAXP];           // P mod q_i
    u64 Pinv[BLB_MAXP], Pinv_sh[BLB_MAXP];  // P^{-1} mod q_i
};

struct blb_keys {
    const blb_params *params;
    std::vector<uint32_t> galois;       // parallel arrays
    std::vector<u64 *> data;            // device [beta_top][2][K+np][N]
};

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
void blb_set_error(const char *fmt, ...);
extern unsigned long long g_blb_counters[8];
#define BLB_COUNT_LAUNCH(n) (__atomic_fetch_add(&g_blb_counters[0], (unsigned long long)(n), __ATOMIC_RELAXED))
#define BLB_COUNT(i, n) (__atomic_fetch_add(&g_blb_counters[i], (unsigned long long)(n), __ATOMIC_RELAXED))

// live timing of tracked kernels (api.cu): returns a recorded start event or nullptr
cudaEvent_t blb_timing_begin(cudaStream_t st);
void blb_timing_end(int category, cudaEvent_t start, cudaStream_t st, double alg_bytes);

#define BLB_CUDA_TRY(expr)                                                                        \
    do {                                                                                          \
        cudaError_t _e = (expr);                                                                  \
        if (_e != cudaSuccess) {                                                                  \
            blb_set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(_e), __FILE__, __LINE__, \
                          cudaGetErrorString(_e));                                                \
            return BLB_E_CUDA;                                                                    \
        }                                                                                         \
    } while (0)
#define BLB_CHECK_LAUNCH() BLB_CUDA_TRY(cudaGetLastError())
#define BLB_TRY(expr)                     \
    do {                                  \
        blb_status _s = (expr);           \
        if (_s != BLB_OK) return _s;      \
    } while (0)

// ---------------------------------------------------------------------------
// internal launchers (kernels.cu / ntt.cu / encode.cu)
// ---------------------------------------------------------------------------
// A batch of NTT rows: row r = p * limbs + l is at base + p * poly_stride + (limb0 + l) * N,
// modulus index prime[l].
struct RowBatch {
    u64 *base;
    long long poly_stride;  // in u64 elements
    int n_polys, limbs, limb0;
    int prime[BLB_MAXP];
    // optional: skip rows whose limb l lies in digit (p % skip_beta) of size
    // skip_alpha among the first skip_kmax limbs (ModUp: a digit's own limbs
    // are copied, not recomputed)
    int skip_alpha = 0, skip_beta = 1, skip_kmax = 0;
    // optional limb selection (N = 2^16 kernels): nsel > 0 -> rows = n_polys * nsel, row -> limb sel[row % nsel]
    int nsel = 0;
    int sel[BLB_MAXP];
};
blb_status launch_ntt(const blb_params *P, const RowBatch &rb, bool inverse, cudaStream_t st);

// FastBConv / ModUp / ModDown helpers
// ModUp of n polynomials (c1_ntt[t]: [k][N], NTT, host array of device
// pointers, n <= kMaxJobs) -> ext [n][beta][E][N] (contiguous, NTT), using
// coef_scratch [n][k][N].
constexpr int kMaxJobs = 128;
// independent rotations (each with its own ModUp) are key-switched in batches of this many jobs
// (measured per layer: 128 best; 32 -> 76.8 ms, 16 -> 78.3, 8 -> 82.3, 4 -> 91.1 at the time,
// profiles/r1_indep_batch.log: smaller batches are launch-bound)
constexpr int kIndepBatch = kMaxJobs;
blb_status launch_modup(const blb_params *P, int level, const u64 *const *c1_ntt, int n, u64 *ext,
                        u64 *coef_scratch, cudaStream_t st);
inline int blb_beta(const blb_params *P, int level) { return (level + 1 + P->alpha - 1) / P->alpha; }
inline int blb_beta_top(const blb_params *P) { return (P->K + P->alpha - 1) / P->alpha; }
inline size_t bconv_modup_off(const blb_params *P, int level, int digit) {
    return P->bconv_off[(size_t)level * blb_beta_top(P) + digit];
}
inline size_t bconv_moddown_off(const blb_params *P, int level) {
    return P->bconv_off[(size_t)P->K * blb_beta_top(P) + level];
}
struct KsJob {
    const u64 *ext;   // [beta][E][N]
    const u64 *key;   // [beta_top][2][K+np][N]
    const u64 *c0;    // [k][N] input c0 (rotation: sigma_g(c0) is added), nullable (relin: add as is)
    u64 *out;         // [2][k][N]
    uint32_t galois;  // 1 = identity
    uint32_t galois_inv;  // g^{-1} mod 2N (filled by the key-switch launcher)
    int add_mode;     // 0 = none, 1 = add sigma_g(c0) to out0 (rotation), 2 = add c0 / c1 pair (relin)
    // 1: limbs whose prime is < 2^41 are written as the bits of the residue as a double (the MACs'
    // rotation buffers -- the weight MAC's baby steps R, the ct-ct stage-1 / step-3 rotations: their
    // FP64 accumulators then read them without a conversion)
    int out_f64;
    const u64 *c1_add;
};
blb_status launch_keyswitch(const blb_params *P, int level, const KsJob *jobs, int n_jobs, u64 *u_scratch,
                            u64 *conv_scratch, cudaStream_t st);
struct KsJobs {
    KsJob j[kMaxJobs];
};
struct PinvTab {
    u64 v[BLB_MAXP], sh[BLB_MAXP];
};
// Fused prologue / epilogue of the N = 2^16 NTT (ntt.cu):
//   pro = 1: the first pass loads row (p, l) from src + (p / src_div) * src_hi + (p % src_div) * src_lo
//            and reduces it mod the row's modulus (FastBConv of a single-prime digit / P limb);
//   epi = 1: the last (forward) pass finishes ModDown: out = (u_i - v) * P^{-1} (+ sigma_g(c0) / (c0, c1))
//            written to jobs.j[p / 2].out (rows p = 2 t + b, limb i), u = [jobs][2][E][N].
struct PtrTab {
    const u64 *p[kMaxJobs];
};
// pro = 2 (inverse, contiguous first pass): row (p, l) is loaded from srcp.p[p] + l * N (ModUp: the
//          ciphertexts' c1 rows straight into the coefficient scratch, no gather copy);
// copy_own (with pro = 1, alpha = 1): the rows a digit owns (skipped by the transform) are copied from
//          srcp.p[p / src_div] + l * N by the first pass (ModUp: the digit's own residues, NTT form).
struct NttFuse {
    int pro = 0, epi = 0, copy_own = 0;
    PtrTab srcp;
    const u64 *src = nullptr;
    long long src_hi = 0, src_lo = 0;
    int src_div = 1;
    // pro = 1, host side: the modulus of source digit j (row p reads digit p % src_div), 0 = unknown.
    // launch_ntt_fused turns them into per-launch bit masks over j: red0 = already below every target
    // prime of the launch (no reduction), red1 = below twice it (one conditional subtraction).
    int src_nq = 0;
    u64 src_q[8] = {};
    uint32_t red0 = 0, red1 = 0;
    const u64 *u = nullptr;
    int E = 0, k = 0;
    PinvTab pinv;
    KsJobs jobs;
    // pro = 3 (blb_matmul_coeffs_to_pts): row (p, l) is plaintext p's compact 5-byte coefficients
    //          (coef + p 5N: N low words, N high bytes) reduced mod the row's prime;
    // epi = 2: the last (forward) pass writes plaintext p (plan entry pk_e0 + p) limb l straight into the
    //          blocked width-packed MAC layout (k_block_pts's addressing)
    const unsigned char *coef = nullptr;
    unsigned char *pk_dst = nullptr;
    const int *pk_ent_o = nullptr, *pk_ent_start = nullptr;
    int pk_e0 = 0, pk_ebase = 0;
    long long pk_bpp = 0;
    long long pk_loff[BLB_MAXP] = {};
    int pk_w[BLB_MAXP] = {};
};
// double hoisting: rotations kept in Q_l u P written to jobs[t].out ([2][E][N]);
// ModDown of n contiguous extended ciphertexts u [n][2][E][N] -> out [n][2][k][N]
blb_status launch_keyswitch_ext(const blb_params *P, int level, const KsJob *jobs, int n, cudaStream_t st);
blb_status launch_moddown(const blb_params *P, int level, u64 *u, int n, u64 *out, u64 *conv, cudaStream_t st);
blb_status launch_moddown(const blb_params *P, int level, u64 *u, int n, u64 *const *outs, u64 *conv,
                          cudaStream_t st);
// f64: limbs with q < 2^41 written as double bits (the ct-ct mask MACs' rotation buffers, KsJob::out_f64)
blb_status launch_lift_ext(const blb_params *P, int level, const u64 *in, u64 *out, cudaStream_t st, bool f64 = false);
// ModDown fused with rescale (reading C17): u [n][2][level+1+np][N] (its q_level and P limbs are
// INTT'd in place) -> round(X / (q_level P)) as [2][level][N] NTT ciphertexts; conv scratch
// kMaxJobs x [2][level][N]
blb_status launch_moddown_rescale(const blb_params *P, int level, u64 *u, int n, u64 *const *outs, u64 *conv,
                                  cudaStream_t st);
blb_status launch_moddown_rescale(const blb_params *P, int level, u64 *u, int n, u64 *out, u64 *conv,
                                  cudaStream_t st);
blb_status launch_ntt_fused(const blb_params *P, const RowBatch &rb, bool inverse, const NttFuse &fz,
                            cudaStream_t st);
size_t keyswitch_scratch_elems(const blb_params *P, int level, int n_jobs);  // u + conv, in u64

blb_status launch_rescale(const blb_params *P, const u64 *in, int level, int n_polys, u64 *out, u64 *scratch,
                          cudaStream_t st);
// np_ext > 0: also write residues mod p_0..p_{np_ext-1} after the q limbs (extended-basis plaintexts)
blb_status launch_encode(const blb_params *P, const double *slots, int n_pts, double scale, int level, u64 *out,
                         double *dd_scratch, int *d_flag, cudaStream_t st, int np_ext = 0);
size_t encode_scratch_doubles(const blb_params *P, int n_pts);
blb_status launch_encode_coef5(const blb_params *P, const double *slots, int n_pts, double scale, unsigned char *coef,
                               double *buf, int *d_flag, cudaStream_t st);
blb_status launch_coef5_to_rns(const blb_params *P, const unsigned char *coef, int n_pts, int level, u64 *out,
                               cudaStream_t st);

// MAC: acc[o] = sum_{e in [ent_start[o0+o], ent_start[o0+o+1])} pt[ent_pt[e] or e - e_base] (.) R[ent_r[e]]
// (pt entries [k][N], R entries [2][k][N], acc [n_o][2][k][N]; 128-bit lazy accumulation)
// kq >= 0: the first kq limbs are q_0..q_{kq-1} and limbs kq.. are p_0.. (extended basis)
blb_status launch_mac(const blb_params *P, const u64 *pt, const u64 *R, u64 *acc, const int *ent_r, const int *ent_pt,
                      const int *ent_start, int o0, int e_base, int n_o, int n_entries, int k, cudaStream_t st,
                      int kq = -1, int jg = 1);

// ChaCha / sampling
enum { TAG_SECRET = 1, TAG_KEY_A = 2, TAG_KEY_E = 3, TAG_ENC_A = 4, TAG_ENC_E = 5, TAG_MASK = 6,
       TAG_RR_V = 7, TAG_RR_E0 = 8, TAG_RR_E1 = 9 };  // 7-9: S13 re-randomisation draws (reading C22)
struct ChachaKey {
    uint32_t k[8];
};
ChachaKey chacha_key_from_bytes(const uint8_t seed[32]);
