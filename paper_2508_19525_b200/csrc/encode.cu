// encode.cu -- CKKS encode / decode on sm_100a (Eq. eq:ckks_encode; C3).
//
// Encode(z) = round(Delta * pi^{-1}(z)).  pi evaluates m(X) at the roots
// zeta^{5^j} (slot j) and their conjugates; pi^{-1} is therefore the inverse
// negacyclic transform with psi -> zeta = e^{i pi / N}: place z_j at the
// "NTT-domain" position k with 2 brv(k) + 1 == 5^j (mod 2N) and its conjugate
// at N - 1 - k, run the Gentleman-Sande network with zeta^{-brv(m+i)}
// twiddles and divide by N.  All of it runs in double-double (~106-bit)
// complex arithmetic so that the final rounding is correct (reading C3): a
// plain double transform would mis-round ~1e5 coefficients per BERT layer.
// Decode runs the Cooley-Tukey network (zeta^{brv(m+i)}) on the centred lift.
// The transforms are radix-2 stage kernels over global memory: encode is the
// offline weight precompute (row a0), timed separately from the hot path.
#include "blb_internal.cuh"

namespace {
constexpr int kTB = 256;

struct dd {
    double hi, lo;
};
__device__ __forceinline__ dd two_sum(double a, double b) {
    const double s = a + b;
    const double bb = s - a;
    return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
    const double s = a + b;
    return {s, b - (s - a)};
}
__device__ __forceinline__ dd dd_add(dd x, dd y) {
    dd s = two_sum(x.hi, y.hi);
    const dd t = two_sum(x.lo, y.lo);
    s.lo += t.hi;
    s = quick_two_sum(s.hi, s.lo);
    s.lo += t.lo;
    return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_neg(dd x) { return {-x.hi, -x.lo}; }
__device__ __forceinline__ dd dd_sub(dd x, dd y) { return dd_add(x, dd_neg(y)); }
__device__ __forceinline__ dd dd_mul(dd x, dd y) {
    const double p = x.hi * y.hi;
    double e = fma(x.hi, y.hi, -p);
    e += x.hi * y.lo + x.lo * y.hi;
    return quick_two_sum(p, e);
}
__device__ __forceinline__ dd dd_mul_d(dd x, double y) {
    const double p = x.hi * y;
    double e = fma(x.hi, y, -p);
    e += x.lo * y;
    return quick_two_sum(p, e);
}
struct cdd {
    dd re, im;
};
__device__ __forceinline__ cdd cmul(cdd a, cdd b) {
    return {dd_sub(dd_mul(a.re, b.re), dd_mul(a.im, b.im)), dd_add(dd_mul(a.re, b.im), dd_mul(a.im, b.re))};
}
__device__ __forceinline__ cdd cadd(cdd a, cdd b) { return {dd_add(a.re, b.re), dd_add(a.im, b.im)}; }
__device__ __forceinline__ cdd csub(cdd a, cdd b) { return {dd_sub(a.re, b.re), dd_sub(a.im, b.im)}; }
__device__ __forceinline__ cdd cld(const double *p) { return {{p[0], p[1]}, {p[2], p[3]}}; }
__device__ __forceinline__ void cst(double *p, cdd v) {
    p[0] = v.re.hi; p[1] = v.re.lo; p[2] = v.im.hi; p[3] = v.im.lo;
}

// buf[p][pos] = (z, 0), buf[p][N-1-pos] = (z, 0)
__global__ void k_scatter(const double *slots, const int32_t *slot_pos, double *buf, int n_pts, int N) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int p = blockIdx.y;
    const int n = N / 2;
    if (j >= n) return;
    const double z = slots[(long long)p * n + j];
    const int pos = slot_pos[j];
    double *b = buf + (long long)p * N * 4;
    cst(b + 4ll * pos, {{z, 0.0}, {0.0, 0.0}});
    cst(b + 4ll * (N - 1 - pos), {{z, 0.0}, {0.0, 0.0}});
}

// one Gentleman-Sande stage (inverse=1) or Cooley-Tukey stage (inverse=0), m blocks of 2t
__global__ void k_stage(double *buf, const double *zeta, int m, int logN, int inverse) {
    const int N = 1 << logN;
    const int bidx = blockIdx.x * blockDim.x + threadIdx.x;
    const int p = blockIdx.y;
    if (bidx >= N / 2) return;
    const int t = N / (2 * m);
    const int i = bidx / t, jj = bidx - i * t;
    const int j = 2 * i * t + jj;
    double *b = buf + (long long)p * N * 4;
    cdd X = cld(b + 4ll * j), Y = cld(b + 4ll * (j + t));
    cdd W = cld(zeta + 4ll * (m + i));
    if (inverse) {
        W.im = dd_neg(W.im);  // zeta^{-brv(m+i)} = conj(zeta^{brv(m+i)})
        cst(b + 4ll * j, cadd(X, Y));
        cst(b + 4ll * (j + t), cmul(csub(X, Y), W));
    } else {
        const cdd V = cmul(Y, W);
        cst(b + 4ll * j, cadd(X, V));
        cst(b + 4ll * (j + t), csub(X, V));
    }
}

// N = 2^16 encode: the 16 Gentleman-Sande stages in two shared-memory passes instead of 16 global
// passes (the stage kernel above reads and writes the whole 32-byte-per-element buffer per stage).
// Pass A: stages t = 1 .. 128 (pairs inside 256-element blocks); pass B: t = 256 .. N/2 (pairs inside
// the stride-256 columns).  A CTA holds 2048 elements (64 KB); every butterfly is the stage kernel's
// (same double-double operations in the same order), so the results are identical.
constexpr int kEncElems = 2048;
__device__ __forceinline__ void gs_bfly(double *sm, int a, int b, const double *zeta, int widx) {
    cdd X = cld(sm + 4 * a), Y = cld(sm + 4 * b);
    cdd W = cld(zeta + 4ll * widx);
    W.im = dd_neg(W.im);
    cst(sm + 4 * a, cadd(X, Y));
    cst(sm + 4 * b, cmul(csub(X, Y), W));
}
__global__ void __launch_bounds__(kTB) k_enc16_A(double *buf, const double *zeta) {
    extern __shared__ double esm[];
    constexpr int N = 1 << 16;
    double *b = buf + (long long)blockIdx.y * N * 4 + (long long)blockIdx.x * kEncElems * 4;
    for (int i = threadIdx.x; i < kEncElems * 4; i += kTB) esm[i] = b[i];
    __syncthreads();
    const int e0 = blockIdx.x * kEncElems;
    for (int t = 1; t <= 128; t <<= 1) {
        const int m = N / (2 * t);
        for (int bf = threadIdx.x; bf < kEncElems / 2; bf += kTB) {
            const int jl = (bf / t) * 2 * t + (bf % t);
            gs_bfly(esm, jl, jl + t, zeta, m + (e0 + jl) / (2 * t));
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < kEncElems * 4; i += kTB) b[i] = esm[i];
}
// pass B: the CTA's 8 columns lo0 .. lo0 + 7 (element j = mid * 256 + lo), smem [mid][8][4]
__global__ void __launch_bounds__(kTB) k_enc16_B(double *buf, const double *zeta) {
    extern __shared__ double esm[];
    constexpr int N = 1 << 16, C = kEncElems / 256;
    double *b = buf + (long long)blockIdx.y * N * 4;
    const int lo0 = blockIdx.x * C;
    for (int i = threadIdx.x; i < kEncElems * 4; i += kTB) {
        const int mid = i / (C * 4), r = i % (C * 4);
        esm[i] = b[((long long)mid * 256 + lo0) * 4 + r];
    }
    __syncthreads();
    for (int tp = 1; tp <= 128; tp <<= 1) {       // t = 256 tp
        const int m = N / (2 * 256 * tp);
        for (int bf = threadIdx.x; bf < kEncElems / 2; bf += kTB) {
            const int c = bf % C, q = bf / C;       // q < 128: butterfly within the column
            const int mid = (q / tp) * 2 * tp + (q % tp);
            gs_bfly(esm, mid * C + c, (mid + tp) * C + c, zeta, m + mid / (2 * tp));
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < kEncElems * 4; i += kTB) {
        const int mid = i / (C * 4), r = i % (C * 4);
        b[((long long)mid * 256 + lo0) * 4 + r] = esm[i];
    }
}

// coefficient k = round_half_even(Re(buf[k]) * scale / N) (false: |.| >= 2^52, flag set)
__device__ __forceinline__ bool enc_round(const double *b, double scale, int logN, int *flag, long long &c) {
    dd v = {b[0], b[1]};
    v = dd_mul_d(v, scale);
    v = {ldexp(v.hi, -logN), ldexp(v.lo, -logN)};  // exact division by N
    if (!(fabs(v.hi) < 4503599627370496.0)) {     // 2^52
        atomicExch(flag, 1);
        return false;
    }
    double r = rint(v.hi);
    const double d = (v.hi - r) + v.lo;  // v.hi - r is exact
    const bool odd = fmod(r, 2.0) != 0.0;
    if (d > 0.5 || (d == 0.5 && odd)) r += 1.0;
    else if (d < -0.5 || (d == -0.5 && odd)) r -= 1.0;
    c = (long long)r;
    return true;
}
// residues of the signed coefficient c mod q_0..q_level (and the np_ext special primes) of plaintext p
__device__ __forceinline__ void enc_residues(long long c, u64 *out, const Primes &pr, int level, int np_ext, int Kfull,
                                             int p, int k, int N) {
    const int k1 = level + 1 + np_ext;
    for (int i = 0; i < k1; i++) {
        const ModConst &mc = pr.m[i <= level ? i : Kfull + (i - level - 1)];
        u64 res;
        if (c >= 0) res = mod64((u64)c, mc);
        else {
            const u64 t = mod64((u64)(-c), mc);
            res = t ? mc.q - t : 0;
        }
        out[((long long)p * k1 + i) * N + k] = res;
    }
}
// coefficient k = round_half_even(Re(buf[k]) * scale / N), residues mod q_0..q_level
__global__ void k_encode_finalize(const double *buf, u64 *out, Primes pr, double scale, int level, int logN,
                                  int *flag, int np_ext, int Kfull) {
    const int N = 1 << logN;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int p = blockIdx.y;
    if (k >= N) return;
    long long c;
    if (!enc_round(buf + ((long long)p * N + k) * 4, scale, logN, flag, c)) return;
    enc_residues(c, out, pr, level, np_ext, Kfull, p, k, N);
}
// Compact coefficient form (config 5, blb_matmul_encode_coeffs): the same rounded coefficient c,
// stored as 40-bit two's complement in 5 bytes -- plaintext p: N low 32-bit words, then N high bytes --
// when |c| < 2^39 (flag = 2 otherwise)
__global__ void k_encode_coef5(const double *buf, unsigned char *coef, double scale, int logN, int *flag) {
    const int N = 1 << logN;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int p = blockIdx.y;
    if (k >= N) return;
    long long c;
    if (!enc_round(buf + ((long long)p * N + k) * 4, scale, logN, flag, c)) return;
    if (c >= (1ll << 39) || c < -(1ll << 39)) {
        atomicExch(flag, 2);
        return;
    }
    unsigned char *b = coef + (long long)p * 5 * N;
    reinterpret_cast<uint32_t *>(b)[k] = (uint32_t)(unsigned long long)c;
    b[4 * N + k] = (unsigned char)((unsigned long long)c >> 32);
}
__global__ void k_coef5_residues(const unsigned char *coef, u64 *out, Primes pr, int level, int logN) {
    const int N = 1 << logN;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int p = blockIdx.y;
    if (k >= N) return;
    const unsigned char *b = coef + (long long)p * 5 * N;
    const unsigned long long u = (unsigned long long)reinterpret_cast<const uint32_t *>(b)[k] |
                                 ((unsigned long long)b[4 * N + k] << 32);
    const long long c = (long long)(u << 24) >> 24;  // sign-extend bit 39
    enc_residues(c, out, pr, level, 0, 0, p, k, N);
}

// centred lift of the q_0 residue -> double-double complex (imag 0)
__global__ void k_decode_lift(const u64 *coef, double *buf, Primes pr, int N) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= N) return;
    const u64 q = pr.m[0].q;
    const u64 v = coef[k];
    long long c = v > q / 2 ? -(long long)(q - v) : (long long)v;
    const double hi = (double)c;
    const double lo = (double)(c - (long long)hi);
    cst(buf + 4ll * k, {{hi, lo}, {0.0, 0.0}});
}

__global__ void k_decode_extract(const double *buf, const int32_t *slot_pos, double *out, double inv_scale, int N) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= N / 2) return;
    const double *b = buf + 4ll * slot_pos[j];
    out[j] = (b[0] + b[1]) * inv_scale;
}

__global__ void k_copy(const u64 *src, u64 *dst, int n) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x < n) dst[x] = src[x];
}

// ---------------------------------------------------------------------------
// Row f3: local fixed-point Decode of a secret share over Z_{2^128} (reading C18; P:684-685,
// App. C.4).  Same Cooley-Tukey network as the decode above (zeta^{brv(m+i)} twiddles), in
// wrapping 128-bit integer complex arithmetic with an arithmetic right shift by ft after each
// twiddle product (local truncation).  Twiddles W = round(2^ft zeta^e) from the double-double
// zeta table (no ties: the entries are irrational or exact integers).
// ---------------------------------------------------------------------------
typedef unsigned __int128 u128d;
typedef __int128 i128d;
__device__ __forceinline__ long long dd_round_scaled(double hi, double lo, int ft) {
    const double h = ldexp(hi, ft), l = ldexp(lo, ft);  // exact (power-of-two scaling)
    double r = rint(h);
    const double d = (h - r) + l;
    if (d > 0.5) r += 1.0;
    else if (d < -0.5) r -= 1.0;
    return (long long)r;
}
__global__ void k_fxp_tw(const double *zeta, long long *tw, int ft, int N) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const double *z = zeta + 4ll * i;
    tw[2 * i] = dd_round_scaled(z[0], z[1], ft);
    tw[2 * i + 1] = dd_round_scaled(z[2], z[3], ft);
}
__global__ void k_fxp_lift(const u64 *x, u128d *re, u128d *im, int N) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= N) return;
    re[k] = (u128d)x[2 * k] | ((u128d)x[2 * k + 1] << 64);
    im[k] = 0;
}
__global__ void k_fxp_stage(u128d *re, u128d *im, const long long *tw, int m, int N, int ft) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= N / 2) return;
    const int t = N / (2 * m);
    const int i = b / t, jj = b - i * t;
    const int j = 2 * i * t + jj;
    const u128d Wr = (u128d)(i128d)tw[2 * (m + i)], Wi = (u128d)(i128d)tw[2 * (m + i) + 1];
    const u128d yr = re[j + t], yi = im[j + t];
    const u128d vr = (u128d)((i128d)(yr * Wr - yi * Wi) >> ft);
    const u128d vi = (u128d)((i128d)(yr * Wi + yi * Wr) >> ft);
    const u128d xr = re[j], xi = im[j];
    re[j] = xr + vr;
    im[j] = xi + vi;
    re[j + t] = xr - vr;
    im[j + t] = xi - vi;
}
__global__ void k_fxp_extract(const u128d *re, const int32_t *slot_pos, u64 *y, int N, int s_out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= N / 2) return;
    const u128d v = (u128d)((i128d)re[slot_pos[j]] >> s_out);
    y[2 * j] = (u64)v;
    y[2 * j + 1] = (u64)(v >> 64);
}
// Row f3: local fixed-point Encode of a slot-vector share (reading C20; Alg. 2 line 1 P:647): the
// slot value at zeta^{5^j} and at its conjugate position, then the Gentleman-Sande network (the
// encode's k_stage inverse order) with conj(W) twiddles and >>_a ft after each twiddle product.
__global__ void k_fxp_scatter(const u64 *y, const int32_t *slot_pos, u128d *re, u128d *im, int N) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= N / 2) return;
    const u128d v = (u128d)y[2 * j] | ((u128d)y[2 * j + 1] << 64);
    const int pos = slot_pos[j];
    re[pos] = v;
    re[N - 1 - pos] = v;  // zeta^{-5^j}: 2 brv(N-1-pos) + 1 = 2N - 5^j
    im[pos] = 0;
    im[N - 1 - pos] = 0;
}
__global__ void k_fxp_stage_inv(u128d *re, u128d *im, const long long *tw, int m, int N, int ft) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= N / 2) return;
    const int t = N / (2 * m);
    const int i = b / t, jj = b - i * t;
    const int j = 2 * i * t + jj;
    const u128d Wr = (u128d)(i128d)tw[2 * (m + i)], Wi = (u128d)(i128d)(-tw[2 * (m + i) + 1]);  // conj(W)
    const u128d xr = re[j], xi = im[j], yr = re[j + t], yi = im[j + t];
    const u128d dr = xr - yr, di = xi - yi;
    re[j] = xr + yr;
    im[j] = xi + yi;
    re[j + t] = (u128d)((i128d)(dr * Wr - di * Wi) >> ft);
    im[j + t] = (u128d)((i128d)(dr * Wi + di * Wr) >> ft);
}
__global__ void k_fxp_coef(const u128d *re, u64 *x, int N, int s_out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= N) return;
    const u128d v = (u128d)((i128d)re[k] >> s_out);
    x[2 * k] = (u64)v;
    x[2 * k + 1] = (u64)(v >> 64);
}
}  // namespace

size_t encode_scratch_doubles(const blb_params *P, int n_pts) { return (size_t)n_pts * P->N * 4; }

blb_status launch_encode(const blb_params *P, const double *slots, int n_pts, double scale, int level, u64 *out,
                         double *buf, int *d_flag, cudaStream_t st, int np_ext) {
    const int N = P->N, logN = P->logN;
    if (n_pts <= 0) return BLB_OK;
    dim3 gs((N / 2 + kTB - 1) / kTB, n_pts);
    k_scatter<<<gs, kTB, 0, st>>>(slots, P->d_slot_pos, buf, n_pts, N);
    if (logN == 16) {
        constexpr size_t smem = (size_t)kEncElems * 32;
        blb_smem_optin(k_enc16_A, smem);
        blb_smem_optin(k_enc16_B, smem);
        k_enc16_A<<<dim3(N / kEncElems, n_pts), kTB, smem, st>>>(buf, P->d_zeta);
        k_enc16_B<<<dim3(256 / (kEncElems / 256), n_pts), kTB, smem, st>>>(buf, P->d_zeta);
    } else {
        for (int m = N / 2; m >= 1; m >>= 1) k_stage<<<gs, kTB, 0, st>>>(buf, P->d_zeta, m, logN, 1);
    }
    k_encode_finalize<<<dim3((N + kTB - 1) / kTB, n_pts), kTB, 0, st>>>(buf, out, P->pr, scale, level, logN, d_flag,
                                                                        np_ext, P->K);
    BLB_COUNT_LAUNCH(logN == 16 ? 4 : 2 + logN);
    BLB_CHECK_LAUNCH();
    RowBatch rb{};
    rb.base = out; rb.poly_stride = (long long)(level + 1 + np_ext) * N; rb.n_polys = n_pts; rb.limbs = level + 1 + np_ext;
    rb.limb0 = 0;
    for (int i = 0; i < rb.limbs; i++) rb.prime[i] = i <= level ? i : P->K + (i - level - 1);
    return launch_ntt(P, rb, false, st);
}

// slots -> compact 5-byte coefficients (k_encode_coef5); flag: 1 = |c| >= 2^52, 2 = |c| >= 2^39
blb_status launch_encode_coef5(const blb_params *P, const double *slots, int n_pts, double scale, unsigned char *coef,
                               double *buf, int *d_flag, cudaStream_t st) {
    const int N = P->N, logN = P->logN;
    if (n_pts <= 0) return BLB_OK;
    dim3 gs((N / 2 + kTB - 1) / kTB, n_pts);
    k_scatter<<<gs, kTB, 0, st>>>(slots, P->d_slot_pos, buf, n_pts, N);
    if (logN == 16) {
        constexpr size_t smem = (size_t)kEncElems * 32;
        blb_smem_optin(k_enc16_A, smem);
        blb_smem_optin(k_enc16_B, smem);
        k_enc16_A<<<dim3(N / kEncElems, n_pts), kTB, smem, st>>>(buf, P->d_zeta);
        k_enc16_B<<<dim3(256 / (kEncElems / 256), n_pts), kTB, smem, st>>>(buf, P->d_zeta);
    } else {
        for (int m = N / 2; m >= 1; m >>= 1) k_stage<<<gs, kTB, 0, st>>>(buf, P->d_zeta, m, logN, 1);
    }
    k_encode_coef5<<<dim3((N + kTB - 1) / kTB, n_pts), kTB, 0, st>>>(buf, coef, scale, logN, d_flag);
    BLB_COUNT_LAUNCH(logN == 16 ? 4 : 2 + logN);
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}
// compact coefficients -> NTT-form residues mod q_0..q_level (out [n_pts][level+1][N]): identical to
// launch_encode's output for the same slots
blb_status launch_coef5_to_rns(const blb_params *P, const unsigned char *coef, int n_pts, int level, u64 *out,
                               cudaStream_t st) {
    const int N = P->N;
    if (n_pts <= 0) return BLB_OK;
    k_coef5_residues<<<dim3((N + kTB - 1) / kTB, n_pts), kTB, 0, st>>>(coef, out, P->pr, level, P->logN);
    BLB_COUNT_LAUNCH(1);
    BLB_CHECK_LAUNCH();
    RowBatch rb{};
    rb.base = out; rb.poly_stride = (long long)(level + 1) * N; rb.n_polys = n_pts; rb.limbs = level + 1; rb.limb0 = 0;
    for (int i = 0; i < rb.limbs; i++) rb.prime[i] = i;
    return launch_ntt(P, rb, false, st);
}

// decode: scratch = N u64 + 4N doubles
blb_status launch_decode(const blb_params *P, const u64 *pt, double scale, double *slots_out, void *scratch,
                         cudaStream_t st) {
    const int N = P->N, logN = P->logN;
    u64 *coef = (u64 *)scratch;
    double *buf = (double *)(coef + N);
    k_copy<<<(N + kTB - 1) / kTB, kTB, 0, st>>>(pt, coef, N);
    RowBatch rb{};
    rb.base = coef; rb.poly_stride = N; rb.n_polys = 1; rb.limbs = 1; rb.limb0 = 0; rb.prime[0] = 0;
    BLB_TRY(launch_ntt(P, rb, true, st));
    k_decode_lift<<<(N + kTB - 1) / kTB, kTB, 0, st>>>(coef, buf, P->pr, N);
    dim3 gs((N / 2 + kTB - 1) / kTB, 1);
    for (int m = 1; m < N; m <<= 1) k_stage<<<gs, kTB, 0, st>>>(buf, P->d_zeta, m, logN, 0);
    k_decode_extract<<<(N / 2 + kTB - 1) / kTB, kTB, 0, st>>>(buf, P->d_slot_pos, slots_out, 1.0 / scale, N);
    BLB_COUNT_LAUNCH(3 + logN);
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}

extern "C" blb_status blb_share_decode(const blb_params *P, const uint64_t *x, int ft, int s_out, uint64_t *y, void *ws,
                                       size_t ws_bytes, void *stream) {
    if (!P || !x || !y || !ws || ft < 1 || ft > 52 || s_out < 0 || s_out > 126) return BLB_E_INVALID_ARG;
    const int N = P->N, logN = P->logN;
    if (ws_bytes < (size_t)N * 48) {
        blb_set_error("blb_share_decode: workspace needs %zu bytes", (size_t)N * 48);
        return BLB_E_NOMEM;
    }
    cudaStream_t st = (cudaStream_t)stream;
    u128d *re = (u128d *)ws, *im = re + N;
    long long *tw = (long long *)(im + N);
    k_fxp_tw<<<(N + kTB - 1) / kTB, kTB, 0, st>>>(P->d_zeta, tw, ft, N);
    k_fxp_lift<<<(N + kTB - 1) / kTB, kTB, 0, st>>>(x, re, im, N);
    for (int m = 1; m < N; m <<= 1) k_fxp_stage<<<(N / 2 + kTB - 1) / kTB, kTB, 0, st>>>(re, im, tw, m, N, ft);
    k_fxp_extract<<<(N / 2 + kTB - 1) / kTB, kTB, 0, st>>>(re, P->d_slot_pos, y, N, s_out);
    BLB_COUNT_LAUNCH(3 + logN);
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}

extern "C" blb_status blb_share_encode(const blb_params *P, const uint64_t *y, int ft, int s_out, uint64_t *x, void *ws,
                                       size_t ws_bytes, void *stream) {
    if (!P || !x || !y || !ws || ft < 1 || ft > 52 || s_out < 0 || s_out > 126) return BLB_E_INVALID_ARG;
    const int N = P->N;
    if (ws_bytes < (size_t)N * 48) {
        blb_set_error("blb_share_encode: workspace needs %zu bytes", (size_t)N * 48);
        return BLB_E_NOMEM;
    }
    cudaStream_t st = (cudaStream_t)stream;
    u128d *re = (u128d *)ws, *im = re + N;
    long long *tw = (long long *)(im + N);
    k_fxp_tw<<<(N + kTB - 1) / kTB, kTB, 0, st>>>(P->d_zeta, tw, ft, N);
    k_fxp_scatter<<<(N / 2 + kTB - 1) / kTB, kTB, 0, st>>>(y, P->d_slot_pos, re, im, N);
    for (int m = N / 2; m >= 1; m >>= 1)
        k_fxp_stage_inv<<<(N / 2 + kTB - 1) / kTB, kTB, 0, st>>>(re, im, tw, m, N, ft);
    k_fxp_coef<<<(N + kTB - 1) / kTB, kTB, 0, st>>>(re, x, N, s_out);
    BLB_COUNT_LAUNCH(3 + P->logN);
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}
