// api.cu -- the C ABI of include/blb.h: parameters, keys, encode/decode,
// encrypt/decrypt, rotation, rescale, products and the CKKS->MPC mask.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <algorithm>
#include "blb_internal.cuh"

extern "C" int blbh_is_prime(u64 n);
extern "C" int blbh_prime_chain(int logN, const int *bits, int count, u64 *out);
extern "C" u64 blbh_min_psi(u64 q, int logN);
extern "C" u64 blbh_shoup(u64 w, u64 q);
extern "C" u64 blbh_mulmod(u64 a, u64 b, u64 q);
extern "C" u64 blbh_powmod(u64 a, u64 e, u64 q);
extern "C" u64 blbh_invmod(u64 a, u64 q);
extern "C" void blbh_twiddles(u64 q, u64 psi, int logN, u64 *out);
extern "C" void blbh_zeta_dd(int logN, double *out);

blb_status launch_decode(const blb_params *P, const u64 *pt, double scale, double *slots_out, void *scratch,
                         cudaStream_t st);
blb_status blb_launch_sample_uniform(const blb_params *P, u64 *out, long long row_stride, int n_rows, const int *prime,
                                     const int *nonce, const uint8_t seed[32], uint32_t tag, u64 id, cudaStream_t st);
blb_status blb_launch_sample_small(const blb_params *P, u64 *out, long long row_stride, int n_rows, const int *prime,
                                   const uint8_t seed[32], uint32_t tag, u64 id, int mode, cudaStream_t st);
blb_status blb_launch_keygen_combine(const blb_params *P, u64 *b, const u64 *a, const u64 *s, long long stride,
                                     int n_rows, const int *prime, uint32_t galois, int relin, const u64 *gadget_dev,
                                     cudaStream_t st);
blb_status blb_launch_encrypt_combine(const blb_params *P, u64 *c0, const u64 *c1, const u64 *s, const u64 *pt, int k,
                                      cudaStream_t st);
blb_status blb_launch_decrypt(const blb_params *P, const u64 *c0, const u64 *c1, const u64 *s, u64 *out, int k,
                              cudaStream_t st);
blb_status blb_launch_mul_pt(const blb_params *P, const u64 *in, const u64 *pt, u64 *out, int k, cudaStream_t st);
blb_status blb_launch_sub(const blb_params *P, const u64 *a, const u64 *b, u64 *out, int k, int npoly,
                          cudaStream_t st);
blb_status blb_launch_add(const blb_params *P, const u64 *a, const u64 *b, u64 *out, int k, int npoly,
                          cudaStream_t st);
blb_status blb_launch_tensor(const blb_params *P, const u64 *a, const u64 *b, u64 *d, int k, cudaStream_t st);
blb_status blb_launch_tensor_n(const blb_params *P, const u64 *const *a, const u64 *const *b, int n, u64 *d, int k,
                               cudaStream_t st);
blb_status blb_launch_mul_pt_n(const blb_params *P, const u64 *const *in, const u64 *const *pt, int n, u64 *out, int k,
                               cudaStream_t st);
blb_status blb_launch_mask(const blb_params *P, const u64 *const *in, int n, int level, const uint8_t key[32],
                           u64 id0, u64 *masked, u64 *share, cudaStream_t st);

// ------------------------------------------------------------ errors
static thread_local char g_err[512] = "";
unsigned long long g_blb_counters[8] = {0, 0, 0, 0, 0, 0, 0, 0};

void blb_set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}
extern "C" const char *blb_last_error(void) { return g_err; }
extern "C" void blb_counters_get(uint64_t out[8]) {
    for (int i = 0; i < 8; i++) out[i] = __atomic_load_n(&g_blb_counters[i], __ATOMIC_RELAXED);
}
extern "C" void blb_counters_reset(void) {
    for (int i = 0; i < 8; i++) __atomic_store_n(&g_blb_counters[i], 0ull, __ATOMIC_RELAXED);
}

// ------------------------------------------------------------ live timing
#include <mutex>
namespace {
struct TimedLaunch {
    cudaEvent_t a, b;
    double bytes;
};
std::mutex g_tmu;
bool g_timing = false;
std::vector<TimedLaunch> g_tl[5];
std::vector<cudaEvent_t> g_pool;
cudaEvent_t take_event() {
    if (!g_pool.empty()) {
        cudaEvent_t e = g_pool.back();
        g_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}
}  // namespace
cudaEvent_t blb_timing_begin(cudaStream_t st) {
    std::lock_guard<std::mutex> lk(g_tmu);
    if (!g_timing) return nullptr;
    cudaEvent_t e = take_event();
    cudaEventRecord(e, st);
    return e;
}
void blb_timing_end(int cat, cudaEvent_t start, cudaStream_t st, double bytes) {
    if (!start) return;
    std::lock_guard<std::mutex> lk(g_tmu);
    cudaEvent_t e = take_event();
    cudaEventRecord(e, st);
    g_tl[cat].push_back({start, e, bytes});
}
// per-(kernel, device) record of the dynamic shared-memory opt-in (blb_smem_optin)
bool blb_smem_optin_needed(const void *kernel, size_t bytes) {
    static std::mutex mu;
    static std::vector<std::pair<const void *, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    (void)bytes;
    std::lock_guard<std::mutex> lk(mu);
    for (auto &d : done)
        if (d.first == kernel && d.second == dev) return false;
    done.push_back({kernel, dev});
    return true;
}
extern "C" void blb_timing_enable(int on) {
    std::lock_guard<std::mutex> lk(g_tmu);
    g_timing = on != 0;
}
extern "C" void blb_timing_reset(void) {
    std::lock_guard<std::mutex> lk(g_tmu);
    for (auto &v : g_tl) {
        for (auto &t : v) { g_pool.push_back(t.a); g_pool.push_back(t.b); }
        v.clear();
    }
}
extern "C" blb_status blb_timing_read(int cat, double *total_ms, uint64_t *launches, double *bytes) {
    if (cat < 0 || cat > 4) return BLB_E_INVALID_ARG;
    std::lock_guard<std::mutex> lk(g_tmu);
    double ms = 0, by = 0;
    for (auto &t : g_tl[cat]) {
        BLB_CUDA_TRY(cudaEventSynchronize(t.b));
        float f = 0;
        BLB_CUDA_TRY(cudaEventElapsedTime(&f, t.a, t.b));
        ms += f;
        by += t.bytes;
    }
    if (total_ms) *total_ms = ms;
    if (launches) *launches = g_tl[cat].size();
    if (bytes) *bytes = by;
    return BLB_OK;
}

// ------------------------------------------------------------ params
extern "C" blb_status blb_prime_chain(int log_n, const int *bits, int count, uint64_t *out) {
    if (!bits || !out || count <= 0 || log_n < 2 || log_n > 16) {
        blb_set_error("blb_prime_chain: invalid argument");
        return BLB_E_INVALID_ARG;
    }
    if (blbh_prime_chain(log_n, bits, count, out) != 0) {
        blb_set_error("blb_prime_chain: width outside [log_n+2, 61] or no prime left");
        return BLB_E_PARAM;
    }
    return BLB_OK;
}

static inline u64 host_brv(u64 x, int bits) {
    u64 r = 0;
    for (int i = 0; i < bits; i++) r |= ((x >> i) & 1ull) << (bits - 1 - i);
    return r;
}

static blb_status build_bconv(blb_params *P) {
    const int K = P->K, np = P->np, alpha = P->alpha;
    const int bt = (K + alpha - 1) / alpha;
    std::vector<u64> tab;
    P->bconv_off.assign((size_t)K * bt + K, 0);
    for (int lvl = 0; lvl < K; lvl++) {
        const int k = lvl + 1, E = k + np, beta = (k + alpha - 1) / alpha;
        for (int j = 0; j < beta; j++) {
            const int lo = j * alpha, hi = std::min((j + 1) * alpha, k), nd = hi - lo;
            P->bconv_off[(size_t)lvl * bt + j] = tab.size();
            std::vector<u64> inv(nd), invsh(nd), chat((size_t)nd * E);
            for (int d = 0; d < nd; d++) {
                const u64 ci = P->mod[lo + d];
                u64 h = 1 % ci;
                for (int e = 0; e < nd; e++)
                    if (e != d) h = blbh_mulmod(h, P->mod[lo + e] % ci, ci);
                inv[d] = blbh_invmod(h, ci);
                invsh[d] = blbh_shoup(inv[d], ci);
                for (int m = 0; m < E; m++) {
                    const u64 tm = P->mod[m < k ? m : K + (m - k)];
                    u64 hm = 1 % tm;
                    for (int e = 0; e < nd; e++)
                        if (e != d) hm = blbh_mulmod(hm, P->mod[lo + e] % tm, tm);
                    chat[(size_t)d * E + m] = hm;
                }
            }
            tab.insert(tab.end(), inv.begin(), inv.end());
            tab.insert(tab.end(), invsh.begin(), invsh.end());
            tab.insert(tab.end(), chat.begin(), chat.end());
        }
    }
    for (int lvl = 0; lvl < K; lvl++) {
        const int k = lvl + 1;
        P->bconv_off[(size_t)K * bt + lvl] = tab.size();
        std::vector<u64> inv(np), invsh(np), chat((size_t)np * k);
        for (int d = 0; d < np; d++) {
            const u64 pd = P->mod[K + d];
            u64 h = 1 % pd;
            for (int e = 0; e < np; e++)
                if (e != d) h = blbh_mulmod(h, P->mod[K + e] % pd, pd);
            inv[d] = blbh_invmod(h, pd);
            invsh[d] = blbh_shoup(inv[d], pd);
            for (int i = 0; i < k; i++) {
                const u64 qi = P->mod[i];
                u64 hm = 1 % qi;
                for (int e = 0; e < np; e++)
                    if (e != d) hm = blbh_mulmod(hm, P->mod[K + e] % qi, qi);
                chat[(size_t)d * k + i] = hm;
            }
        }
        tab.insert(tab.end(), inv.begin(), inv.end());
        tab.insert(tab.end(), invsh.begin(), invsh.end());
        tab.insert(tab.end(), chat.begin(), chat.end());
    }
    BLB_CUDA_TRY(cudaMalloc(&P->d_bconv, sizeof(u64) * std::max<size_t>(tab.size(), 1)));
    BLB_CUDA_TRY(cudaMemcpy(P->d_bconv, tab.data(), sizeof(u64) * tab.size(), cudaMemcpyHostToDevice));
    return BLB_OK;
}

extern "C" void blb_params_destroy(blb_params *P) {
    if (!P) return;
    if (P->aux) cudaStreamDestroy(P->aux);
    for (auto &e : P->ev)
        if (e) cudaEventDestroy(e);
    cudaFree(P->d_tw);
    cudaFree(P->d_twd);
    cudaFree(P->d_zeta);
    cudaFree(P->d_slot_pos);
    cudaFree(P->d_bconv);
    delete P;
}

extern "C" blb_status blb_params_create(blb_params **out, int log_n, const uint64_t *q, int nq, const uint64_t *p,
                                        int np, int dnum, int cuda_device) {
    if (!out || !q || !p) {
        blb_set_error("blb_params_create: null argument");
        return BLB_E_INVALID_ARG;
    }
    if (log_n < 2 || log_n > 16 || nq < 1 || np < 1 || nq + np > BLB_MAXP || dnum < 1 || dnum > nq) {
        blb_set_error("blb_params_create: log_n=%d nq=%d np=%d dnum=%d out of range", log_n, nq, np, dnum);
        return BLB_E_PARAM;
    }
    const u64 N = 1ull << log_n;
    std::vector<u64> mods(q, q + nq);
    mods.insert(mods.end(), p, p + np);
    for (size_t i = 0; i < mods.size(); i++) {
        const u64 m = mods[i];
        if (m >= (1ull << 61) || (m - 1) % (2 * N) || !blbh_is_prime(m)) {
            blb_set_error("modulus %llu is not a prime < 2^61 with p == 1 mod 2N", (unsigned long long)m);
            return BLB_E_PARAM;
        }
        for (size_t j = 0; j < i; j++)
            if (mods[j] == m) {
                blb_set_error("duplicate modulus %llu", (unsigned long long)m);
                return BLB_E_PARAM;
            }
    }
    BLB_CUDA_TRY(cudaSetDevice(cuda_device));
    auto *P = new blb_params();
    cudaDeviceGetAttribute(&P->num_sms, cudaDevAttrMultiProcessorCount, cuda_device);
    if (cudaStreamCreateWithFlags(&P->aux, cudaStreamNonBlocking) != cudaSuccess) P->aux = nullptr;
    for (auto &e : P->ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    P->logN = log_n; P->N = (int)N; P->K = nq; P->np = np; P->dnum = dnum; P->device = cuda_device;
    P->alpha = (nq + dnum - 1) / dnum;
    const int Lk = nq + np;
    for (int i = 0; i < Lk; i++) {
        const u64 m = mods[i];
        P->mod[i] = m;
        P->psi[i] = blbh_min_psi(m, log_n);
        ModConst &c = P->pr.m[i];
        c.q = m;
        c.ninv = blbh_invmod(N % m, m);
        c.ninv_sh = blbh_shoup(c.ninv, m);
        c.r64 = (u64)(((u128)1 << 64) % m);
        c.r64_sh = blbh_shoup(c.r64, m);
        c.mu = ~0ull / m;
    }
    for (int i = 0; i < nq; i++) {
        u64 Pm = 1 % P->mod[i];
        for (int t = 0; t < np; t++) Pm = blbh_mulmod(Pm, P->mod[nq + t] % P->mod[i], P->mod[i]);
        P->P_mod_q[i] = Pm;
        P->Pinv[i] = blbh_invmod(Pm, P->mod[i]);
        P->Pinv_sh[i] = blbh_shoup(P->Pinv[i], P->mod[i]);
    }
    // tables
    std::vector<u64> tw((size_t)Lk * 4 * N);
    for (int i = 0; i < Lk; i++) blbh_twiddles(P->mod[i], P->psi[i], log_n, tw.data() + (size_t)i * 4 * N);
    std::vector<double> zeta((size_t)4 * N);
    blbh_zeta_dd(log_n, zeta.data());
    std::vector<int32_t> pos(N / 2);
    u64 e = 1;
    for (u64 j = 0; j < N / 2; j++) {
        pos[j] = (int32_t)host_brv((e - 1) / 2, log_n);
        e = (e * 5) % (2 * N);
    }
    // FP64 NTT table (ntt.cu): the twiddles of the primes < 2^41 as doubles, [prime][2][N]
    std::vector<double> twd((size_t)Lk * 2 * N, 0.0);
    for (int i = 0; i < Lk; i++) {
        if (P->mod[i] >= (1ull << 41)) continue;
        for (size_t j = 0; j < (size_t)2 * N; j++) twd[(size_t)i * 2 * N + j] = (double)tw[(size_t)i * 4 * N + 2 * j];
    }
    cudaError_t err = cudaMalloc(&P->d_tw, sizeof(u64) * tw.size());
    if (err == cudaSuccess) err = cudaMemcpy(P->d_tw, tw.data(), sizeof(u64) * tw.size(), cudaMemcpyHostToDevice);
    if (err == cudaSuccess) err = cudaMalloc(&P->d_twd, sizeof(double) * twd.size());
    if (err == cudaSuccess) err = cudaMemcpy(P->d_twd, twd.data(), sizeof(double) * twd.size(), cudaMemcpyHostToDevice);
    if (err == cudaSuccess) err = cudaMalloc(&P->d_zeta, sizeof(double) * zeta.size());
    if (err == cudaSuccess)
        err = cudaMemcpy(P->d_zeta, zeta.data(), sizeof(double) * zeta.size(), cudaMemcpyHostToDevice);
    if (err == cudaSuccess) err = cudaMalloc(&P->d_slot_pos, sizeof(int32_t) * pos.size());
    if (err == cudaSuccess)
        err = cudaMemcpy(P->d_slot_pos, pos.data(), sizeof(int32_t) * pos.size(), cudaMemcpyHostToDevice);
    if (err != cudaSuccess) {
        blb_set_error("blb_params_create: %s", cudaGetErrorString(err));
        blb_params_destroy(P);
        return BLB_E_CUDA;
    }
    blb_status s = build_bconv(P);
    if (s != BLB_OK) {
        blb_params_destroy(P);
        return s;
    }
    *out = P;
    return BLB_OK;
}

extern "C" blb_status blb_params_query(const blb_params *P, int *log_n, int *nq, int *np, int *alpha, uint64_t *moduli,
                                       uint64_t *psi) {
    if (!P) return BLB_E_INVALID_ARG;
    if (log_n) *log_n = P->logN;
    if (nq) *nq = P->K;
    if (np) *np = P->np;
    if (alpha) *alpha = P->alpha;
    for (int i = 0; i < P->K + P->np; i++) {
        if (moduli) moduli[i] = P->mod[i];
        if (psi) psi[i] = P->psi[i];
    }
    return BLB_OK;
}

extern "C" uint32_t blb_galois_element(const blb_params *P, int32_t step) {
    const long long n = P->N / 2;
    long long s = step % n;
    if (s < 0) s += n;
    return (uint32_t)blbh_powmod(5, (u64)s, 2ull * P->N);
}

// ------------------------------------------------------------ NTT
static blb_status ntt_common(const blb_params *P, uint64_t *data, const int32_t *prime_idx, int n_limbs, int n_polys,
                             void *stream, bool inv) {
    if (!P || !data || !prime_idx || n_limbs < 1 || n_limbs > BLB_MAXP || n_polys < 0) {
        blb_set_error("blb_ntt: invalid argument");
        return BLB_E_INVALID_ARG;
    }
    RowBatch rb{};
    rb.base = data; rb.poly_stride = (long long)n_limbs * P->N; rb.n_polys = n_polys; rb.limbs = n_limbs; rb.limb0 = 0;
    for (int l = 0; l < n_limbs; l++) {
        if (prime_idx[l] < 0 || prime_idx[l] >= P->K + P->np) {
            blb_set_error("blb_ntt: prime index %d out of range", prime_idx[l]);
            return BLB_E_INVALID_ARG;
        }
        rb.prime[l] = prime_idx[l];
    }
    return launch_ntt(P, rb, inv, (cudaStream_t)stream);
}
extern "C" blb_status blb_ntt(const blb_params *P, uint64_t *data, const int32_t *prime_idx, int n_limbs, int n_polys,
                              void *stream) {
    return ntt_common(P, data, prime_idx, n_limbs, n_polys, stream, false);
}
extern "C" blb_status blb_intt(const blb_params *P, uint64_t *data, const int32_t *prime_idx, int n_limbs, int n_polys,
                               void *stream) {
    return ntt_common(P, data, prime_idx, n_limbs, n_polys, stream, true);
}

// ------------------------------------------------------------ encode / decode
extern "C" blb_status blb_encode(const blb_params *P, const double *slots, int n_pts, double scale, int level,
                                 uint64_t *out, void *stream) {
    if (!P || !slots || !out || n_pts < 0 || !(scale > 0)) {
        blb_set_error("blb_encode: invalid argument");
        return BLB_E_INVALID_ARG;
    }
    if (level < 0 || level >= P->K) {
        blb_set_error("blb_encode: level %d out of range", level);
        return BLB_E_LEVEL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int chunk = 64;
    double *buf = nullptr;
    int *flag = nullptr;
    BLB_CUDA_TRY(cudaMallocAsync(&buf, sizeof(double) * encode_scratch_doubles(P, std::min(chunk, std::max(n_pts, 1))), st));
    BLB_CUDA_TRY(cudaMallocAsync(&flag, sizeof(int), st));
    BLB_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int), st));
    blb_status s = BLB_OK;
    for (int p0 = 0; p0 < n_pts && s == BLB_OK; p0 += chunk) {
        const int cnt = std::min(chunk, n_pts - p0);
        s = launch_encode(P, slots + (size_t)p0 * (P->N / 2), cnt, scale, level, out + (size_t)p0 * (level + 1) * P->N,
                          buf, flag, st);
    }
    int h = 0;
    cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(buf, st);
    cudaFreeAsync(flag, st);
    BLB_CUDA_TRY(cudaStreamSynchronize(st));
    if (s != BLB_OK) return s;
    if (h) {
        blb_set_error("encode overflow: |scale * m_k| >= 2^52");
        return BLB_E_OVERFLOW;
    }
    return BLB_OK;
}

extern "C" blb_status blb_decode(const blb_params *P, const uint64_t *pt, int level, double scale, double *slots_out,
                                 void *stream) {
    if (!P || !pt || !slots_out || !(scale > 0) || level < 0 || level >= P->K) {
        blb_set_error("blb_decode: invalid argument");
        return BLB_E_INVALID_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    void *scratch = nullptr;
    BLB_CUDA_TRY(cudaMallocAsync(&scratch, (size_t)P->N * (8 + 32), st));
    blb_status s = launch_decode(P, pt, scale, slots_out, scratch, st);
    cudaFreeAsync(scratch, st);
    return s;
}

// ------------------------------------------------------------ keys
extern "C" blb_status blb_keys_create(const blb_params *P, blb_keys **out) {
    if (!P || !out) return BLB_E_INVALID_ARG;
    auto *k = new blb_keys();
    k->params = P;
    *out = k;
    return BLB_OK;
}
extern "C" void blb_keys_destroy(blb_keys *k) {
    if (!k) return;
    for (auto *d : k->data) cudaFree(d);
    delete k;
}
static size_t key_elems(const blb_params *P) { return (size_t)blb_beta_top(P) * 2 * (P->K + P->np) * P->N; }

static u64 *keys_slot(blb_keys *K, uint32_t g, blb_status *st) {
    for (size_t i = 0; i < K->galois.size(); i++)
        if (K->galois[i] == g) return K->data[i];
    u64 *d = nullptr;
    cudaError_t e = cudaMalloc(&d, sizeof(u64) * key_elems(K->params));
    if (e != cudaSuccess) {
        blb_set_error("key allocation: %s", cudaGetErrorString(e));
        *st = BLB_E_NOMEM;
        return nullptr;
    }
    K->galois.push_back(g);
    K->data.push_back(d);
    return d;
}

// Rotation keys are stored pre-permuted for the key-switch inner product (kernels.cu):
// k'[y] = k[perm_{g^-1}(y)] on every row, so the kernel reads keys and extended digits contiguously
// and scatters only its two outputs.  The relinearisation key (g = 0) is stored as is.
namespace {
__global__ void k_key_perm(const u64 *in, u64 *out, uint32_t ginv, int logN) {
    const int y = blockIdx.x * blockDim.x + threadIdx.x;
    const long long row = blockIdx.y;
    const int N = 1 << logN;
    if (y >= N) return;
    out[row * N + y] = in[row * N + galois_perm((uint32_t)y, ginv, logN)];
}
uint32_t host_galois_inverse(uint32_t g, int logN) {
    const u64 m = 2ull << logN;
    u64 r = 1, b = g % m, e = (1ull << logN) - 1;
    while (e) {
        if (e & 1) r = r * b % m;
        b = b * b % m;
        e >>= 1;
    }
    return (uint32_t)r;
}
}  // namespace
static blb_status store_key(const blb_params *P, u64 *slot, const u64 *natural, uint32_t g, cudaStream_t st) {
    const size_t n = key_elems(P);
    if (g == 0 || g == 1) {
        if (slot != natural) BLB_CUDA_TRY(cudaMemcpyAsync(slot, natural, sizeof(u64) * n, cudaMemcpyDefault, st));
        return BLB_OK;
    }
    u64 *tmp = nullptr;
    BLB_CUDA_TRY(cudaMallocAsync(&tmp, sizeof(u64) * n, st));
    BLB_CUDA_TRY(cudaMemcpyAsync(tmp, natural, sizeof(u64) * n, cudaMemcpyDefault, st));
    const unsigned rows = (unsigned)(n / P->N);
    k_key_perm<<<dim3((P->N + 255) / 256, rows), 256, 0, st>>>(tmp, slot, host_galois_inverse(g, P->logN), P->logN);
    BLB_COUNT_LAUNCH(1);
    BLB_CHECK_LAUNCH();
    cudaFreeAsync(tmp, st);
    return BLB_OK;
}

extern "C" blb_status blb_keys_add(blb_keys *K, uint32_t galois, const uint64_t *swk, void *stream) {
    if (!K || !swk) return BLB_E_INVALID_ARG;
    blb_status s = BLB_OK;
    u64 *d = keys_slot(K, galois, &s);
    if (!d) return s;
    return store_key(K->params, d, swk, galois, (cudaStream_t)stream);
}
extern "C" int blb_keys_has(const blb_keys *K, uint32_t galois) {
    if (!K) return 0;
    for (uint32_t g : K->galois)
        if (g == galois) return 1;
    return 0;
}

extern "C" blb_status blb_keygen(const blb_params *P, const uint8_t seed[32], const int32_t *rot_steps, int n_steps,
                                 int with_relin, blb_keys *K, uint64_t *secret_out, void *stream) {
    if (!P || !seed || !K || (n_steps > 0 && !rot_steps)) return BLB_E_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const int Lk = P->K + P->np, N = P->N, bt = blb_beta_top(P);
    int prime[BLB_MAXP], nonce[BLB_MAXP];
    for (int i = 0; i < Lk; i++) { prime[i] = i; nonce[i] = i; }
    u64 *s = secret_out;
    u64 *gadget = nullptr;
    if (!s) BLB_CUDA_TRY(cudaMallocAsync(&s, sizeof(u64) * Lk * N, st));
    BLB_TRY(blb_launch_sample_small(P, s, N, Lk, prime, seed, TAG_SECRET, 0, 0, st));
    RowBatch rb{};
    rb.base = s; rb.poly_stride = (long long)Lk * N; rb.n_polys = 1; rb.limbs = Lk; rb.limb0 = 0;
    for (int i = 0; i < Lk; i++) rb.prime[i] = i;
    BLB_TRY(launch_ntt(P, rb, false, st));
    // gadget P * pi_j per digit: [bt][Lk]
    std::vector<u64> gh((size_t)bt * Lk, 0);
    for (int j = 0; j < bt; j++)
        for (int i = j * P->alpha; i < std::min((j + 1) * P->alpha, P->K); i++) gh[(size_t)j * Lk + i] = P->P_mod_q[i];
    BLB_CUDA_TRY(cudaMallocAsync(&gadget, sizeof(u64) * gh.size(), st));
    BLB_CUDA_TRY(cudaMemcpyAsync(gadget, gh.data(), sizeof(u64) * gh.size(), cudaMemcpyHostToDevice, st));
    std::vector<uint32_t> gl;
    for (int t = 0; t < n_steps; t++) {
        const uint32_t g = blb_galois_element(P, rot_steps[t]);
        if (g != 1 && std::find(gl.begin(), gl.end(), g) == gl.end()) gl.push_back(g);
    }
    if (with_relin) gl.push_back(0);
    blb_status status = BLB_OK;
    for (uint32_t g : gl) {
        u64 *key = keys_slot(K, g, &status);
        if (!key) break;
        for (int j = 0; j < bt && status == BLB_OK; j++) {
            const u64 kid = (u64)g * 64 + (u64)j;
            u64 *b = key + ((size_t)j * 2 + 0) * Lk * N, *a = key + ((size_t)j * 2 + 1) * Lk * N;
            status = blb_launch_sample_uniform(P, a, N, Lk, prime, nonce, seed, TAG_KEY_A, kid, st);
            if (status == BLB_OK) status = blb_launch_sample_small(P, b, N, Lk, prime, seed, TAG_KEY_E, kid, 1, st);
            if (status == BLB_OK) {
                RowBatch eb = rb;
                eb.base = b;
                status = launch_ntt(P, eb, false, st);
            }
            if (status == BLB_OK)
                status = blb_launch_keygen_combine(P, b, a, s, N, Lk, prime, g == 0 ? 1u : g, g == 0,
                                                   gadget + (size_t)j * Lk, st);
        }
        if (status == BLB_OK) status = store_key(P, key, key, g, st);  // pre-permuted storage
        if (status != BLB_OK) break;
    }
    cudaFreeAsync(gadget, st);
    if (!secret_out) cudaFreeAsync(s, st);
    BLB_CUDA_TRY(cudaStreamSynchronize(st));
    return status;
}

// ------------------------------------------------------------ encrypt / decrypt
extern "C" blb_status blb_encrypt(const blb_params *P, const uint64_t *secret, const uint64_t *pt, int level,
                                  const uint8_t seed[32], uint64_t ct_id, double scale, blb_ct *out, void *stream) {
    if (!P || !secret || !pt || !seed || !out || !out->data) return BLB_E_INVALID_ARG;
    if (level < 0 || level >= P->K) {
        blb_set_error("blb_encrypt: level %d out of range", level);
        return BLB_E_LEVEL;
    }
    if (ct_id >> 56) {
        blb_set_error("blb_encrypt: ct_id must be < 2^56 (object id = ct_id << 8 | limb)");
        return BLB_E_INVALID_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int k = level + 1, N = P->N;
    int prime[BLB_MAXP], nonce[BLB_MAXP];
    for (int i = 0; i < k; i++) { prime[i] = i; nonce[i] = i; }
    u64 *c0 = out->data, *c1 = out->data + (size_t)k * N;
    BLB_TRY(blb_launch_sample_uniform(P, c1, N, k, prime, nonce, seed, TAG_ENC_A, ct_id, st));
    BLB_TRY(blb_launch_sample_small(P, c0, N, k, prime, seed, TAG_ENC_E, ct_id, 1, st));
    RowBatch rb{};
    rb.base = c0; rb.poly_stride = (long long)k * N; rb.n_polys = 1; rb.limbs = k; rb.limb0 = 0;
    for (int i = 0; i < k; i++) rb.prime[i] = i;
    BLB_TRY(launch_ntt(P, rb, false, st));
    BLB_TRY(blb_launch_encrypt_combine(P, c0, c1, secret, pt, k, st));
    out->level = level;
    out->scale = scale;
    return BLB_OK;
}

extern "C" blb_status blb_decrypt(const blb_params *P, const uint64_t *secret, const blb_ct *ct, uint64_t *pt_out,
                                  void *stream) {
    if (!P || !secret || !ct || !ct->data || !pt_out) return BLB_E_INVALID_ARG;
    if (ct->level < 0 || ct->level >= P->K) return BLB_E_LEVEL;
    const int k = ct->level + 1;
    return blb_launch_decrypt(P, ct->data, ct->data + (size_t)k * P->N, secret, pt_out, k, (cudaStream_t)stream);
}

// ------------------------------------------------------------ operations
extern "C" size_t blb_workspace_bytes(const blb_params *P, blb_op op, int level) {
    if (!P || level < 0 || level >= P->K) return 0;
    const size_t N = P->N, k = level + 1, E = k + P->np, beta = blb_beta(P, level);
    switch (op) {
        case BLB_OP_ROTATE: return sizeof(u64) * (beta * E * N + k * N + keyswitch_scratch_elems(P, level, 1));
        case BLB_OP_RESCALE: return sizeof(u64) * (2 + 2 * k) * N;
        case BLB_OP_MASK: return 0;
        case BLB_OP_ENCODE: return sizeof(double) * encode_scratch_doubles(P, 1);
    }
    return 0;
}

static const u64 *find_key(const blb_keys *K, uint32_t g) {
    for (size_t i = 0; i < K->galois.size(); i++)
        if (K->galois[i] == g) return K->data[i];
    return nullptr;
}

extern "C" blb_status blb_rotate(const blb_params *P, const blb_keys *K, const blb_ct *in, int32_t step, blb_ct *out,
                                 void *ws, size_t ws_bytes, void *stream) {
    if (!P || !K || !in || !in->data || !out || !out->data || in->data == out->data) {
        blb_set_error("blb_rotate: invalid argument");
        return BLB_E_INVALID_ARG;
    }
    const int level = in->level;
    if (level < 0 || level >= P->K) return BLB_E_LEVEL;
    cudaStream_t st = (cudaStream_t)stream;
    const int k = level + 1, N = P->N, E = k + P->np, beta = blb_beta(P, level);
    const uint32_t g = blb_galois_element(P, step);
    if (g == 1) {
        BLB_CUDA_TRY(cudaMemcpyAsync(out->data, in->data, sizeof(u64) * 2 * k * N, cudaMemcpyDeviceToDevice, st));
        out->level = level;
        out->scale = in->scale;
        return BLB_OK;
    }
    const u64 *key = find_key(K, g);
    if (!key) {
        blb_set_error("missing rotation key for step %d (galois %u)", step, g);
        return BLB_E_MISSING_KEY;
    }
    if (!ws || ws_bytes < blb_workspace_bytes(P, BLB_OP_ROTATE, level)) {
        blb_set_error("blb_rotate: workspace too small");
        return BLB_E_NOMEM;
    }
    u64 *ext = (u64 *)ws, *coef = ext + (size_t)beta * E * N, *u = coef + (size_t)k * N;
    u64 *conv = u + (size_t)2 * E * N;
    const u64 *c1 = in->data + (size_t)k * N;
    BLB_TRY(launch_modup(P, level, &c1, 1, ext, coef, st));
    KsJob J{};
    J.ext = ext; J.key = key; J.c0 = in->data; J.out = out->data; J.galois = g; J.add_mode = 1;
    BLB_TRY(launch_keyswitch(P, level, &J, 1, u, conv, st));
    out->level = level;
    out->scale = in->scale;
    return BLB_OK;
}

extern "C" blb_status blb_rescale(const blb_params *P, const blb_ct *in, blb_ct *out, void *ws, size_t ws_bytes,
                                  void *stream) {
    if (!P || !in || !in->data || !out || !out->data || in->data == out->data) return BLB_E_INVALID_ARG;
    if (in->level < 1 || in->level >= P->K) {
        blb_set_error("blb_rescale: level %d (depth exhausted)", in->level);
        return BLB_E_LEVEL;
    }
    if (!ws || ws_bytes < blb_workspace_bytes(P, BLB_OP_RESCALE, in->level)) {
        blb_set_error("blb_rescale: workspace too small");
        return BLB_E_NOMEM;
    }
    BLB_TRY(launch_rescale(P, in->data, in->level, 2, out->data, (u64 *)ws, (cudaStream_t)stream));
    out->level = in->level - 1;
    out->scale = in->scale / (double)P->mod[in->level];
    return BLB_OK;
}

extern "C" blb_status blb_mul_pt(const blb_params *P, const blb_ct *in, const uint64_t *pt, double pt_scale,
                                 blb_ct *out, void *stream) {
    if (!P || !in || !in->data || !pt || !out || !out->data) return BLB_E_INVALID_ARG;
    if (in->level < 0 || in->level >= P->K) return BLB_E_LEVEL;
    BLB_TRY(blb_launch_mul_pt(P, in->data, pt, out->data, in->level + 1, (cudaStream_t)stream));
    out->level = in->level;
    out->scale = in->scale * pt_scale;
    return BLB_OK;
}

extern "C" blb_status blb_add(const blb_params *P, const blb_ct *a, const blb_ct *b, blb_ct *out, void *stream) {
    if (!P || !a || !b || !out || !a->data || !b->data || !out->data) return BLB_E_INVALID_ARG;
    if (a->level != b->level) {
        blb_set_error("blb_add: level mismatch %d vs %d", a->level, b->level);
        return BLB_E_LEVEL;
    }
    const double r = a->scale / b->scale;
    if (r > 2.0 || r < 0.5) {
        blb_set_error("blb_add: scale mismatch > 1 bit");
        return BLB_E_SCALE;
    }
    BLB_TRY(blb_launch_add(P, a->data, b->data, out->data, a->level + 1, 2, (cudaStream_t)stream));
    out->level = a->level;
    out->scale = a->scale;
    return BLB_OK;
}

// ewadd_cp: out = (c0 + pt, c1) (pt: [level+1][N] NTT at the ciphertext's scale); out may alias in
extern "C" blb_status blb_add_pt(const blb_params *P, const blb_ct *in, const uint64_t *pt, blb_ct *out, void *stream) {
    if (!P || !in || !pt || !out || !in->data || !out->data) return BLB_E_INVALID_ARG;
    const int k = in->level + 1;
    cudaStream_t st = (cudaStream_t)stream;
    if (out->data != in->data)
        BLB_CUDA_TRY(cudaMemcpyAsync(out->data + (size_t)k * P->N, in->data + (size_t)k * P->N,
                                     sizeof(u64) * (size_t)k * P->N, cudaMemcpyDeviceToDevice, st));
    BLB_TRY(blb_launch_add(P, in->data, pt, out->data, k, 1, st));
    out->level = in->level;
    out->scale = in->scale;
    return BLB_OK;
}

// exact level drop (C9): out = the limbs q_0..q_level of in ([2][level+1][N])
extern "C" blb_status blb_drop_level(const blb_params *P, const blb_ct *in, int level, blb_ct *out, void *stream) {
    if (!P || !in || !out || !in->data || !out->data) return BLB_E_INVALID_ARG;
    if (level < 0 || level > in->level) {
        blb_set_error("blb_drop_level: level %d outside [0, %d]", level, in->level);
        return BLB_E_LEVEL;
    }
    const size_t N = P->N, kin = in->level + 1, k = level + 1;
    cudaStream_t st = (cudaStream_t)stream;
    for (int p = 0; p < 2; p++)
        BLB_CUDA_TRY(cudaMemcpyAsync(out->data + p * k * N, in->data + p * kin * N, sizeof(u64) * k * N,
                                     cudaMemcpyDeviceToDevice, st));
    out->level = level;
    out->scale = in->scale;
    return BLB_OK;
}

blb_status blb_launch_rerand(const blb_params *P, u64 *const *rr, int n, const u64 *pk, int kpk, const uint8_t seed[32],
                             u64 id0, int flood_bits, u64 *vee, cudaStream_t st);

// S13 (reading C22): CKKS->MPC with re-randomisation -- each input dropped to q_0, plus a fresh
// public-key encryption of zero with flooding noise, then the mask of blb_ckks_to_mpc
extern "C" size_t blb_ckks_to_mpc_rr_workspace_bytes(const blb_params *P, int n_ct) {
    return P && n_ct > 0 ? sizeof(u64) * (size_t)n_ct * 5 * P->N : 0;
}
extern "C" blb_status blb_ckks_to_mpc_rr(const blb_params *P, const blb_ct *pk, const blb_ct *in, int n_ct,
                                         const uint8_t mask_key[32], const uint8_t rr_seed[32], uint64_t first_ct_id,
                                         int flood_bits, uint64_t *masked, uint64_t *share, void *ws, size_t ws_bytes,
                                         void *stream) {
    if (!P || n_ct < 0) return BLB_E_INVALID_ARG;
    if (n_ct == 0) return BLB_OK;
    if (!pk || !pk->data || !in || !mask_key || !rr_seed || !masked || !share || !ws) return BLB_E_INVALID_ARG;
    if (flood_bits < 0 || flood_bits > 58) {
        blb_set_error("blb_ckks_to_mpc_rr: flood_bits must be in [0, 58]");
        return BLB_E_INVALID_ARG;
    }
    if ((first_ct_id + (u64)n_ct) >> 56) {
        blb_set_error("blb_ckks_to_mpc_rr: ct ids must be < 2^56");
        return BLB_E_INVALID_ARG;
    }
    if (ws_bytes < blb_ckks_to_mpc_rr_workspace_bytes(P, n_ct)) return BLB_E_NOMEM;
    const int N = P->N;
    cudaStream_t st = (cudaStream_t)stream;
    u64 *rrb = (u64 *)ws, *vee = rrb + (size_t)n_ct * 2 * N;
    std::vector<u64 *> rr(n_ct);
    std::vector<const u64 *> rrc(n_ct);
    for (int t = 0; t < n_ct; t++) {
        if (!in[t].data || in[t].level < 0) return BLB_E_INVALID_ARG;
        rr[t] = rrb + (size_t)t * 2 * N;
        rrc[t] = rr[t];
        const size_t kN = (size_t)(in[t].level + 1) * N;
        BLB_CUDA_TRY(cudaMemcpyAsync(rr[t], in[t].data, sizeof(u64) * N, cudaMemcpyDeviceToDevice, st));
        BLB_CUDA_TRY(cudaMemcpyAsync(rr[t] + N, in[t].data + kN, sizeof(u64) * N, cudaMemcpyDeviceToDevice, st));
    }
    BLB_TRY(blb_launch_rerand(P, rr.data(), n_ct, pk->data, pk->level + 1, rr_seed, first_ct_id, flood_bits, vee, st));
    return blb_launch_mask(P, rrc.data(), n_ct, 0, mask_key, first_ct_id, masked, share, st);
}

extern "C" blb_status blb_sub(const blb_params *P, const blb_ct *a, const blb_ct *b, blb_ct *out, void *stream) {
    if (!P || !a || !b || !out || !a->data || !b->data || !out->data) return BLB_E_INVALID_ARG;
    if (a->level != b->level) {
        blb_set_error("blb_sub: level mismatch %d vs %d", a->level, b->level);
        return BLB_E_LEVEL;
    }
    const double r = a->scale / b->scale;
    if (r > 2.0 || r < 0.5) {
        blb_set_error("blb_sub: scale mismatch > 1 bit");
        return BLB_E_SCALE;
    }
    BLB_TRY(blb_launch_sub(P, a->data, b->data, out->data, a->level + 1, 2, (cudaStream_t)stream));
    out->level = a->level;
    out->scale = a->scale;
    return BLB_OK;
}

extern "C" blb_status blb_ckks_to_mpc(const blb_params *P, const blb_ct *in, int n_ct, const uint8_t mask_key[32],
                                      uint64_t first_ct_id, uint64_t *masked, uint64_t *share, void *ws,
                                      size_t ws_bytes, void *stream) {
    (void)ws; (void)ws_bytes;
    if (!P || n_ct < 0) return BLB_E_INVALID_ARG;
    if (n_ct == 0) return BLB_OK;  // nothing to mask (output pointers may be null)
    if (!in || !mask_key || !masked || !share) return BLB_E_INVALID_ARG;
    if ((first_ct_id + (u64)n_ct) >> 56) {
        blb_set_error("blb_ckks_to_mpc: ct ids must be < 2^56");
        return BLB_E_INVALID_ARG;
    }
    const int level = in[0].level;
    std::vector<const u64 *> ptrs(n_ct);
    for (int t = 0; t < n_ct; t++) {
        if (!in[t].data) return BLB_E_INVALID_ARG;
        if (in[t].level != level) {
            blb_set_error("blb_ckks_to_mpc: all inputs must share one level");
            return BLB_E_LEVEL;
        }
        ptrs[t] = in[t].data;
    }
    return blb_launch_mask(P, ptrs.data(), n_ct, level, mask_key, first_ct_id, masked, share, (cudaStream_t)stream);
}

// ------------------------------------------------------------ row f3: MPC -> CKKS ingest
namespace {
__global__ void k_share_rns(const u64 *x, u64 *out, Primes pr, PinvTab two_w, int sub, int N) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y;
    if (j >= N) return;
    const ModConst &mc = pr.m[i];
    const u64 v = mod64(x[j], mc);
    out[(long long)i * N + j] = sub ? submod(v, two_w.v[i], mc.q) : v;
}
}  // namespace

extern "C" blb_status blb_share_to_rns(const blb_params *P, const uint64_t *x, int w, int sub, int level, uint64_t *out,
                                       void *stream) {
    if (!P || !x || !out || w < 1 || w > 64) return BLB_E_INVALID_ARG;
    if (level < 0 || level >= P->K) return BLB_E_LEVEL;
    const int k = level + 1, N = P->N;
    PinvTab tw{};
    for (int i = 0; i < k; i++) tw.v[i] = (u64)(((u128)1 << w) % P->mod[i]);
    cudaStream_t st = (cudaStream_t)stream;
    k_share_rns<<<dim3((N + 255) / 256, k), 256, 0, st>>>(x, out, P->pr, tw, sub ? 1 : 0, N);
    BLB_COUNT_LAUNCH(1);
    BLB_CHECK_LAUNCH();
    RowBatch rb{};
    rb.base = out; rb.poly_stride = (long long)k * N; rb.n_polys = 1; rb.limbs = k; rb.limb0 = 0;
    for (int i = 0; i < k; i++) rb.prime[i] = i;
    return launch_ntt(P, rb, false, st);
}

extern "C" blb_status blb_mpc_to_ckks(const blb_params *P, blb_ct *ct, const uint64_t *x1, int w, void *ws,
                                      size_t ws_bytes, void *stream) {
    if (!P || !ct || !ct->data || !x1 || !ws) return BLB_E_INVALID_ARG;
    const int k = ct->level + 1;
    if (ws_bytes < (size_t)k * P->N * sizeof(u64)) {
        blb_set_error("blb_mpc_to_ckks: workspace needs %zu bytes", (size_t)k * P->N * sizeof(u64));
        return BLB_E_NOMEM;
    }
    u64 *s = (u64 *)ws;
    BLB_TRY(blb_share_to_rns(P, x1, w, 1, ct->level, s, stream));
    return blb_launch_add(P, ct->data, s, ct->data, k, 1, (cudaStream_t)stream);
}

// 128-bit shares (w <= 128): x [N][2] little-endian words; v = (hi * 2^64 + lo) mod q_i
namespace {
__global__ void k_share_rns128(const u64 *x, u64 *out, Primes pr, PinvTab two_w, int sub, int N) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y;
    if (j >= N) return;
    const ModConst &mc = pr.m[i];
    const u64 v = reduce128(x[2 * j + 1], x[2 * j], mc);
    out[(long long)i * N + j] = sub ? submod(v, two_w.v[i], mc.q) : v;
}
}  // namespace

extern "C" blb_status blb_share_to_rns128(const blb_params *P, const uint64_t *x, int w, int sub, int level,
                                          uint64_t *out, void *stream) {
    if (!P || !x || !out || w < 1 || w > 128) return BLB_E_INVALID_ARG;
    if (level < 0 || level >= P->K) return BLB_E_LEVEL;
    const int k = level + 1, N = P->N;
    PinvTab tw{};
    for (int i = 0; i < k; i++) {
        const u64 q = P->mod[i];
        const u64 r64 = (u64)(((u128)1 << 64) % q);
        tw.v[i] = w < 128 ? (u64)(((u128)1 << w) % q) : (u64)(((u128)r64 * r64) % q);
    }
    cudaStream_t st = (cudaStream_t)stream;
    k_share_rns128<<<dim3((N + 255) / 256, k), 256, 0, st>>>(x, out, P->pr, tw, sub ? 1 : 0, N);
    BLB_COUNT_LAUNCH(1);
    BLB_CHECK_LAUNCH();
    RowBatch rb{};
    rb.base = out; rb.poly_stride = (long long)k * N; rb.n_polys = 1; rb.limbs = k; rb.limb0 = 0;
    for (int i = 0; i < k; i++) rb.prime[i] = i;
    return launch_ntt(P, rb, false, st);
}

extern "C" blb_status blb_mpc_to_ckks128(const blb_params *P, blb_ct *ct, const uint64_t *x1, int w, void *ws,
                                         size_t ws_bytes, void *stream) {
    if (!P || !ct || !ct->data || !x1 || !ws) return BLB_E_INVALID_ARG;
    const int k = ct->level + 1;
    if (ws_bytes < (size_t)k * P->N * sizeof(u64)) {
        blb_set_error("blb_mpc_to_ckks128: workspace needs %zu bytes", (size_t)k * P->N * sizeof(u64));
        return BLB_E_NOMEM;
    }
    u64 *s = (u64 *)ws;
    BLB_TRY(blb_share_to_rns128(P, x1, w, 1, ct->level, s, stream));
    return blb_launch_add(P, ct->data, s, ct->data, k, 1, (cudaStream_t)stream);
}

extern "C" blb_status blb_mhp_column_map(int d, int heads, int L, int log_n, int32_t *map_out, int *len) {
    if (!len || d <= 0 || heads <= 0 || d % heads || L <= 0 || log_n < 2) return BLB_E_INVALID_ARG;
    const int n = 1 << (log_n - 1);
    if (n % L) return BLB_E_LAYOUT;
    const int c = n / L;
    int Hp = 1;
    while (Hp < heads) Hp <<= 1;
    if (c % Hp) {
        blb_set_error("MHP: padded heads %d must divide c = %d", Hp, c);
        return BLB_E_LAYOUT;
    }
    const int dh = d / heads, g = c / Hp, J = (dh + g - 1) / g;
    const int need = J * c;
    if (map_out) {
        if (*len < need) {
            blb_set_error("MHP map buffer too small (%d < %d)", *len, need);
            return BLB_E_INVALID_ARG;
        }
        for (int j = 0; j < J; j++)
            for (int cc = 0; cc < g; cc++)
                for (int h = 0; h < Hp; h++) {
                    const int within = j * g + cc;
                    map_out[j * c + cc * Hp + h] = (h < heads && within < dh) ? h * dh + within : -1;
                }
    }
    *len = need;
    return BLB_OK;
}

// ------------------------------------------------------------ row f2: other fused-block HE ops
extern "C" size_t blb_f2_workspace_bytes(const blb_params *P, int level) {
    if (!P || level < 0 || level >= P->K) return 0;
    const size_t N = P->N, k = level + 1;
    // tensor [3][k][N] + one rotation workspace + a temporary ciphertext [2][k][N]
    return sizeof(u64) * (3 * k * N + 2 * k * N) + blb_workspace_bytes(P, BLB_OP_ROTATE, level);
}

extern "C" blb_status blb_mul_relin(const blb_params *P, const blb_keys *K, const blb_ct *a, const blb_ct *b,
                                    blb_ct *out, void *ws, size_t ws_bytes, void *stream) {
    if (!P || !K || !a || !b || !out || !a->data || !b->data || !out->data || !ws) return BLB_E_INVALID_ARG;
    if (a->level != b->level || a->level < 0 || a->level >= P->K) {
        blb_set_error("blb_mul_relin: operands must share one level");
        return BLB_E_LEVEL;
    }
    const u64 *rlk = find_key(K, 0);
    if (!rlk) {
        blb_set_error("missing relinearisation key");
        return BLB_E_MISSING_KEY;
    }
    const int level = a->level, k = level + 1, N = P->N, E = k + P->np, beta = blb_beta(P, level);
    if (ws_bytes < blb_f2_workspace_bytes(P, level)) return BLB_E_NOMEM;
    cudaStream_t st = (cudaStream_t)stream;
    u64 *d = (u64 *)ws;
    u64 *ext = d + (size_t)3 * k * N, *coef = ext + (size_t)beta * E * N, *u = coef + (size_t)k * N;
    u64 *conv = u + (size_t)2 * E * N;
    BLB_TRY(blb_launch_tensor(P, a->data, b->data, d, k, st));
    const u64 *d2 = d + (size_t)2 * k * N;
    BLB_TRY(launch_modup(P, level, &d2, 1, ext, coef, st));
    KsJob J{};
    J.ext = ext; J.key = rlk; J.c0 = d; J.c1_add = d + (size_t)k * N; J.out = out->data; J.galois = 1; J.add_mode = 2;
    BLB_TRY(launch_keyswitch(P, level, &J, 1, u, conv, st));
    BLB_COUNT(3, 1);
    out->level = level;
    out->scale = a->scale * b->scale;
    return BLB_OK;
}

// Batched ewmul_cc: n independent pairs in one tensor launch, one ModUp batch, one key-switch batch
// (the relinearisation key read once per tile for the whole batch) and one rescale batch -- the
// same operations, per pair, as blb_mul_relin followed by blb_rescale.
static size_t mrb_elems(const blb_params *P, int level, int n) {
    const size_t N = P->N, k = level + 1, E = k + P->np, beta = blb_beta(P, level);
    // tensors, extended digits, coefficient scratch, key-switch outputs, key-switch scratch (which
    // also takes the rescaled [n][2][level][N]), rescale scratch (last limbs + lifted residues)
    return (size_t)n * (3 * k + beta * E + k + 2 * k) * N + keyswitch_scratch_elems(P, level, n) +
           (size_t)n * 2 * (1 + k) * N;
}
extern "C" size_t blb_mul_relin_batch_workspace_bytes(const blb_params *P, int level, int n) {
    if (!P || level < 0 || level >= P->K || n < 1) return 0;
    return sizeof(u64) * mrb_elems(P, level, std::min(n, kMaxJobs));
}
extern "C" blb_status blb_mul_relin_batch(const blb_params *P, const blb_keys *K, const blb_ct *a, const blb_ct *b,
                                          int n, int rescale, blb_ct *out, void *ws, size_t ws_bytes, void *stream) {
    if (!P || !K || n < 0 || (n > 0 && (!a || !b || !out || !ws))) return BLB_E_INVALID_ARG;
    if (n == 0) return BLB_OK;
    const int level = a[0].level;
    for (int t = 0; t < n; t++) {
        if (!a[t].data || !b[t].data || !out[t].data) return BLB_E_INVALID_ARG;
        if (a[t].level != level || b[t].level != level) {
            blb_set_error("blb_mul_relin_batch: all operands must share one level");
            return BLB_E_LEVEL;
        }
    }
    if (level < (rescale ? 1 : 0) || level >= P->K) return BLB_E_LEVEL;
    const u64 *rlk = find_key(K, 0);
    if (!rlk) {
        blb_set_error("missing relinearisation key");
        return BLB_E_MISSING_KEY;
    }
    if (ws_bytes < blb_mul_relin_batch_workspace_bytes(P, level, n)) return BLB_E_NOMEM;
    const int k = level + 1, N = P->N, E = k + P->np, beta = blb_beta(P, level);
    cudaStream_t st = (cudaStream_t)stream;
    for (int t0 = 0; t0 < n; t0 += kMaxJobs) {
        const int m = std::min(kMaxJobs, n - t0);
        u64 *d = (u64 *)ws;
        u64 *ext = d + (size_t)m * 3 * k * N, *coef = ext + (size_t)m * beta * E * N;
        u64 *tmp = coef + (size_t)m * k * N, *ks = tmp + (size_t)m * 2 * k * N;
        u64 *resc = ks + keyswitch_scratch_elems(P, level, m);
        u64 *ks_u = ks, *ks_conv = ks + (size_t)m * 2 * E * N;
        std::vector<const u64 *> pa(m), pb(m), d2(m);
        for (int t = 0; t < m; t++) {
            pa[t] = a[t0 + t].data;
            pb[t] = b[t0 + t].data;
            d2[t] = d + ((size_t)t * 3 + 2) * k * N;
        }
        BLB_TRY(blb_launch_tensor_n(P, pa.data(), pb.data(), m, d, k, st));
        BLB_TRY(launch_modup(P, level, d2.data(), m, ext, coef, st));
        std::vector<KsJob> jobs(m);
        for (int t = 0; t < m; t++) {
            KsJob J{};
            J.ext = ext + (size_t)t * beta * E * N; J.key = rlk; J.c0 = d + (size_t)t * 3 * k * N;
            J.c1_add = J.c0 + (size_t)k * N;
            J.out = rescale ? tmp + (size_t)t * 2 * k * N : out[t0 + t].data;
            J.galois = 1; J.add_mode = 2;
            jobs[t] = J;
        }
        BLB_TRY(launch_keyswitch(P, level, jobs.data(), m, ks_u, ks_conv, st));
        BLB_COUNT(3, m);
        if (rescale) {
            // [m][2][k][N] -> [m][2][level][N] contiguous in ks scratch, then to the outputs
            u64 *r = ks;
            BLB_TRY(launch_rescale(P, tmp, level, 2 * m, r, resc, st));
            for (int t = 0; t < m; t++)
                BLB_CUDA_TRY(cudaMemcpyAsync(out[t0 + t].data, r + (size_t)t * 2 * level * N,
                                             sizeof(u64) * 2 * level * N, cudaMemcpyDeviceToDevice, st));
        }
        for (int t = 0; t < m; t++) {
            out[t0 + t].level = rescale ? level - 1 : level;
            out[t0 + t].scale = rescale ? (a[t0 + t].scale * b[t0 + t].scale) / (double)P->mod[level]
                                        : a[t0 + t].scale * b[t0 + t].scale;
        }
    }
    return BLB_OK;
}

// Batched ewmul_cp + rescale: out[t] = rescale(in[t] (x) pt[t]) -- one product launch and one
// rescale batch for n ciphertexts at one level (the per-ciphertext bits of blb_mul_pt + blb_rescale)
extern "C" size_t blb_mul_pt_rescale_batch_workspace_bytes(const blb_params *P, int level, int n) {
    if (!P || level < 1 || level >= P->K || n < 1) return 0;
    const size_t m = std::min(n, kMaxJobs), k = level + 1, N = P->N;
    return sizeof(u64) * (m * 2 * k * N + m * 2 * level * N + m * 2 * (1 + k) * N);
}
extern "C" blb_status blb_mul_pt_rescale_batch(const blb_params *P, const blb_ct *in, const uint64_t *const *pt,
                                               const double *pt_scale, int n, blb_ct *out, void *ws, size_t ws_bytes,
                                               void *stream) {
    if (!P || n < 0 || (n > 0 && (!in || !pt || !pt_scale || !out || !ws))) return BLB_E_INVALID_ARG;
    if (n == 0) return BLB_OK;
    const int level = in[0].level;
    for (int t = 0; t < n; t++) {
        if (!in[t].data || !pt[t] || !out[t].data) return BLB_E_INVALID_ARG;
        if (in[t].level != level) {
            blb_set_error("blb_mul_pt_rescale_batch: all inputs must share one level");
            return BLB_E_LEVEL;
        }
    }
    if (level < 1 || level >= P->K) return BLB_E_LEVEL;
    if (ws_bytes < blb_mul_pt_rescale_batch_workspace_bytes(P, level, n)) return BLB_E_NOMEM;
    const int k = level + 1, N = P->N;
    cudaStream_t st = (cudaStream_t)stream;
    for (int t0 = 0; t0 < n; t0 += kMaxJobs) {
        const int m = std::min(kMaxJobs, n - t0);
        u64 *prod = (u64 *)ws, *r = prod + (size_t)m * 2 * k * N, *resc = r + (size_t)m * 2 * level * N;
        std::vector<const u64 *> pi(m), pp(m);
        for (int t = 0; t < m; t++) { pi[t] = in[t0 + t].data; pp[t] = pt[t0 + t]; }
        BLB_TRY(blb_launch_mul_pt_n(P, pi.data(), pp.data(), m, prod, k, st));
        BLB_TRY(launch_rescale(P, prod, level, 2 * m, r, resc, st));
        for (int t = 0; t < m; t++) {
            BLB_CUDA_TRY(cudaMemcpyAsync(out[t0 + t].data, r + (size_t)t * 2 * level * N, sizeof(u64) * 2 * level * N,
                                         cudaMemcpyDeviceToDevice, st));
            out[t0 + t].level = level - 1;
            out[t0 + t].scale = (in[t0 + t].scale * pt_scale[t0 + t]) / (double)P->mod[level];
        }
    }
    return BLB_OK;
}

// Rotate-and-sum: m^0 = m, m^i = m^{i-1} + Rot^{2^{i-1} L}(m^{i-1}), i = 1..log2 D,
// left rotations for sum (direction = +1), right rotations for broadcast (direction = -1).
static blb_status rotate_and_sum(const blb_params *P, const blb_keys *K, const blb_ct *in, int L, int D, int dir,
                                 blb_ct *out, void *ws, size_t ws_bytes, cudaStream_t st) {
    if (!P || !K || !in || !out || !in->data || !out->data || !ws || in->data == out->data) return BLB_E_INVALID_ARG;
    if (L <= 0 || D <= 0 || (D & (D - 1))) {
        blb_set_error("rotate-and-sum: D must be a power of two (pad otherwise)");
        return BLB_E_LAYOUT;
    }
    const int level = in->level, k = level + 1, N = P->N;
    if (ws_bytes < blb_f2_workspace_bytes(P, level)) return BLB_E_NOMEM;
    u64 *tmp = (u64 *)ws + (size_t)3 * k * N;
    u64 *rws = tmp + (size_t)2 * k * N;
    const size_t rbytes = blb_workspace_bytes(P, BLB_OP_ROTATE, level);
    BLB_CUDA_TRY(cudaMemcpyAsync(out->data, in->data, sizeof(u64) * 2 * k * N, cudaMemcpyDeviceToDevice, st));
    out->level = level;
    out->scale = in->scale;
    for (int step = L; step < L * D; step *= 2) {
        blb_ct cur = *out, t{tmp, level, 0, in->scale};
        BLB_TRY(blb_rotate(P, K, &cur, dir * step, &t, rws, rbytes, st));
        BLB_TRY(blb_launch_add(P, out->data, tmp, out->data, k, 2, st));
    }
    return BLB_OK;
}
extern "C" blb_status blb_rotate_sum(const blb_params *P, const blb_keys *K, const blb_ct *in, int L, int D,
                                     blb_ct *out, void *ws, size_t ws_bytes, void *stream) {
    return rotate_and_sum(P, K, in, L, D, +1, out, ws, ws_bytes, (cudaStream_t)stream);
}
extern "C" blb_status blb_broadcast(const blb_params *P, const blb_keys *K, const blb_ct *in, int L, int D,
                                    blb_ct *out, void *ws, size_t ws_bytes, void *stream) {
    return rotate_and_sum(P, K, in, L, D, -1, out, ws, ws_bytes, (cudaStream_t)stream);
}
