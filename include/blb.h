/*
 * blb.h -- C ABI of the B200-native BLB CKKS fused-linear hot path.
 *
 * BLB = "Breaking the Layer Barrier: Remodeling Private Transformer Inference
 * with Hybrid CKKS and MPC" (arXiv 2508.19525).  This library evaluates, on one
 * sm_100a GPU, the server side of the paper's fused linear blocks under CKKS:
 * limb-batched negacyclic NTT, encode, hoisted rotations with hybrid key
 * switching (ModUp / ModDown), the ct-pt MatMul protocol with BSGS, rescale,
 * and the CKKS->MPC mask of Algorithm 1.  Citations: P:n = PAPER.md line n,
 * C<k> / S<k> = the readings listed in DESIGN.md.
 *
 * Conventions for every entry point
 *   * Ownership: every uint64_t* / double* / void* data argument is memory owned
 *     by the caller (device memory unless the comment says "host").  The
 *     library never frees or retains it.  blb_params / blb_keys /
 *     blb_matmul_plan are library-owned (create / destroy pairs) and immutable
 *     once built; they may be shared by threads and streams.
 *   * Layout: a polynomial is N contiguous uint64 residues per RNS limb, limbs
 *     consecutive ("limb-major").  Ciphertext = [2][level+1][N] (c0 then c1),
 *     plaintext = [level+1][N], both in NTT form (NTT(a)[k] = a(psi^{2brv(k)+1})
 *     mod q, C2) unless stated.  Every residue is canonical, in [0, q).
 *   * Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy
 *     default).  All device work is stream-ordered and asynchronous; argument
 *     errors are reported synchronously before any launch; asynchronous faults
 *     surface as BLB_E_CUDA from a later call.
 *   * Errors: every function returns a blb_status; blb_last_error() returns a
 *     thread-local message for the last non-OK status.
 *   * Scratch: hot calls never allocate; they take a caller workspace `ws` of at
 *     least the bytes the matching *_workspace_bytes query returns.
 */
#ifndef BLB_H
#define BLB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BLB_MAX_PRIMES 24

typedef enum {
    BLB_OK = 0,
    BLB_E_INVALID_ARG = 1, /* null pointer, bad size or range                        */
    BLB_E_PARAM = 2,       /* prime != 1 mod 2N, not prime, >= 2^61, duplicate, bad N/dnum */
    BLB_E_MISSING_KEY = 3, /* rotation / relinearisation key absent       */
    BLB_E_LEVEL = 4,       /* level mismatch or depth exhausted    */
    BLB_E_SCALE = 5,       /* scale mismatch                                    */
    BLB_E_LAYOUT = 6,      /* shape / packing mismatch                  */
    BLB_E_OVERFLOW = 7,    /* encode magnitude |round(scale * m_k)| >= 2^52     */
    BLB_E_CUDA = 8,        /* CUDA runtime error                                        */
    BLB_E_NOMEM = 9,       /* allocation failure / workspace too small                  */
} blb_status;

typedef struct blb_params blb_params;
typedef struct blb_keys blb_keys;
typedef struct blb_matmul_plan blb_matmul_plan;

/* A ciphertext view (device memory owned by the caller): data = [2][level+1][N]
 * uint64, NTT form; scale = the CKKS scaling factor Delta tracked as a double. */
typedef struct {
    uint64_t *data;
    int32_t level;
    int32_t reserved;
    double scale;
} blb_ct;

typedef enum { BLB_PACK_SPATIAL = 0, BLB_PACK_DIAGONAL = 1 } blb_packing;

typedef enum {
    BLB_OP_ROTATE = 0,
    BLB_OP_RESCALE = 1,
    BLB_OP_MASK = 2,
    BLB_OP_ENCODE = 3,
} blb_op;

/* ------------------------------------------------------------------ */
/* errors, counters                                                     */
/* ------------------------------------------------------------------ */
const char *blb_last_error(void);

/* Process-wide counters: [0] kernel launches, [1] key switches (rotations +
 * relinearisations), [2] limb NTT/INTT transforms, [3] ct-pt products,
 * [4] rescales, [5] masks, [6] limb transforms on primes >= 2^41 (integer NTT kernel),
 * [7] reserved (0).  Host memory out[8]. */
void blb_counters_get(uint64_t out[8]);
void blb_counters_reset(void);

/* Live kernel timing (bench instrumentation).  When enabled, the library
 * records a CUDA event pair on the launching stream around every launch of
 * the tracked kernels: category 0 = ct-pt weight MAC (k_mac_tma4 / k_mac_tma), 1 = NTT/INTT passes,
 * 2 = key-switch inner product, 3 = ct-ct mask MAC (k_mac / k_mac_j), 4 = ct-ct tensor J-sum (k_tensor_sum).  blb_timing_read synchronises the recorded
 * events and returns, for `category`, the summed device milliseconds, the
 * number of launches and the summed ALGORITHMIC bytes (MAC: k*N*8 per
 * plaintext; NTT: 2*N*8 per limb; inner product: 2*beta*(k+np)*N*8 key bytes
 * per key switch).  Host outputs, nullable. */
/* Measured arithmetic-pipe peaks of device `device` (the integer-pipe fraction of the
 * NTT needs a denominator measured on the box): ops/s of 32-bit IMAD (fma-heavy pipe, mad.lo.u32)
 * and of DFMA (FP64 pipe), best of 3 timed launches of independent dependency chains, 8 CTAs per
 * SM.  Benchmark instrumentation, not a hot-path call; synchronises.  BLB_E_INVALID_ARG on null
 * outputs, BLB_E_CUDA on a CUDA error. */
blb_status blb_measure_pipe_peaks(int device, double *imad_per_s, double *dfma_per_s, void *stream);
void blb_timing_enable(int on);
void blb_timing_reset(void);
blb_status blb_timing_read(int category, double *total_ms, uint64_t *launches, double *alg_bytes);

/* ------------------------------------------------------------------ */
/* parameters (C1; Table 6 P:716-720 for the chain shape)               */
/* ------------------------------------------------------------------ */
/* Host helper, C1 prime-list rule: for each width bits[i] (chain order), the
 * largest prime < 2^bits[i] with p == 1 (mod 2N) not already chosen.
 * out: host [count].  BLB_E_PARAM if a width is outside [log_n+2, 61]. */
blb_status blb_prime_chain(int log_n, const int *bits, int count, uint64_t *out);

/* Create the parameter set of ring A_{N,q} = Z_q[x]/(x^N+1) in RNS:
 * ciphertext chain q[0..nq) (q[0] first, rescale drops q[nq-1] first) and
 * special primes p[0..np) for hybrid key switching (reading S2; P:233 says
 * only "rotation").  dnum = number of key-switch digits; the digit size is
 * alpha = ceil(nq / dnum), digit j = {q_i : j*alpha <= i < (j+1)*alpha}.
 * q, p: host arrays.  log_n in [2, 16].  Uploads twiddle / base-conversion
 * tables to `cuda_device`.  Errors: BLB_E_PARAM. */
blb_status blb_params_create(blb_params **out, int log_n, const uint64_t *q, int nq, const uint64_t *p, int np,
                             int dnum, int cuda_device);
void blb_params_destroy(blb_params *params);

/* Host outputs: log_n, nq, np, alpha; moduli[nq+np] (q then p) and the minimal
 * primitive 2N-th roots psi[nq+np] (C1).  Any output pointer may be NULL. */
blb_status blb_params_query(const blb_params *params, int *log_n, int *nq, int *np, int *alpha, uint64_t *moduli,
                            uint64_t *psi);

/* Galois element of a left rotation by `step` slots: 5^(step mod N/2) mod 2N
 * ("by default, we use left rotation"; reading S4). */
uint32_t blb_galois_element(const blb_params *params, int32_t step);

/* ------------------------------------------------------------------ */
/* NTT (row a1; C2)                                                     */
/* ------------------------------------------------------------------ */
/* In-place forward / inverse negacyclic NTT of n_polys x n_limbs rows,
 * data = [n_polys][n_limbs][N]; row (p, l) is reduced with modulus index
 * prime_idx[l] (host array, indices into q then p).  Input residues must be
 * in [0, q); output is canonical.  INTT includes the factor N^{-1}. */
blb_status blb_ntt(const blb_params *params, uint64_t *data, const int32_t *prime_idx, int n_limbs, int n_polys,
                   void *stream);
blb_status blb_intt(const blb_params *params, uint64_t *data, const int32_t *prime_idx, int n_limbs, int n_polys,
                    void *stream);

/* ------------------------------------------------------------------ */
/* encode / decode (Eq. eq:ckks_encode; C3)                  */
/* ------------------------------------------------------------------ */
/* Encode n_pts real slot vectors slots[n_pts][N/2] (device, float64) as
 * plaintexts out[n_pts][level+1][N] (NTT form): coefficient k is the
 * correctly rounded (ties-to-even) integer nearest to scale * m_k with
 * m = pi^{-1}(z), slot j <-> root zeta^{5^j}, zeta = e^{i pi / N}; the inverse
 * canonical embedding is evaluated in double-double arithmetic.  Real slots
 * only (footnote P:540).  BLB_E_OVERFLOW if some |scale * m_k| >= 2^52.
 * Synchronises `stream` (to read the overflow flag). */
blb_status blb_encode(const blb_params *params, const double *slots, int n_pts, double scale, int level,
                      uint64_t *out, void *stream);

/* Decode a plaintext pt[level+1][N] (NTT form) to slots_out[N/2] (device):
 * z_j = Re(m(zeta^{5^j})) / scale with m the centred lift of limb q_0
 * (precondition: every |coefficient| < q_0 / 2, true for decrypted outputs
 * at scale ~ 2^40 with the BLB presets). */
blb_status blb_decode(const blb_params *params, const uint64_t *pt, int level, double scale, double *slots_out,
                      void *stream);

/* ------------------------------------------------------------------ */
/* keys (C5) -- generated by the client; the server only loads them      */
/* ------------------------------------------------------------------ */
blb_status blb_keys_create(const blb_params *params, blb_keys **out);
void blb_keys_destroy(blb_keys *keys);

/* Copy one switching key swk[beta_top][2][nq+np][N] (device or host, NTT form, natural
 * coefficient order; [.][0] = b, [.][1] = a, beta_top = ceil(nq/alpha)) into `keys` under
 * Galois element `galois` (0 = relinearisation key for s^2).  Rotation keys are stored
 * pre-permuted (row y holds entry perm_{g^-1}(y)) so the key-switch inner product reads
 * keys and digits contiguously; the storage is internal to the library. */
blb_status blb_keys_add(blb_keys *keys, uint32_t galois, const uint64_t *swk, void *stream);
int blb_keys_has(const blb_keys *keys, uint32_t galois);

/* Test / client helper: generate the ternary secret s from `seed` (ChaCha20,
 * reading C4) and the switching keys for the given rotation steps (and s^2
 * if with_relin) into `keys`.  secret_out (nullable, device) receives
 * NTT(s) over all nq+np primes, [nq+np][N].  Synchronises `stream`. */
blb_status blb_keygen(const blb_params *params, const uint8_t seed[32], const int32_t *rot_steps, int n_steps,
                      int with_relin, blb_keys *keys, uint64_t *secret_out, void *stream);

/* ------------------------------------------------------------------ */
/* encrypt / decrypt (C6) -- client side, used by tests and the bench    */
/* ------------------------------------------------------------------ */
/* Symmetric encryption at `level`: c1 = a (uniform, NTT domain, ChaCha ENC_A),
 * c0 = -a*s + pt + e (e centred binomial eta = 21, ChaCha ENC_E), object id =
 * ct_id.  secret: [nq+np][N] NTT; pt: [level+1][N]; out->data [2][level+1][N]. */
blb_status blb_encrypt(const blb_params *params, const uint64_t *secret, const uint64_t *pt, int level,
                       const uint8_t seed[32], uint64_t ct_id, double scale, blb_ct *out, void *stream);
/* Dec(ct) = c0 + c1*s mod Q_level (NTT form) -> pt_out [level+1][N]. */
blb_status blb_decrypt(const blb_params *params, const uint64_t *secret, const blb_ct *ct, uint64_t *pt_out,
                       void *stream);

/* ------------------------------------------------------------------ */
/* homomorphic operations                                               */
/* ------------------------------------------------------------------ */
size_t blb_workspace_bytes(const blb_params *params, blb_op op, int level);

/* Left rotation by `step` slots, hoisted form (C8):
 * (sigma_g(c0) + c0', c1') with (c0', c1') = ModDown(sum_j sigma_g(ModUp(D_j(c1))) (.) rk_{g,j}).
 * `out` may not alias `in`.  BLB_E_MISSING_KEY if the key for g is absent. */
blb_status blb_rotate(const blb_params *params, const blb_keys *keys, const blb_ct *in, int32_t step, blb_ct *out,
                      void *ws, size_t ws_bytes, void *stream);

/* Rescale (reading S7 / C10): out = round(in / q_level) exactly, level-1,
 * scale / q_level.  out->data [2][level][N], may not alias in. */
blb_status blb_rescale(const blb_params *params, const blb_ct *in, blb_ct *out, void *ws, size_t ws_bytes,
                       void *stream);

/* ct (x) pt (C9): out = (c0 * pt, c1 * pt), scale = in.scale * pt_scale. */
blb_status blb_mul_pt(const blb_params *params, const blb_ct *in, const uint64_t *pt, double pt_scale, blb_ct *out,
                      void *stream);
/* ct + ct (same level): out = a + b (may alias a). BLB_E_SCALE if scales differ by > 1 bit. */
blb_status blb_add(const blb_params *params, const blb_ct *a, const blb_ct *b, blb_ct *out, void *stream);
/* ewadd_cp (e.g. the "+1" of negExp and the "+beta" of LayerNorm):
 * out = (c0 + pt, c1), pt device [level+1][N] NTT form encoded at the ciphertext's scale and
 * level; out may alias in; scale / level of in. */
blb_status blb_add_pt(const blb_params *params, const blb_ct *in, const uint64_t *pt, blb_ct *out, void *stream);
/* Exact level drop (C9: levels are aligned by dropping limbs): out = the residues mod
 * q_0..q_level of in; out [2][level+1][N] must not overlap in; BLB_E_LEVEL if level > in->level. */
blb_status blb_drop_level(const blb_params *params, const blb_ct *in, int level, blb_ct *out, void *stream);
/* ct - ct (same level; sadd_cc with a negated operand, e.g. X - Xbar of Softmax and X - mu of
 * LayerNorm): out = a - b limb-wise (may alias a), scale a.scale; BLB_E_LEVEL /
 * BLB_E_SCALE as blb_add. */
blb_status blb_sub(const blb_params *params, const blb_ct *a, const blb_ct *b, blb_ct *out, void *stream);

/* CKKS->MPC masking, server half of Algorithm 1 line 1 (F_C2M items 1
 * and 4; reading C14): for each of n_ct ciphertexts, drop to q_0,
 * INTT both polynomials, sample r uniform over Z_{q0}^N (ChaCha20 MASK,
 * object id first_ct_id + t), output masked[t] = (c0 + r, c1) and
 * share[t] = -r mod q_0, coefficient form.  masked: [n_ct][2][N], share:
 * [n_ct][N].  in[t].data must be distinct ciphertexts (not modified). */
blb_status blb_ckks_to_mpc(const blb_params *params, const blb_ct *in, int n_ct, const uint8_t mask_key[32],
                           uint64_t first_ct_id, uint64_t *masked, uint64_t *share, void *ws, size_t ws_bytes,
                           void *stream);

/* Optional re-randomisation before the mask (S13; the paper is silent on circuit privacy: Alg. 1
 * sends (c0 + r, c1), while the proof simulates P0's view as a fresh encryption, P:1031;
 * reading C22).  Each input is dropped to q_0 and a fresh public-key encryption of zero is added:
 * (c0 + v b + e0, c1 + v a + e1) mod q_0 with pk = (b, a) the client's encryption of zero (blb_encrypt
 * of 0 at the top level, id 2^55), v ternary (ChaCha tag 7), e1 centred binomial (tag 9) and e0 the
 * flooding noise (tag 8): uniform in [-2^f, 2^f) from the low f+1 bits of each draw (f = flood_bits
 * in [1, 58]) or centred binomial for f = 0; every draw keyed by rr_seed and the conversion's id
 * first_ct_id + t; then exactly the mask of blb_ckks_to_mpc.  ws >= n_ct * 5 N * 8 bytes
 * (blb_ckks_to_mpc_rr_workspace_bytes).  Errors as blb_ckks_to_mpc, BLB_E_INVALID_ARG for f > 58. */
size_t blb_ckks_to_mpc_rr_workspace_bytes(const blb_params *params, int n_ct);
blb_status blb_ckks_to_mpc_rr(const blb_params *params, const blb_ct *pk, const blb_ct *in, int n_ct,
                              const uint8_t mask_key[32], const uint8_t rr_seed[32], uint64_t first_ct_id, int flood_bits,
                              uint64_t *masked, uint64_t *share, void *ws, size_t ws_bytes, void *stream);

/* Row f3, MPC -> CKKS ingest (Algorithm 2; ring-to-field, App. C.3).
 * blb_share_to_rns: a secret share x over Z_{2^w} (device u64 [N], values < 2^w, 1 <= w <= 64,
 * coefficient order) mapped to the field per limb i <= level: x mod q_i (P0's share, sub = 0)
 * or x - 2^w mod q_i (P1's share, sub = 1), then NTT (C2).  out: device [level+1][N].
 * blb_mpc_to_ckks: the server (P1) half of Alg. 2 line 4 -- ct (the client's encryption of
 * its field share, level l, NTT) is updated in place: c0 += NTT(x1 - 2^w mod q_i).  The result
 * encrypts x0 + x1 - 2^w = m whenever x0 + x1 = m + 2^w (probability >= 1 - 2^-40 for
 * w = l + 40).  ws: device scratch >= (level+1) * N * 8 bytes.  Errors:
 * BLB_E_INVALID_ARG (null / w out of range), BLB_E_LEVEL, BLB_E_NOMEM (workspace). */
blb_status blb_share_to_rns(const blb_params *params, const uint64_t *x, int w, int sub, int level, uint64_t *out,
                            void *stream);
blb_status blb_mpc_to_ckks(const blb_params *params, blb_ct *ct, const uint64_t *x1, int w, void *ws,
                           size_t ws_bytes, void *stream);
/* The same for shares over Z_{2^w} with w <= 128 (the paper's ring-to-field runs on Z_{2^{l+40}},
 * l = 43 -> w = 83): x / x1 device [N][2] u64 little-endian words (x < 2^w). */
blb_status blb_share_to_rns128(const blb_params *params, const uint64_t *x, int w, int sub, int level, uint64_t *out,
                               void *stream);
blb_status blb_mpc_to_ckks128(const blb_params *params, blb_ct *ct, const uint64_t *x1, int w, void *ws,
                              size_t ws_bytes, void *stream);
/* Row f3, local fixed-point Decode of a share ("O(N log N) FFT ... extend the shares to
 * a larger ring and conduct local truncations"; App. C.4; reading C18).  Each MPC party
 * runs it on its own share; the outputs are additive shares of the real slots of Decode(m) scaled
 * by 2^-s_out (with plaintext scale Delta = 2^d: fixed-point precision d - s_out bits).
 * x: device [N][2] u64 = little-endian Z_{2^128} share of the coefficient vector.  Cooley-Tukey
 * network over Z_{2^128}[i] with twiddles W = round(2^ft zeta^{brv(m+i)}) and an arithmetic right
 * shift by ft after every twiddle product; slot j is read at the position of zeta^{5^j} (C3) and
 * shifted right by s_out.  y: device [N/2][2] u64.  ws: device scratch >= 48 N bytes.
 * 1 <= ft <= 52, 0 <= s_out <= 126, else BLB_E_INVALID_ARG; BLB_E_NOMEM (workspace). */
blb_status blb_share_decode(const blb_params *params, const uint64_t *x, int ft, int s_out, uint64_t *y, void *ws,
                            size_t ws_bytes, void *stream);
/* Row f3, local fixed-point Encode of a share (Alg. 2 line 1: each party "locally evaluates
 * the CKKS encoding"; P:684-685 / App. C.4: FFT with local truncations on the extended
 * ring; reading C20).  y: device [N/2][2] u64 = little-endian Z_{2^128} share of the real slot
 * vector (fixed point).  The value of slot j is placed at zeta^{5^j} and its conjugate (C3), the
 * Gentleman-Sande network over Z_{2^128}[i] runs with conj(W), W = round(2^ft zeta^{brv(m+i)}), and
 * an arithmetic right shift by ft after every twiddle product; coefficient k = Re_k >>_a s_out
 * (s_out = log N + f - log2 Delta for a share with f fractional bits).  x: device [N][2] u64, the
 * share of the integer coefficients of Encode.  ws >= 48 N bytes.  1 <= ft <= 52,
 * 0 <= s_out <= 126, else BLB_E_INVALID_ARG; BLB_E_NOMEM (workspace). */
blb_status blb_share_encode(const blb_params *params, const uint64_t *y, int ft, int s_out, uint64_t *x, void *ws,
                            size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------ */
/* ct-pt MatMul (rows a2-a6; C11 / C12; BSGS App. C.1)      */
/* ------------------------------------------------------------------ */
/* MHP output-column map (reading S16): heads padded to
 * H_p = next power of two >= heads; virtual column v = j*c + cc*H_p + h holds
 * source column h*d_h + j*g + cc (c = N/(2L), g = c / H_p, d_h = d / heads),
 * or -1 for padded heads.  map_out: host, capacity *len on entry; *len = the
 * map length on return. */
blb_status blb_mhp_column_map(int d, int heads, int L, int log_n, int32_t *map_out, int *len);

/* Plan Y = X W for X in R^{L x D_in} packed in ciphertexts at `level`.
 *  BLB_PACK_SPATIAL  (C11): input spatial-first: ciphertext b holds
 *     column b*c + tau at slots tau*L + i.  W: w_rows x w_cols row-major with
 *     w_rows = D_in; col_map (host, nullable) gives for each of D_out virtual
 *     output columns the source column of W or -1 (zero) -- e.g. the MHP map;
 *     NULL means D_out = w_cols, identity.
 *  BLB_PACK_DIAGONAL (C12, App. C.2): input = dense multi-head diagonal
 *     packing of Att_h (heads x L x d_h): block beta = d*heads + h holds
 *     Att_h[i, (i+d) mod d_h]; W = W_O with w_rows = heads*d_h, D_out = w_cols.
 *  BSGS: t = g*B + i over c = N/(2L) block rotations; all-zero diagonals are
 *  skipped (bit-neutral).  Output: ceil(D_out / c) spatial-first ciphertexts
 *  at level-1, scale = input scale (plaintexts are encoded at scale q_level). */
blb_status blb_matmul_plan_create(const blb_params *params, int L, int w_rows, int w_cols, blb_packing packing,
                                  int heads, const int32_t *col_map, int D_out, int bsgs_B, int level,
                                  blb_matmul_plan **out);
void blb_matmul_plan_destroy(blb_matmul_plan *plan);
/* Multi-GPU form: the plan restricted to the baby-step window
 * i in [i_first, i_first + i_count) of [0, B) (i_count = -1: to B).  Its plaintexts, baby steps and
 * MAC entries are those of the window; its giant steps are the whole plan's.  Windows of the ranks
 * partition [0, B): the MAC accumulators of all windows sum (exactly, mod q_l) to those of the
 * whole plan, so blb_ct_pt_matmul_acc on every rank + a cross-rank sum + blb_ct_pt_matmul_finish
 * at each output's owner gives the bits of blb_ct_pt_matmul at any number of ranks.
 * BLB_E_INVALID_ARG for a window outside [0, B). */
blb_status blb_matmul_plan_create_window(const blb_params *params, int L, int w_rows, int w_cols,
                                         blb_packing packing, int heads, const int32_t *col_map, int D_out,
                                         int bsgs_B, int level, int i_first, int i_count, blb_matmul_plan **out);

/* Host outputs (nullable): number of input / output ciphertexts, total
 * non-zero plaintexts, baby / giant rotations, B, G. */
blb_status blb_matmul_plan_info(const blb_matmul_plan *plan, int *n_in, int *n_out, int *n_pt, int *n_baby,
                                int *n_giant, int *B, int *G);
/* Distinct rotation steps (slots) the plan needs keys for; steps: host array of
 * capacity *n on entry. */
blb_status blb_matmul_plan_rotations(const blb_matmul_plan *plan, int32_t *steps, int *n);
/* Plaintexts owned by outputs [out_first, out_first+out_count). */
blb_status blb_matmul_pt_count(const blb_matmul_plan *plan, int out_first, int out_count, int *n_pt);

/* Bytes of the encoded plaintexts of outputs [out_first, out_first+out_count):
 * n_pt * sum_l w_l * N with w_l = 5 bytes per coefficient for limbs whose prime
 * is below 2^40 and 8 bytes otherwise (see blb_matmul_encode_weights).  Host out. */
blb_status blb_matmul_pt_bytes(const blb_matmul_plan *plan, int out_first, int out_count, size_t *bytes);

/* Offline precompute (row a0): build and encode the plaintexts of outputs
 * [out_first, out_first+out_count) from W (host, row-major w_rows x w_cols,
 * float64) into pt_dev (device, at least blb_matmul_pt_bytes bytes, 16-byte
 * aligned).  The buffer is opaque: it holds the NTT-form plaintexts in the
 * library's blocked MAC layout (per output: [limb][512-coefficient tile]
 * [plaintext][tile]) so that the MAC streams each output's weights
 * contiguously; a tile of a limb with prime < 2^40 is stored as 512 low 32-bit
 * words followed by 512 high bytes (the residues are < 2^40: a lossless 5-byte
 * packing of the dominant HBM stream), other limbs as 512 words.  W may be host or device memory
 * (unified addressing: per-layer re-encode from device-resident weights).  Synchronises. */
blb_status blb_matmul_encode_weights(const blb_matmul_plan *plan, const double *W, int out_first, int out_count,
                                     uint64_t *pt_dev, void *stream);

/* Config 5 (many layers on one GPU): the weights of a slice in
 * a compact, prime-independent form -- the rounded integer coefficients m_k = round(scale * iDFT(z))_k
 * of each plaintext (the first half of blb_matmul_encode_weights: slots, inverse embedding, rounding),
 * 5 bytes each (40-bit two's complement: per plaintext N low 32-bit words then N high bytes; opaque).
 * blb_matmul_coeff_bytes gives the size.  blb_matmul_encode_coeffs (offline, synchronises) fails with
 * BLB_E_OVERFLOW if some |m_k| >= 2^39.  blb_matmul_coeffs_to_pts (no synchronisation) expands them --
 * residues mod q_0..q_level, NTT, the blocked width-packed layout -- into pt_dev, bit-identical to
 * blb_matmul_encode_weights of the same W and slice.  coef_dev, pt_dev: device memory, caller-owned. */
blb_status blb_matmul_coeff_bytes(const blb_matmul_plan *plan, int out_first, int out_count, size_t *bytes);
blb_status blb_matmul_encode_coeffs(const blb_matmul_plan *plan, const double *W, int out_first, int out_count,
                                    void *coef_dev, void *stream);
blb_status blb_matmul_coeffs_to_pts(const blb_matmul_plan *plan, const void *coef_dev, int out_first, int out_count,
                                    uint64_t *pt_dev, void *stream);

size_t blb_matmul_workspace_bytes(const blb_matmul_plan *plan, int out_count);

/* Evaluate outputs [out_first, out_first+out_count) of the plan on the n_in
 * input ciphertexts (all at the plan level, NTT form): hoisted baby-step
 * rotations of every input, the MAC against pt_dev (the slice encoded for the
 * same output range), giant-step key switches, one rescale per output.
 * out[t] receives output ciphertext out_first + t ([2][level][N]). */
blb_status blb_ct_pt_matmul(const blb_matmul_plan *plan, const blb_keys *keys, const blb_ct *in, int n_in,
                            const uint64_t *pt_dev, int out_first, int out_count, blb_ct *out, void *ws,
                            size_t ws_bytes, void *stream);

/* The two phases of blb_ct_pt_matmul for a windowed plan (multi-GPU):
 * _acc: hoisted ModUp of the inputs, the window's baby-step rotations and the MAC of its
 *   plaintexts (pt_dev encoded for ALL outputs of the windowed plan) into acc_out, device
 *   [n_out][G][2][level+1][N] u64 (NTT form, residues < q_i; entries the window does not touch are
 *   0).  Needs the window's baby-step keys.  ws: blb_matmul_workspace_bytes(plan, 0).
 * _finish: outputs [out_first, out_first + out_count) from acc_in, device
 *   [out_count][G][2][level+1][N] u64 holding the SUM over the windows (u64 sums of residues,
 *   < 2^64, reduced mod q_i here): giant steps in Q_l u P, the fused ModDown + rescale (C11, C17),
 *   out[t] at level-1 with scale `scale` (the input scale).  Needs the giant-step keys.
 *   ws: blb_matmul_workspace_bytes(plan, out_count).  acc_in is not modified. */
/* Row f4 (throughput variant): n_batch independent input sets in[b * n_in .. (b+1) * n_in) against the
 * SAME plaintexts -- each set's ModUp / baby steps / giant steps as blb_ct_pt_matmul, but ONE
 * weight-stationary MAC whose every staged plaintext tile feeds two input sets (the plaintext stream,
 * the step's dominant HBM traffic, is read once per pair of sets).  out[b * out_count + t] receives
 * output out_first + t of set b, bit-identical to blb_ct_pt_matmul on that set alone.  ws: n_batch times
 * blb_matmul_workspace_bytes(plan, out_count).  Full (non-windowed) plans only. */
blb_status blb_ct_pt_matmul_batch(const blb_matmul_plan *plan, const blb_keys *keys, const blb_ct *in, int n_in,
                                  int n_batch, const uint64_t *pt_dev, int out_first, int out_count, blb_ct *out,
                                  void *ws, size_t ws_bytes, void *stream);
blb_status blb_ct_pt_matmul_acc(const blb_matmul_plan *plan, const blb_keys *keys, const blb_ct *in, int n_in,
                                const uint64_t *pt_dev, uint64_t *acc_out, void *ws, size_t ws_bytes, void *stream);
blb_status blb_ct_pt_matmul_finish(const blb_matmul_plan *plan, const blb_keys *keys, const uint64_t *acc_in,
                                   int out_first, int out_count, double scale, blb_ct *out, void *ws, size_t ws_bytes,
                                   void *stream);

/* ------------------------------------------------------------------ */
/* row f2: other HE operators of the fused blocks                       */
/* ------------------------------------------------------------------ */
size_t blb_f2_workspace_bytes(const blb_params *params, int level);

/* ct (x) ct with relinearisation (C9; ewmul_cc of Table 2, e.g. the squarings of
 * Softmax's negExp (1 + x/2^6)^{2^6}, and GeLU's x^2 / x^4):
 * out = (d0, d1) + KeySwitch(d2, rlk), same level, scale a.scale * b.scale (the
 * caller rescales).  Needs the relinearisation key (Galois element 0). */
blb_status blb_mul_relin(const blb_params *params, const blb_keys *keys, const blb_ct *a, const blb_ct *b,
                         blb_ct *out, void *ws, size_t ws_bytes, void *stream);

/* Batched ewmul_cc (+ rescale): out[t] = mul_relin(a[t], b[t]) (then rescaled when rescale != 0),
 * t < n -- one tensor launch, one ModUp and one key-switch batch (the relinearisation key is read
 * once per tile for the whole batch), one rescale batch; the per-pair bits of blb_mul_relin +
 * blb_rescale.  All operands at one level (BLB_E_LEVEL otherwise); out[t] [2][level(-1)][N];
 * ws: blb_mul_relin_batch_workspace_bytes(level, n). */
size_t blb_mul_relin_batch_workspace_bytes(const blb_params *params, int level, int n);
blb_status blb_mul_relin_batch(const blb_params *params, const blb_keys *keys, const blb_ct *a, const blb_ct *b, int n,
                               int rescale, blb_ct *out, void *ws, size_t ws_bytes, void *stream);

/* Batched ewmul_cp + rescale: out[t] = rescale(in[t] (x) pt[t]) for t < n (pt[t]: device
 * [level+1][N] NTT plaintexts, host array of pointers; pt_scale[t] their scales, host), all inputs at
 * one level >= 1 -- the per-ciphertext bits of blb_mul_pt + blb_rescale in one product launch and
 * one rescale batch.  out[t] [2][level][N], scale (in.scale * pt_scale) / q_level.
 * ws: blb_mul_pt_rescale_batch_workspace_bytes(level, n). */
size_t blb_mul_pt_rescale_batch_workspace_bytes(const blb_params *params, int level, int n);
blb_status blb_mul_pt_rescale_batch(const blb_params *params, const blb_ct *in, const uint64_t *const *pt,
                                    const double *pt_scale, int n, blb_ct *out, void *ws, size_t ws_bytes, void *stream);

/* Rotate-and-sum of BLB's summation operator (Table 3) on a
 * spatial-first ciphertext with L rows and D (power of two) columns:
 * m^0 = in, m^i = m^{i-1} + Rot_l^{2^{i-1} L}(m^{i-1}), out = m^{log2 D}: log2 D
 * rotations, no multiplication -- the fused form (Table 3 "BLB (w/ fusion)": the
 * result is replicated across the D column blocks, ready for a following scalar
 * operator).  The unfused form multiplies by the [1..1, 0..0] mask (blb_mul_pt).
 * blb_broadcast is the same with right rotations (m_r).  out may not alias in. */
blb_status blb_rotate_sum(const blb_params *params, const blb_keys *keys, const blb_ct *in, int L, int D,
                          blb_ct *out, void *ws, size_t ws_bytes, void *stream);
blb_status blb_broadcast(const blb_params *params, const blb_keys *keys, const blb_ct *in, int L, int D,
                         blb_ct *out, void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------ */
/* ct-ct MatMul Q_h K_h^T for all heads (row a7; sec. 5.1,    */
/* App. C.1; reading C13)                                   */
/* ------------------------------------------------------------------ */
typedef struct blb_qk_plan blb_qk_plan;

/* Plan C_h = Q_h K_h^T for `heads` heads of L x d_h, operands in multi-head
 * packing: heads padded to H_p = next power of two, g = N/(2 L H_p)
 * columns per head per ciphertext, J = ceil(d_h / g) ciphertexts per operand;
 * block c*H_p + h of ciphertext j holds column j*g + c of head h (this is the
 * layout blb_mhp_column_map gives the QKV ct-pt MatMul outputs).
 * BSGS: t = u*B + i, B*G = L, g | B (bsgs_B = 0 selects B = g).  Consumes 3
 * levels: operands at `level` >= 3, outputs at level-3.  Output o (< L/g) is
 * diagonal-packed: block e*H_p + h, row p holds C_h[p, (p + o*g + e) mod L]. */
blb_status blb_qk_plan_create(const blb_params *params, int L, int heads, int d_h, int bsgs_B, int level,
                              blb_qk_plan **out);
void blb_qk_plan_destroy(blb_qk_plan *plan);
/* Host outputs (nullable): J, number of outputs, g, B, G, rotations, mask plaintexts. */
blb_status blb_qk_plan_info(const blb_qk_plan *plan, int *J, int *n_out, int *g, int *B, int *G, int *n_rotations,
                            int *n_masks);
/* Rotation steps needed (the relinearisation key, Galois element 0, is needed too). */
blb_status blb_qk_plan_rotations(const blb_qk_plan *plan, int32_t *steps, int *n);
/* Offline precompute (row a0): encode all mask plaintexts into `masks` (device,
 * blb_qk_mask_bytes bytes; an opaque buffer for blb_ct_ct_qk: the residues of limbs
 * whose prime is below 2^41 are stored as IEEE doubles).  Synchronises. */
size_t blb_qk_mask_bytes(const blb_qk_plan *plan);
blb_status blb_qk_encode_masks(const blb_qk_plan *plan, uint64_t *masks, void *stream);
size_t blb_qk_workspace_bytes(const blb_qk_plan *plan);
/* Evaluate: Q[0..J), K[0..J) at the plan level -> out[0..L/g) at level-3.
 * Scale of every output = (Q.scale * K.scale) / q_{level-1} (masks are encoded at
 * the scale of the prime their rescale drops). */
blb_status blb_ct_ct_qk(const blb_qk_plan *plan, const blb_keys *keys, const blb_ct *Q, const blb_ct *K, int J,
                        const uint64_t *masks, blb_ct *out, void *ws, size_t ws_bytes, void *stream);

/* Multi-GPU form: the plan restricted to the baby-index window
 * i in [i_first, i_first + i_count) of [0, B) (i_count = -1: to B).  Windows of the ranks
 * partition [0, B); the step-3 accumulators A_{u,w,f} (reading C13, before their ModDown +
 * rescale) of all windows sum exactly (mod each prime of Q_{level-2} u P) to those of the whole
 * plan, so blb_ct_ct_qk_acc on every rank + a cross-rank sum + blb_ct_ct_qk_finish at each
 * output's owner gives the bits of blb_ct_ct_qk at any number of ranks. */
blb_status blb_qk_plan_create_window(const blb_params *params, int L, int heads, int d_h, int bsgs_B, int level,
                                     int i_first, int i_count, blb_qk_plan **out);
/* Bytes of the accumulator array: [NA][2][level-1+np][N] u64, accumulators sorted by output. */
size_t blb_qk_acc_bytes(const blb_qk_plan *plan);
/* Accumulator slots [*slot_first, *slot_first + *slot_count) that outputs [out_first, +out_count)
 * read (host outputs). */
blb_status blb_qk_acc_range(const blb_qk_plan *plan, int out_first, int out_count, int *slot_first, int *slot_count);
/* Phase A: the window's stages 1-3 (K'_i for i in the window, every Q_u, products, relinearisation,
 * step-3 rotations and masks) into acc_out (device, blb_qk_acc_bytes; residues < q_i).
 * Phase B: outputs [out_first, +out_count) from acc_in = the cross-rank SUM of the accumulator
 * slots blb_qk_acc_range gives (u64 sums < 2^64 of residues, reduced here; acc_in points at the
 * first of those slots): ModDown + rescale (C17), deferred giant rotations, one ModDown per output.
 * scale_q / scale_k: the operands' scales.  Both need the plan's keys; ws: blb_qk_workspace_bytes. */
blb_status blb_ct_ct_qk_acc(const blb_qk_plan *plan, const blb_keys *keys, const blb_ct *Q, const blb_ct *K, int J,
                            const uint64_t *masks, uint64_t *acc_out, void *ws, size_t ws_bytes, void *stream);
blb_status blb_ct_ct_qk_finish(const blb_qk_plan *plan, const blb_keys *keys, const uint64_t *acc_in, int out_first,
                               int out_count, double scale_q, double scale_k, blb_ct *out, void *ws, size_t ws_bytes,
                               void *stream);

#ifdef __cplusplus
}
#endif
#endif /* BLB_H */
