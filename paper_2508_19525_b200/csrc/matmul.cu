// matmul.cu -- the ct-pt MatMul protocol of BLB on sm_100a (rows a2-a6).
//
// C11 (spatial-first input, BOLT's protocol as referenced at P:361 / P:511 /
// P:515) and C12 (diagonal input for W_O, App. C.2), both with
// BSGS (App. C.1):
//     Y_b' = sum_g Rot^{gBL}( sum_b sum_i P_{b,b',g,i} (.) Rot^{iL}(X_b) ),
//     P_{b,b',g,i} = Rot^{-gBL}(Pi_{b,b',gB+i}),
// Pi block tau = W[b c + (tau + t) mod c, b' c + tau] (C11) or the
// "duplicated spatial-first" vector w[i] = W_O[h d_h + (i+d) mod d_h, col]
// with (d, h) = divmod(b c + (tau+t) mod c, heads) (C12).
//
// Hot path of one call:
//   1. ModUp of every input c1, once (hoisting, C8);
//   2. all baby-step rotations of all inputs, batched 32 key switches per
//      launch group (inner product with the automorphism as a load gather);
//   3. the MAC: acc[b',g] = sum_{b,i} P (.) R[b][i], one launch, 128-bit lazy
//      accumulation, plaintexts streamed from HBM exactly once, R re-read from
//      L2 (the output index is the fastest grid dimension);
//   4. giant-step key switches of acc[b', g >= 1] and the sum over g;
//   5. one rescale per output.
#include <algorithm>
#include <map>
#include <type_traits>
#include "blb_internal.cuh"

extern "C" u64 blbh_shoup(u64 w, u64 q);

struct blb_matmul_plan {
    const blb_params *P;
    int L, n, c, w_rows, w_cols, nblk_in, D_out, n_in, n_out, B, G, level, packing, heads, dh;
    int i_first = 0, i_count = 0;                       // baby-step window of this rank (section 8(e))
    std::vector<int32_t> col_map;                       // D_out entries, -1 = zero column
    std::vector<int> ent_start;                         // CSR over (b', g): n_out*G + 1
    std::vector<int> ent_b, ent_i;                      // entries in plan order
    std::vector<std::vector<int>> baby;                 // per input: i >= 1 used
    std::vector<std::vector<int>> giant;                // per output: g >= 1 used
    std::vector<int32_t> rot_steps;
    std::vector<char> same_next;                        // entry list of (b', g) == that of the next one
    int *d_ent = nullptr;                               // device: (b * B + i) per entry
    int *d_ent_start = nullptr;                         // device copy of ent_start
    int32_t *d_col_map = nullptr;
};

namespace {
constexpr int kTB = 256;
#ifndef BLB_MAC_STG
#define BLB_MAC_STG 4
#endif
#ifndef BLB_MAC_MINB
#define BLB_MAC_MINB 3
#endif
#ifndef BLB_MAC_P
#define BLB_MAC_P 2   // outputs (b', g) per CTA sharing each staged R tile (4 measured slower)
#endif
#ifndef BLB_MAC_STGP
#define BLB_MAC_STGP 4   // ring stages for the width-packed limbs (5 measured equal: profiles/r2_mac_ring_depth_ab.log)
#endif

// Build the slot vectors of entries [e0, e0 + cnt) (plan order) into slots[cnt][n].
struct PlanDev {
    int L, n, c, B, G, w_rows, w_cols, nblk_in, D_out, packing, heads, dh;
};
__global__ void k_build_slots(PlanDev pd, const int *ent_bi, const int *ent_o, int e0, const double *W,
                              const int32_t *col_map, double *slots) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    const int e = blockIdx.y;
    if (s >= pd.n) return;
    const int bi = ent_bi[e0 + e];
    const int b = bi / pd.B, i = bi % pd.B;
    const int o = ent_o[e0 + e];  // b' * G + g
    const int bp = o / pd.G, g = o % pd.G;
    const int t = g * pd.B + i;
    // P[s] = Pi[(s - gBL) mod n]
    int sp = s - g * pd.B * pd.L;
    sp %= pd.n;
    if (sp < 0) sp += pd.n;
    const int tau = sp / pd.L, row = sp - tau * pd.L;
    const int r = b * pd.c + (tau + t) % pd.c;
    const int col = bp * pd.c + tau;
    double v = 0.0;
    if (col < pd.D_out) {
        if (pd.packing == BLB_PACK_SPATIAL) {
            const int src = col_map[col];
            if (r < pd.w_rows && src >= 0) v = W[(long long)r * pd.w_cols + src];
        } else {
            if (r < pd.nblk_in) {
                const int d = r / pd.heads, h = r % pd.heads;
                v = W[(long long)(h * pd.dh + (row + d) % pd.dh) * pd.w_cols + col];
            }
        }
    }
    slots[(long long)e * pd.n + s] = v;
}

// acc[o][p][l][x] = sum_{e in o} pt[pt_e][l][x] * R[r_e][p][l][x]   (o = local output)
// pt_e = ent_pt[e] (or e - e_base when ent_pt == nullptr: plaintexts stored in entry order).
// 1-D grid: bid = (l * n_tiles + tile) * n_o + o  -> the output index varies
// fastest, so concurrent CTAs share the same R tile through L2.
__global__ void __launch_bounds__(kTB) k_mac(const u64 *__restrict__ pt, const u64 *__restrict__ R,
                                             u64 *__restrict__ acc, const int *__restrict__ ent_r,
                                             const int *__restrict__ ent_pt, const int *__restrict__ ent_start,
                                             int o0, int e_base, int n_o, int k, int kq, int Kfull, int logN,
                                             Primes pr) {
    const int N = 1 << logN;
    const int n_tiles = N / (2 * kTB);
    int bid = blockIdx.x;
    const int o = bid % n_o;
    bid /= n_o;
    const int tile = bid % n_tiles;
    const int l = bid / n_tiles;
    const int x = tile * 2 * kTB + 2 * threadIdx.x;
    const long long kN = (long long)k * N;
    const int e_lo = ent_start[o0 + o], e_hi = ent_start[o0 + o + 1];
    const long long lx = (long long)l * N + x;
    // limbs l >= kq are the special primes of the extended basis Q_l u P (double hoisting)
    const ModConst &mc = pr.m[l < kq ? l : Kfull + (l - kq)];
    u64 *out = acc + (long long)o * 2 * kN + lx;
    if (mc.q < (1ull << 41)) {
        // limbs below 2^41: masks and rotations stored as doubles (blb_qk_encode_masks,
        // KsJob::out_f64), all four sums on the grid-split FP64 accumulator
        const double qd = (double)mc.q, qinv = 1.0 / qd;
        AccG a00, a01, a10, a11;
        a00.zero(); a01.zero(); a10.zero(); a11.zero();
        int cnt = 0;
#pragma unroll 4
        for (int e = e_lo; e < e_hi; e++) {
            const int bi = ent_r[e];
            const int pe = ent_pt ? ent_pt[e] : e - e_base;
            const double2 pv = *reinterpret_cast<const double2 *>(pt + (long long)pe * kN + lx);
            const double2 r0 = *reinterpret_cast<const double2 *>(R + (long long)bi * 2 * kN + lx);
            const double2 r1 = *reinterpret_cast<const double2 *>(R + ((long long)bi * 2 + 1) * kN + lx);
            a00.macd(pv.x, r0.x); a01.macd(pv.y, r0.y);
            a10.macd(pv.x, r1.x); a11.macd(pv.y, r1.y);
            if (++cnt == 512) {  // AccG bound: <= 512 products between folds
                a00.fold(qd, qinv); a01.fold(qd, qinv); a10.fold(qd, qinv); a11.fold(qd, qinv);
                cnt = 0;
            }
        }
        *reinterpret_cast<ulonglong2 *>(out) = make_ulonglong2(a00.reduce(qd, qinv), a01.reduce(qd, qinv));
        *reinterpret_cast<ulonglong2 *>(out + kN) = make_ulonglong2(a10.reduce(qd, qinv), a11.reduce(qd, qinv));
        return;
    }
    Acc128 a00, a01, a10, a11;  // [poly][coefficient]
    a00.zero(); a01.zero(); a10.zero(); a11.zero();
#pragma unroll 4
    for (int e = e_lo; e < e_hi; e++) {
        const int bi = ent_r[e];
        const int pe = ent_pt ? ent_pt[e] : e - e_base;
        const ulonglong2 pv = *reinterpret_cast<const ulonglong2 *>(pt + (long long)pe * kN + lx);
        const ulonglong2 r0 = *reinterpret_cast<const ulonglong2 *>(R + (long long)bi * 2 * kN + lx);
        const ulonglong2 r1 = *reinterpret_cast<const ulonglong2 *>(R + ((long long)bi * 2 + 1) * kN + lx);
        a00.mac(pv.x, r0.x); a01.mac(pv.y, r0.y);
        a10.mac(pv.x, r1.x); a11.mac(pv.y, r1.y);
    }
    *reinterpret_cast<ulonglong2 *>(out) = make_ulonglong2(a00.reduce(mc), a01.reduce(mc));
    *reinterpret_cast<ulonglong2 *>(out + kN) = make_ulonglong2(a10.reduce(mc), a11.reduce(mc));
}

// Weight MAC (row a3) on the blocked, width-packed plaintext layout written by
// blb_matmul_encode_weights.  Plaintext residues are uniform in [0, q), so a limb whose prime is
// below 2^40 (four of the five BERT chain primes) is stored in 5 bytes per coefficient as two planes
// per 512-coefficient tile -- 512 low 32-bit words then 512 high bytes (2560 B instead of 4096 B);
// other limbs keep 8 bytes.  The plaintext stream is the dominant HBM traffic of the step, and the
// split is exactly the (a0, a1) split the Acc41 accumulator multiplies with.  Layout (bytes): output
// o's plaintexts start at (e_lo(o) - e_base) * bpp (bpp = sum_l w_l N); inside, [limb l][tile][entry]
// [512 * w_l bytes], limb l at n_e N sum_{l' < l} w_l'.
//
// Multi-output kernel: a CTA accumulates kMacP outputs (b', g) that share the same (b, i) entry list
// (so the same R tiles) for one (tile, limb): per pipeline stage one entry = kMacP plaintext tiles +
// the two R tiles, staged by a producer warp with cp.async.bulk into a shared-memory ring (mbarrier
// completion); 8 consumer warps multiply.  R is staged once per kMacP outputs.  kMacP = 1 is the
// general fallback (any plan).
struct PtLayout {
    int w[BLB_MAXP];         // bytes per coefficient of limb l (5 = packed, 8 = plain)
    long long loff[BLB_MAXP];  // sum_{l' < l} w_l' * N (times n_e: the limb offset inside an output block)
    long long bpp;           // bytes per plaintext = sum_l w_l N
};
// Ring geometry: a stage holds PP plaintext tiles (512 * w bytes each) + the two R tiles (4096 bytes
// each).  Packed limbs (w = 5) run STGP stages, 8-byte limbs STG stages, in the same shared memory
// (the packed stages are smaller, so the deeper ring keeps more plaintext bytes in flight).
template <int PP>
__host__ __device__ constexpr unsigned mac4_stage_bytes(int w) { return (unsigned)(PP * 512 * w + 2 * 4096); }
template <int PP, int STG, int STGP>
__host__ __device__ constexpr size_t mac4_ring_bytes() {
    return (size_t)(STG * mac4_stage_bytes<PP>(8) > STGP * mac4_stage_bytes<PP>(5) ? STG * mac4_stage_bytes<PP>(8)
                                                                                    : STGP * mac4_stage_bytes<PP>(5));
}
template <int PP, int STG, int STGP>
constexpr size_t mac4_smem() { return mac4_ring_bytes<PP, STG, STGP>() + 2 * (STG > STGP ? STG : STGP) * 8; }

// SPLIT41 (q < 2^41): every product on the grid-split FP64 accumulator (AccG, FP64 pipe, one
// reduction per output); otherwise (60-bit limbs) Acc128 on the integer pipe, folded every 64.
// The ring geometry is compile-time (tile TB bytes, NST stages) and the stage loop is unrolled by
// NST, so every ring access is a shared load at a constant offset from one per-thread base and the
// barrier addresses are constants: the loop body is the multiply-accumulate and little else.
template <bool SPLIT41, bool PACKED, int kMacP, int NST>
__device__ __forceinline__ void mac4_consume(const unsigned char *ring, uint64_t *full, uint64_t *empty, int n_e, int nP,
                                             u64 *const *outs, long long kN, const ModConst &mc) {
    using A = typename std::conditional<SPLIT41, AccG, Acc128>::type;
    constexpr unsigned TB = PACKED ? 5u * 512u : 8u * 512u;   // bytes of one plaintext tile
    constexpr unsigned SB = (unsigned)kMacP * TB + 2u * 4096u;  // bytes of one stage
    const double qd = (double)mc.q, qinv = 1.0 / qd;
    A a00[kMacP], a01[kMacP], a10[kMacP], a11[kMacP];
#pragma unroll
    for (int j = 0; j < kMacP; j++) { a00[j].zero(); a01[j].zero(); a10[j].zero(); a11[j].zero(); }
    const int t = threadIdx.x;
    const unsigned full0 = smem_u32(full), empty0 = smem_u32(empty);
    const unsigned char *rt_t = ring + kMacP * TB + 16 * t;               // R tiles: c0, then c1 at +4096
    const unsigned char *lo_t = ring + (PACKED ? 8 * t : 16 * t);        // plaintext words (low planes)
    const unsigned char *hi_t = ring + 2048 + 2 * t;                      // packed high bytes
    auto stage = [&](int slot, unsigned phase) {
        mbar_wait_sa(full0 + 8u * slot, phase);
        const unsigned off = (unsigned)slot * SB;
        if constexpr (SPLIT41) {
            // R limbs below 2^41 are stored as doubles by their producers (KsJob::out_f64,
            // k_copy_ct_f64); plaintext values are converted once (shared by c0 and c1)
            const double2 r0 = *reinterpret_cast<const double2 *>(rt_t + off);
            const double2 r1 = *reinterpret_cast<const double2 *>(rt_t + off + 4096);
            const double R0x = r0.x, R0y = r0.y, R1x = r1.x, R1y = r1.y;
#pragma unroll
            for (int j = 0; j < kMacP; j++) {
                // unconditional (slot j >= nP holds stale data, its sums are never stored): no joins
                double Px, Py;
                if constexpr (PACKED) {  // high byte spliced under the 2^52 exponent with one PRMT
                    const uint2 lo = *reinterpret_cast<const uint2 *>(lo_t + off + j * TB);
                    const unsigned hi = *reinterpret_cast<const unsigned short *>(hi_t + off + j * TB);
                    Px = __dsub_rn(__hiloint2double((int)__byte_perm(hi, 0x43300000u, 0x7650), (int)lo.x), 4503599627370496.0);
                    Py = __dsub_rn(__hiloint2double((int)__byte_perm(hi, 0x43300000u, 0x7651), (int)lo.y), 4503599627370496.0);
                } else {
                    const ulonglong2 pv = *reinterpret_cast<const ulonglong2 *>(lo_t + off + j * TB);
                    Px = AccF64::u2d(pv.x);
                    Py = AccF64::u2d(pv.y);
                }
                a00[j].macd(Px, R0x); a01[j].macd(Py, R0y);
                a10[j].macd(Px, R1x); a11[j].macd(Py, R1y);
            }
        } else {
            const ulonglong2 r0 = *reinterpret_cast<const ulonglong2 *>(rt_t + off);
            const ulonglong2 r1 = *reinterpret_cast<const ulonglong2 *>(rt_t + off + 4096);
#pragma unroll
            for (int j = 0; j < kMacP; j++) {
                if (j < nP) {
                    const ulonglong2 pv = *reinterpret_cast<const ulonglong2 *>(lo_t + off + j * TB);
                    a00[j].mac(pv.x, r0.x); a01[j].mac(pv.y, r0.y);
                    a10[j].mac(pv.x, r1.x); a11[j].mac(pv.y, r1.y);
                }
            }
        }
        // every consumer thread arrives (count kTB) once its own reads of the slot are done
        mbar_arrive_sa(empty0 + 8u * slot);
    };
    auto fold = [&]() {
#pragma unroll
        for (int j = 0; j < kMacP; j++) {
            accf(a00[j], mc, qd, qinv); accf(a01[j], mc, qd, qinv);
            accf(a10[j], mc, qd, qinv); accf(a11[j], mc, qd, qinv);
        }
    };
    // folds at chunk boundaries (Acc128: every 64 products < 2^126; AccG: every 512, s < 2^93,
    // l < 2^48); chunks are whole ring rounds, so stage s of a round uses slot s (constant)
    constexpr int kFold = ((SPLIT41 ? 512 : 64) / NST) * NST;
    const int n_full = n_e - n_e % NST;
    unsigned phase = 0;
    int s = 0;
    while (s < n_full) {
        const int s1 = n_full - s < kFold ? n_full : s + kFold;
        for (; s < s1; s += NST) {
#pragma unroll
            for (int i = 0; i < NST; i++) stage(i, phase);
            phase ^= 1u;
        }
        if (s < n_e && s % kFold == 0) fold();
    }
    for (int i = 0; s < n_e; s++, i++) stage(i, phase);  // last partial round (< NST stages)
#pragma unroll
    for (int j = 0; j < kMacP; j++) {
        if (j < nP) {
            u64 *out = outs[j] + 2 * t;
            *reinterpret_cast<ulonglong2 *>(out) = make_ulonglong2(accr(a00[j], mc, qd, qinv), accr(a01[j], mc, qd, qinv));
            *reinterpret_cast<ulonglong2 *>(out + kN) =
                make_ulonglong2(accr(a10[j], mc, qd, qinv), accr(a11[j], mc, qd, qinv));
        }
    }
}

template <int kMacP, int kM4Stages, int MINB, int kM4StagesP = kM4Stages>
__global__ void __launch_bounds__(kTB + 32, MINB) k_mac_tma4(const unsigned char *__restrict__ pt, const u64 *__restrict__ R,
                                                       u64 *__restrict__ acc, const int *__restrict__ ent_r,
                                                       const int *__restrict__ ent_start, int o0, int e_base, int n_o,
                                                       int k, int logN, Primes pr, PtLayout lay, int skip_l) {
    constexpr int kMaxStg = kM4Stages > kM4StagesP ? kM4Stages : kM4StagesP;
    extern __shared__ __align__(128) unsigned char smraw[];
    unsigned char *ring = smraw;
    uint64_t *full = reinterpret_cast<uint64_t *>(smraw + mac4_ring_bytes<kMacP, kM4Stages, kM4StagesP>());
    uint64_t *empty = full + kMaxStg;
    const int N = 1 << logN;
    const int n_tiles = N / (2 * kTB);
    const int n_grp = (n_o + kMacP - 1) / kMacP;
    int bid = blockIdx.x;
    const int og = bid % n_grp;
    bid /= n_grp;
    const int tile = bid % n_tiles;
    const int l = bid / n_tiles;
    if (l == skip_l) return;  // that limb runs in k_mac_q0 (whole CTA exits before any barrier)
    const int oa = og * kMacP, nP = min(kMacP, n_o - oa);
    const long long kN = (long long)k * N;
    const int e_lo = ent_start[o0 + oa], n_e = ent_start[o0 + oa + 1] - e_lo;
    const long long lx0 = (long long)l * N + tile * 2 * kTB;
    const int w = lay.w[l];
    const unsigned tb = 512u * (unsigned)w;  // bytes of one plaintext tile of this limb
    const int nst = w == 5 ? kM4StagesP : kM4Stages;
    const unsigned stage_bytes = (unsigned)kMacP * tb + 2u * 4096u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kTB);  // one arrival per consumer thread (mac4_consume)
        }
        mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x >= kTB) {  // producer warp
        if (threadIdx.x == kTB) {
            const unsigned char *pp[kMacP];
#pragma unroll
            for (int j = 0; j < kMacP; j++)
                pp[j] = pt + (long long)(ent_start[o0 + oa + (j < nP ? j : 0)] - e_base) * lay.bpp +
                        (long long)n_e * lay.loff[l] + (long long)tile * n_e * tb;
            int slot = 0;
            unsigned phase = 0;  // parity of the empty-barrier round being waited for
#ifndef BLB_MAC_L2HINT
#define BLB_MAC_L2HINT 1
#endif
            const uint64_t pol_pt = l2_policy_evict_first(), pol_r = l2_policy_evict_last();
            for (int s = 0; s < n_e; s++) {
                if (s >= nst) {
                    mbar_wait(&empty[slot], phase);
                    fence_proxy_async_smem();
                }
                unsigned char *stb = ring + (size_t)slot * stage_bytes;
                mbar_expect_tx(&full[slot], (unsigned)nP * tb + 2u * 4096u);
                const int bi = ent_r[e_lo + s];
                if (BLB_MAC_L2HINT) {  // plaintexts are read once: evict first; R tiles are re-read by other CTAs
                    for (int j = 0; j < nP; j++)
                        bulk_g2s_hint(stb + j * tb, pp[j] + (long long)s * tb, tb, &full[slot], pol_pt);
                    bulk_g2s_hint(stb + kMacP * tb, R + (long long)bi * 2 * kN + lx0, 4096, &full[slot], pol_r);
                    bulk_g2s_hint(stb + kMacP * tb + 4096, R + ((long long)bi * 2 + 1) * kN + lx0, 4096, &full[slot],
                                  pol_r);
                } else {
                    for (int j = 0; j < nP; j++) bulk_g2s(stb + j * tb, pp[j] + (long long)s * tb, tb, &full[slot]);
                    bulk_g2s(stb + kMacP * tb, R + (long long)bi * 2 * kN + lx0, 4096, &full[slot]);
                    bulk_g2s(stb + kMacP * tb + 4096, R + ((long long)bi * 2 + 1) * kN + lx0, 4096, &full[slot]);
                }
                if (++slot == nst) {
                    slot = 0;
                    if (s >= nst) phase ^= 1u;
                }
            }
        }
        return;
    }
    u64 *outs[kMacP];
#pragma unroll
    for (int j = 0; j < kMacP; j++) outs[j] = acc + (long long)(oa + (j < nP ? j : 0)) * 2 * kN + lx0;
    const ModConst &mc = pr.m[l];
    if (w == 5) mac4_consume<true, true, kMacP, kM4StagesP>(ring, full, empty, n_e, nP, outs, kN, mc);
    else if (mc.q < (1ull << 41)) mac4_consume<true, false, kMacP, kM4Stages>(ring, full, empty, n_e, nP, outs, kN, mc);
    else mac4_consume<false, false, kMacP, kM4Stages>(ring, full, empty, n_e, nP, outs, kN, mc);
}

template <int PP, int STG, int MINB, int STGP = STG>
static void launch_mac4(const unsigned char *pt, const u64 *R, u64 *acc, const int *ent_r, const int *ent_start, int o0,
                        int e_base, int n_o, int k, int logN, const Primes &pr, int n_tiles, const PtLayout &lay,
                        cudaStream_t st, int skip_l = -1) {
    constexpr size_t smem = mac4_smem<PP, STG, STGP>();
    blb_smem_optin(k_mac_tma4<PP, STG, MINB, STGP>, smem);
    const size_t n_grp = (size_t)(n_o + PP - 1) / PP;
    k_mac_tma4<PP, STG, MINB, STGP><<<(unsigned)(n_grp * n_tiles * k), kTB + 32, smem, st>>>(pt, R, acc, ent_r, ent_start,
                                                                                      o0, e_base, n_o, k, logN, pr, lay,
                                                                                      skip_l);
}

// The weight MAC of one 8-byte limb whose prime is >= 2^41 (the 60-bit q0) as its own kernel: 512
// consumers with ONE coefficient each, so the four sums of a thread (2 outputs x c0 / c1) fit the
// carry-save accumulator Acc60W (8 registers each, 10 instructions per product instead of Acc128's
// 64 x 64 -> 128-bit multiply and compare-carried add); launched on the auxiliary stream beside the
// FP64-pipe kernel of the other limbs (the two load different pipes).
#ifndef BLB_Q0_STG
#define BLB_Q0_STG 4
#endif
constexpr int kQ0Cons = 512, kQ0Stages = BLB_Q0_STG;
constexpr unsigned kQ0StageBytes = 2u * 4096u + 2u * 4096u;  // 2 plaintext tiles + (c0, c1) R tiles
__global__ void __launch_bounds__(kQ0Cons + 32, 2) k_mac_q0(const unsigned char *__restrict__ pt, const u64 *__restrict__ R,
                                                           u64 *__restrict__ acc, const int *__restrict__ ent_r,
                                                           const int *__restrict__ ent_start, int o0, int e_base, int n_o,
                                                           int k, int l, int logN, Primes pr, PtLayout lay) {
    extern __shared__ __align__(128) unsigned char smraw[];
    unsigned char *ring = smraw;
    uint64_t *full = reinterpret_cast<uint64_t *>(smraw + (size_t)kQ0Stages * kQ0StageBytes);
    uint64_t *empty = full + kQ0Stages;
    const int N = 1 << logN;
    const int n_grp = (n_o + 1) / 2;
    const int og = blockIdx.x % n_grp, tile = blockIdx.x / n_grp;
    const int oa = og * 2, nP = min(2, n_o - oa);
    const long long kN = (long long)k * N;
    const int e_lo = ent_start[o0 + oa], n_e = ent_start[o0 + oa + 1] - e_lo;
    const long long lx0 = (long long)l * N + tile * 512;
    constexpr unsigned tb = 4096u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kQ0Stages; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kQ0Cons);
        }
        mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x >= kQ0Cons) {  // producer warp
        if (threadIdx.x == kQ0Cons) {
            const unsigned char *pp[2];
            for (int j = 0; j < 2; j++)
                pp[j] = pt + (long long)(ent_start[o0 + oa + (j < nP ? j : 0)] - e_base) * lay.bpp +
                        (long long)n_e * lay.loff[l] + (long long)tile * n_e * tb;
            const uint64_t pol_pt = l2_policy_evict_first(), pol_r = l2_policy_evict_last();
            int slot = 0;
            unsigned phase = 0;
            for (int s = 0; s < n_e; s++) {
                if (s >= kQ0Stages) {
                    mbar_wait(&empty[slot], phase);
                    fence_proxy_async_smem();
                }
                unsigned char *stb = ring + (size_t)slot * kQ0StageBytes;
                mbar_expect_tx(&full[slot], (unsigned)nP * tb + 2u * 4096u);
                for (int j = 0; j < nP; j++) bulk_g2s_hint(stb + j * tb, pp[j] + (long long)s * tb, tb, &full[slot], pol_pt);
                const int bi = ent_r[e_lo + s];
                bulk_g2s_hint(stb + 2 * tb, R + (long long)bi * 2 * kN + lx0, 4096, &full[slot], pol_r);
                bulk_g2s_hint(stb + 2 * tb + 4096, R + ((long long)bi * 2 + 1) * kN + lx0, 4096, &full[slot], pol_r);
                if (++slot == kQ0Stages) {
                    slot = 0;
                    if (s >= kQ0Stages) phase ^= 1u;
                }
            }
        }
        return;
    }
    const int t = threadIdx.x;
    const ModConst &mc = pr.m[l];
    Acc60W a00, a01, a10, a11;  // [output j][c0 / c1]
    a00.zero(); a01.zero(); a10.zero(); a11.zero();
    const unsigned full0 = smem_u32(full), empty0 = smem_u32(empty);
    const unsigned char *p_t = ring + 8 * t, *r_t = ring + 2 * tb + 8 * t;
    auto stage = [&](int slot, unsigned ph) {
        mbar_wait_sa(full0 + 8u * slot, ph);
        const unsigned off = (unsigned)slot * kQ0StageBytes;
        const u64 p0 = *reinterpret_cast<const u64 *>(p_t + off), p1 = *reinterpret_cast<const u64 *>(p_t + off + tb);
        const u64 r0 = *reinterpret_cast<const u64 *>(r_t + off), r1 = *reinterpret_cast<const u64 *>(r_t + off + 4096);
        a00.mac(p0, r0); a01.mac(p0, r1);
        a10.mac(p1, r0); a11.mac(p1, r1);   // (slot 1 of a single-output group is stale, never stored)
        mbar_arrive_sa(empty0 + 8u * slot);
    };
    constexpr int kFold = (128 / kQ0Stages) * kQ0Stages;
    const int n_full = n_e - n_e % kQ0Stages;
    unsigned phase = 0;
    int s = 0;
    while (s < n_full) {
        const int s1 = n_full - s < kFold ? n_full : s + kFold;
        for (; s < s1; s += kQ0Stages) {
#pragma unroll
            for (int i = 0; i < kQ0Stages; i++) stage(i, phase);
            phase ^= 1u;
        }
        if (s < n_e && s % kFold == 0) { a00.fold(mc); a01.fold(mc); a10.fold(mc); a11.fold(mc); }
    }
    for (int i = 0; s < n_e; s++, i++) stage(i, phase);
    u64 *out0 = acc + (long long)oa * 2 * kN + lx0 + t;
    out0[0] = a00.reduce(mc);
    out0[kN] = a01.reduce(mc);
    if (nP > 1) {
        u64 *out1 = out0 + 2 * kN;
        out1[0] = a10.reduce(mc);
        out1[kN] = a11.reduce(mc);
    }
}

// Weight-stationary batched MAC (row f4, blb_ct_pt_matmul_batch): kB independent input sets (each with
// its own baby-step buffer R_b and accumulators acc_b, at a fixed stride) against ONE stream of the
// output's plaintexts -- per pipeline stage one plaintext tile + kB (c0, c1) rotation tile pairs, so each
// plaintext byte read from HBM feeds kB inputs (the single-input kernel above shares R between two
// outputs instead).  Same accumulators, folds and final reduction as mac4_consume.
constexpr int kMbB = 2;       // inputs per CTA
constexpr int kMbStages = 3;  // ring stages (3 x ~20 KB: 3 CTAs per SM)
__host__ __device__ constexpr unsigned macb_stage_bytes(int w) { return (unsigned)(512 * w + kMbB * 8192); }
constexpr size_t macb_smem() { return (size_t)kMbStages * macb_stage_bytes(8) + 2 * kMbStages * 8; }
template <bool SPLIT41, bool PACKED>
__device__ __forceinline__ void macb_consume(const unsigned char *ring, uint64_t *full, uint64_t *empty, int n_e, int nB,
                                             u64 *const *outs, long long kN, const ModConst &mc) {
    using A = typename std::conditional<SPLIT41, AccG, Acc128>::type;
    constexpr int NST = kMbStages;
    constexpr unsigned TB = PACKED ? 5u * 512u : 8u * 512u;
    constexpr unsigned SB = TB + kMbB * 8192u;
    const double qd = (double)mc.q, qinv = 1.0 / qd;
    A a00[kMbB], a01[kMbB], a10[kMbB], a11[kMbB];
#pragma unroll
    for (int b = 0; b < kMbB; b++) { a00[b].zero(); a01[b].zero(); a10[b].zero(); a11[b].zero(); }
    const int t = threadIdx.x;
    const unsigned full0 = smem_u32(full), empty0 = smem_u32(empty);
    const unsigned char *rt_t = ring + TB + 16 * t;                       // R tiles of input b at + 8192 b
    const unsigned char *lo_t = ring + (PACKED ? 8 * t : 16 * t);
    const unsigned char *hi_t = ring + 2048 + 2 * t;
    auto stage = [&](int slot, unsigned phase) {
        mbar_wait_sa(full0 + 8u * slot, phase);
        const unsigned off = (unsigned)slot * SB;
        if constexpr (SPLIT41) {
            double Px, Py;
            if constexpr (PACKED) {
                const uint2 lo = *reinterpret_cast<const uint2 *>(lo_t + off);
                const unsigned hi = *reinterpret_cast<const unsigned short *>(hi_t + off);
                Px = __dsub_rn(__hiloint2double((int)__byte_perm(hi, 0x43300000u, 0x7650), (int)lo.x), 4503599627370496.0);
                Py = __dsub_rn(__hiloint2double((int)__byte_perm(hi, 0x43300000u, 0x7651), (int)lo.y), 4503599627370496.0);
            } else {
                const ulonglong2 pv = *reinterpret_cast<const ulonglong2 *>(lo_t + off);
                Px = AccF64::u2d(pv.x);
                Py = AccF64::u2d(pv.y);
            }
#pragma unroll
            for (int b = 0; b < kMbB; b++) {  // unconditional: a missing input's slot holds stale data, never stored
                const double2 r0 = *reinterpret_cast<const double2 *>(rt_t + off + b * 8192);
                const double2 r1 = *reinterpret_cast<const double2 *>(rt_t + off + b * 8192 + 4096);
                a00[b].macd(Px, r0.x); a01[b].macd(Py, r0.y);
                a10[b].macd(Px, r1.x); a11[b].macd(Py, r1.y);
            }
        } else {
            const ulonglong2 pv = *reinterpret_cast<const ulonglong2 *>(lo_t + off);
#pragma unroll
            for (int b = 0; b < kMbB; b++) {
                if (b < nB) {
                    const ulonglong2 r0 = *reinterpret_cast<const ulonglong2 *>(rt_t + off + b * 8192);
                    const ulonglong2 r1 = *reinterpret_cast<const ulonglong2 *>(rt_t + off + b * 8192 + 4096);
                    a00[b].mac(pv.x, r0.x); a01[b].mac(pv.y, r0.y);
                    a10[b].mac(pv.x, r1.x); a11[b].mac(pv.y, r1.y);
                }
            }
        }
        mbar_arrive_sa(empty0 + 8u * slot);
    };
    constexpr int kFold = ((SPLIT41 ? 512 : 64) / NST) * NST;
    const int n_full = n_e - n_e % NST;
    unsigned phase = 0;
    int s = 0;
    while (s < n_full) {
        const int s1 = n_full - s < kFold ? n_full : s + kFold;
        for (; s < s1; s += NST) {
#pragma unroll
            for (int i = 0; i < NST; i++) stage(i, phase);
            phase ^= 1u;
        }
        if (s < n_e && s % kFold == 0) {
#pragma unroll
            for (int b = 0; b < kMbB; b++) {
                accf(a00[b], mc, qd, qinv); accf(a01[b], mc, qd, qinv);
                accf(a10[b], mc, qd, qinv); accf(a11[b], mc, qd, qinv);
            }
        }
    }
    for (int i = 0; s < n_e; s++, i++) stage(i, phase);
#pragma unroll
    for (int b = 0; b < kMbB; b++) {
        if (b < nB) {
            u64 *out = outs[b] + 2 * t;
            *reinterpret_cast<ulonglong2 *>(out) = make_ulonglong2(accr(a00[b], mc, qd, qinv), accr(a01[b], mc, qd, qinv));
            *reinterpret_cast<ulonglong2 *>(out + kN) =
                make_ulonglong2(accr(a10[b], mc, qd, qinv), accr(a11[b], mc, qd, qinv));
        }
    }
}
// grid: (output fastest, tile, limb, input group); R_b = R + b r_stride, acc_b = acc + b acc_stride (u64)
__global__ void __launch_bounds__(kTB + 32, 3) k_mac_tma4b(const unsigned char *__restrict__ pt, const u64 *__restrict__ R,
                                                          long long r_stride, u64 *__restrict__ acc, long long acc_stride,
                                                          int n_batch, const int *__restrict__ ent_r,
                                                          const int *__restrict__ ent_start, int o0, int e_base, int n_o,
                                                          int k, int logN, Primes pr, PtLayout lay) {
    extern __shared__ __align__(128) unsigned char smraw[];
    unsigned char *ring = smraw;
    uint64_t *full = reinterpret_cast<uint64_t *>(smraw + (size_t)kMbStages * macb_stage_bytes(8));
    uint64_t *empty = full + kMbStages;
    const int N = 1 << logN;
    const int n_tiles = N / (2 * kTB);
    int bid = blockIdx.x;
    const int o = bid % n_o;
    bid /= n_o;
    const int tile = bid % n_tiles;
    bid /= n_tiles;
    const int l = bid % k;
    const int b0 = (bid / k) * kMbB, nB = min(kMbB, n_batch - b0);
    const long long kN = (long long)k * N;
    const int e_lo = ent_start[o0 + o], n_e = ent_start[o0 + o + 1] - e_lo;
    const long long lx0 = (long long)l * N + tile * 2 * kTB;
    const int w = lay.w[l];
    const unsigned tb = 512u * (unsigned)w;
    const unsigned stage_bytes = tb + kMbB * 8192u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kMbStages; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kTB);
        }
        mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x >= kTB) {  // producer warp
        if (threadIdx.x == kTB) {
            const unsigned char *pp = pt + (long long)(e_lo - e_base) * lay.bpp + (long long)n_e * lay.loff[l] +
                                      (long long)tile * n_e * tb;
            const uint64_t pol_pt = l2_policy_evict_first(), pol_r = l2_policy_evict_last();
            int slot = 0;
            unsigned phase = 0;
            for (int s = 0; s < n_e; s++) {
                if (s >= kMbStages) {
                    mbar_wait(&empty[slot], phase);
                    fence_proxy_async_smem();
                }
                unsigned char *stb = ring + (size_t)slot * stage_bytes;
                mbar_expect_tx(&full[slot], tb + (unsigned)nB * 8192u);
                bulk_g2s_hint(stb, pp + (long long)s * tb, tb, &full[slot], pol_pt);
                const int bi = ent_r[e_lo + s];
                for (int b = 0; b < nB; b++) {
                    const u64 *Rb = R + (b0 + b) * r_stride;
                    bulk_g2s_hint(stb + tb + b * 8192, Rb + (long long)bi * 2 * kN + lx0, 4096, &full[slot], pol_r);
                    bulk_g2s_hint(stb + tb + b * 8192 + 4096, Rb + ((long long)bi * 2 + 1) * kN + lx0, 4096, &full[slot],
                                  pol_r);
                }
                if (++slot == kMbStages) {
                    slot = 0;
                    if (s >= kMbStages) phase ^= 1u;
                }
            }
        }
        return;
    }
    u64 *outs[kMbB];
#pragma unroll
    for (int b = 0; b < kMbB; b++) outs[b] = acc + (b0 + (b < nB ? b : 0)) * acc_stride + (long long)o * 2 * kN + lx0;
    const ModConst &mc = pr.m[l];
    if (w == 5) macb_consume<true, true>(ring, full, empty, n_e, nB, outs, kN, mc);
    else if (mc.q < (1ull << 41)) macb_consume<true, false>(ring, full, empty, n_e, nB, outs, kN, mc);
    else macb_consume<false, false>(ring, full, empty, n_e, nB, outs, kN, mc);
}

// scatter standard [cnt][k][N] plaintexts (entries e0..e0+cnt of the plan) into the blocked, width-packed layout
__global__ void k_block_pts(const u64 *src, unsigned char *dst, const int *ent_start, const int *ent_o, int e0,
                            int e_base, int k, int N, PtLayout lay) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int l = blockIdx.y, t = blockIdx.z;
    if (x >= N) return;
    const int e = e0 + t;
    const int o = ent_o[e];
    const int e_lo = ent_start[o], n_e = ent_start[o + 1] - e_lo;
    const int w = lay.w[l];
    unsigned char *tile = dst + (long long)(e_lo - e_base) * lay.bpp + (long long)n_e * lay.loff[l] +
                          ((long long)(x >> 9) * n_e + (e - e_lo)) * 512 * w;
    const u64 v = src[(long long)t * k * N + (long long)l * N + x];
    if (w == 5) {
        reinterpret_cast<uint32_t *>(tile)[x & 511] = (uint32_t)v;
        tile[2048 + (x & 511)] = (unsigned char)(v >> 32);
    } else {
        reinterpret_cast<u64 *>(tile)[x & 511] = v;
    }
}

// Indexed mask MAC for JG consecutive outputs that share their plaintext (mask) list and differ only
// in the rotations they multiply (the ct-ct stage-1 MACs: K'_i^(j) / Q_u^(j) for j in a group, reading
// C13): per pipeline stage one entry = the mask tile + the JG (c0, c1) rotation tiles, staged by a
// producer warp with cp.async.bulk into a 3-stage shared-memory ring.  Each mask tile is read once per
// JG outputs instead of once per output, and the consumers never wait on a global load.
constexpr int kMjStages = 3;
template <int JG>
constexpr size_t macj_smem() { return (size_t)kMjStages * (1 + 2 * JG) * 512 * 8 + 2 * kMjStages * 8; }

// SPLIT41 (q < 2^41): AccG for all four accumulators; else Acc128.  Ring slots are compile-time in the
// stage loop (unrolled by kMjStages), as in mac4_consume.
template <bool SPLIT41, int JG>
__device__ __forceinline__ void macj_consume(const u64 *ring, uint64_t *full, uint64_t *empty, int n_e, u64 *const *outs,
                                             long long kN, const ModConst &mc) {
    using A = typename std::conditional<SPLIT41, AccG, Acc128>::type;
    constexpr int NST = kMjStages;
    const double qd = (double)mc.q, qinv = 1.0 / qd;
    A a00[JG], a01[JG], a10[JG], a11[JG];
#pragma unroll
    for (int j = 0; j < JG; j++) { a00[j].zero(); a01[j].zero(); a10[j].zero(); a11[j].zero(); }
    constexpr int kStageWords = (1 + 2 * JG) * 512;
    const int t = threadIdx.x;
    const unsigned full0 = smem_u32(full), empty0 = smem_u32(empty);
    const u64 *ring_t = ring + 2 * t;
    auto stage = [&](int slot, unsigned phase) {
        mbar_wait_sa(full0 + 8u * slot, phase);
        const u64 *st = ring_t + slot * kStageWords;
        if constexpr (SPLIT41) {  // masks and rotations of these limbs are stored as doubles
            const double2 pv = *reinterpret_cast<const double2 *>(st);
#pragma unroll
            for (int j = 0; j < JG; j++) {
                const double2 r0 = *reinterpret_cast<const double2 *>(st + (1 + 2 * j) * 512);
                const double2 r1 = *reinterpret_cast<const double2 *>(st + (2 + 2 * j) * 512);
                a00[j].macd(pv.x, r0.x); a01[j].macd(pv.y, r0.y);
                a10[j].macd(pv.x, r1.x); a11[j].macd(pv.y, r1.y);
            }
        } else {
            const ulonglong2 pv = *reinterpret_cast<const ulonglong2 *>(st);
#pragma unroll
            for (int j = 0; j < JG; j++) {
                const ulonglong2 r0 = *reinterpret_cast<const ulonglong2 *>(st + (1 + 2 * j) * 512);
                const ulonglong2 r1 = *reinterpret_cast<const ulonglong2 *>(st + (2 + 2 * j) * 512);
                a00[j].mac(pv.x, r0.x); a01[j].mac(pv.y, r0.y);
                a10[j].mac(pv.x, r1.x); a11[j].mac(pv.y, r1.y);
            }
        }
        mbar_arrive_sa(empty0 + 8u * slot);  // count kTB: every consumer thread, after its own reads
    };
    // folds after whole ring rounds: Acc128 <= 64 products (< 2^126), AccG <= 512 (s < 2^93, l < 2^48)
    constexpr int kFold = ((SPLIT41 ? 512 : 64) / NST) * NST;
    const int n_full = n_e - n_e % NST;
    unsigned phase = 0;
    int s = 0;
    while (s < n_full) {
        const int s1 = n_full - s < kFold ? n_full : s + kFold;
        for (; s < s1; s += NST) {
#pragma unroll
            for (int i = 0; i < NST; i++) stage(i, phase);
            phase ^= 1u;
        }
        if (s < n_e && s % kFold == 0) {
#pragma unroll
            for (int j = 0; j < JG; j++) {
                accf(a00[j], mc, qd, qinv); accf(a01[j], mc, qd, qinv);
                accf(a10[j], mc, qd, qinv); accf(a11[j], mc, qd, qinv);
            }
        }
    }
    for (int i = 0; s < n_e; s++, i++) stage(i, phase);  // last partial round
#pragma unroll
    for (int j = 0; j < JG; j++) {
        u64 *out = outs[j] + 2 * t;
        *reinterpret_cast<ulonglong2 *>(out) = make_ulonglong2(accr(a00[j], mc, qd, qinv), accr(a01[j], mc, qd, qinv));
        *reinterpret_cast<ulonglong2 *>(out + kN) = make_ulonglong2(accr(a10[j], mc, qd, qinv), accr(a11[j], mc, qd, qinv));
    }
}

// grid: (group fastest, tile, limb); group gi covers outputs o0 + gi*JG .. + JG - 1 (local o)
template <int JG, int MINB>
__global__ void __launch_bounds__(kTB + 32, MINB) k_mac_j(const u64 *__restrict__ pt, const u64 *__restrict__ R,
                                                     u64 *__restrict__ acc, const int *__restrict__ ent_r,
                                                     const int *__restrict__ ent_pt, const int *__restrict__ ent_start,
                                                     int o0, int n_grp, int k, int kq, int Kfull, int logN, Primes pr) {
    constexpr int kStageWords = (1 + 2 * JG) * 512;
    extern __shared__ __align__(128) unsigned char smraw[];
    u64 *ring = reinterpret_cast<u64 *>(smraw);
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + (size_t)kMjStages * kStageWords);
    uint64_t *empty = full + kMjStages;
    const int N = 1 << logN;
    const int n_tiles = N / (2 * kTB);
    int bid = blockIdx.x;
    const int gi = bid % n_grp;
    bid /= n_grp;
    const int tile = bid % n_tiles;
    const int l = bid / n_tiles;
    const int oa = gi * JG;
    const long long kN = (long long)k * N;
    const int e_lo = ent_start[o0 + oa], n_e = ent_start[o0 + oa + 1] - e_lo;
    const long long lx0 = (long long)l * N + tile * 2 * kTB;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kMjStages; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kTB);  // one arrival per consumer thread (macj_consume)
        }
        mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x >= kTB) {  // producer warp
        if (threadIdx.x == kTB) {
            int eb[JG];
#pragma unroll
            for (int j = 0; j < JG; j++) eb[j] = ent_start[o0 + oa + j];
            for (int s = 0; s < n_e; s++) {
                const int slot = s % kMjStages;
                if (s >= kMjStages) {
                    mbar_wait(&empty[slot], ((s / kMjStages) - 1) & 1);
                    fence_proxy_async_smem();
                }
                u64 *st = ring + (size_t)slot * kStageWords;
                mbar_expect_tx(&full[slot], (unsigned)(1 + 2 * JG) * 4096);
                bulk_g2s(st, pt + (long long)ent_pt[e_lo + s] * kN + lx0, 4096, &full[slot]);
#pragma unroll
                for (int j = 0; j < JG; j++) {
                    const int bi = ent_r[eb[j] + s];
                    bulk_g2s(st + (1 + 2 * j) * 512, R + (long long)bi * 2 * kN + lx0, 4096, &full[slot]);
                    bulk_g2s(st + (2 + 2 * j) * 512, R + ((long long)bi * 2 + 1) * kN + lx0, 4096, &full[slot]);
                }
            }
        }
        return;
    }
    u64 *outs[JG];
#pragma unroll
    for (int j = 0; j < JG; j++) outs[j] = acc + (long long)(oa + j) * 2 * kN + lx0;
    const ModConst &mc = pr.m[l < kq ? l : Kfull + (l - kq)];
    if (mc.q < (1ull << 41)) macj_consume<true, JG>(ring, full, empty, n_e, outs, kN, mc);
    else macj_consume<false, JG>(ring, full, empty, n_e, outs, kN, mc);
}

// dst[o] += src[j] for the jobs of one giant batch (sequential per thread: no races)
struct AccJobs {
    int n;
    u64 *dst[kMaxJobs];
    const u64 *src[kMaxJobs];
};
// limbs l >= kq of an extended (Q_l u P) ciphertext are the special primes K + (l - kq)
__global__ void k_accumulate(AccJobs jobs, Primes pr, int k, int N, int kq, int K) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int l = blockIdx.y, p = blockIdx.z;
    if (x >= N) return;
    const u64 q = pr.m[l < kq ? l : K + (l - kq)].q;
    const long long off = ((long long)p * k + l) * N + x;
    for (int j = 0; j < jobs.n; j++) jobs.dst[j][off] = addmod(jobs.dst[j][off], jobs.src[j][off], q);
}

// R[b][0] = X_b in the baby-step buffer's format: limbs with q < 2^41 as double bits (KsJob::out_f64)
__global__ void k_copy_ct_f64(const u64 *src, u64 *dst, Primes pr, int k, int logN) {
    const long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= (2ll * k) << logN) return;
    const int l = (int)((x >> logN) % k);
    const u64 v = src[x];
    dst[x] = pr.m[l].q < (1ull << 41) ? (u64)__double_as_longlong((double)v) : v;
}
}  // namespace

blb_status launch_mac(const blb_params *P, const u64 *pt, const u64 *R, u64 *acc, const int *ent_r, const int *ent_pt,
                      const int *ent_start, int o0, int e_base, int n_o, int n_entries, int k, cudaStream_t st,
                      int kq, int jg) {
    if (n_o <= 0) return BLB_OK;
    const int N = P->N;
    const int n_tiles = N / (2 * kTB);
    cudaEvent_t t0 = blb_timing_begin(st);
    constexpr int JGc = 2;  // outputs per CTA sharing the mask list (4 measured slower)
    if (jg % JGc == 0 && n_o % JGc == 0 && ent_pt && P->logN >= 9) {
        // groups of JGc outputs sharing the mask list (reading C13 stage 1): k_mac_j
        const int n_grp = n_o / JGc;
        const unsigned grid = (unsigned)((size_t)n_grp * n_tiles * k);
        constexpr size_t smem = macj_smem<JGc>();
        blb_smem_optin(k_mac_j<JGc, 3>, smem);
        k_mac_j<JGc, 3><<<grid, kTB + 32, smem, st>>>(pt, R, acc, ent_r, ent_pt, ent_start, o0, n_grp, k,
                                                      kq < 0 ? k : kq, P->K, P->logN, P->pr);
        BLB_COUNT_LAUNCH(1);
        BLB_COUNT(3, n_entries);
        // bytes staged: one mask tile per entry per group of JGc outputs + the (c0, c1) rotation tiles
        blb_timing_end(3, t0, st, ((double)n_entries / JGc + 2.0 * n_entries) * k * N * 8.0);
        BLB_CHECK_LAUNCH();
        return BLB_OK;
    }
    // (a warp-specialised bulk-copy version of this indexed MAC measured slower: 8.1 vs 7.5 ms per step)
    k_mac<<<(unsigned)((size_t)n_o * n_tiles * k), kTB, 0, st>>>(pt, R, acc, ent_r, ent_pt, ent_start, o0, e_base,
                                                                    n_o, k, kq < 0 ? k : kq, P->K, P->logN, P->pr);
    BLB_COUNT_LAUNCH(1);
    BLB_COUNT(3, n_entries);
    blb_timing_end(3, t0, st, 3.0 * n_entries * k * N * 8.0);  // category 3: ct-ct mask MAC (mask + c0, c1 bytes)
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}

// ------------------------------------------------------------------ plan
static bool nz_entry(const blb_matmul_plan *pl, int b, int bp, int t) {
    for (int tau = 0; tau < pl->c; tau++) {
        const int r = b * pl->c + (tau + t) % pl->c;
        const int col = bp * pl->c + tau;
        if (col >= pl->D_out) continue;
        if (pl->packing == BLB_PACK_SPATIAL) {
            if (r < pl->w_rows && pl->col_map[col] >= 0) return true;
        } else {
            if (r < pl->nblk_in) return true;
        }
    }
    return false;
}

extern "C" blb_status blb_matmul_plan_create(const blb_params *P, int L, int w_rows, int w_cols, blb_packing packing,
                                             int heads, const int32_t *col_map, int D_out, int bsgs_B, int level,
                                             blb_matmul_plan **out) {
    return blb_matmul_plan_create_window(P, L, w_rows, w_cols, packing, heads, col_map, D_out, bsgs_B, level, 0, -1,
                                         out);
}

extern "C" blb_status blb_matmul_plan_create_window(const blb_params *P, int L, int w_rows, int w_cols,
                                                    blb_packing packing, int heads, const int32_t *col_map, int D_out,
                                                    int bsgs_B, int level, int i_first, int i_count,
                                                    blb_matmul_plan **out) {
    if (!P || !out || L <= 0 || w_rows <= 0 || w_cols <= 0 || bsgs_B <= 0) {
        blb_set_error("blb_matmul_plan_create: invalid argument");
        return BLB_E_INVALID_ARG;
    }
    const int n = P->N / 2;
    if (n % L) {
        blb_set_error("blb_matmul_plan_create: L=%d must divide N/2=%d", L, n);
        return BLB_E_LAYOUT;
    }
    if (level < 1 || level >= P->K) {
        blb_set_error("blb_matmul_plan_create: level %d must be in [1, %d) (one rescale)", level, P->K);
        return BLB_E_LEVEL;
    }
    auto *pl = new blb_matmul_plan();
    pl->P = P; pl->L = L; pl->n = n; pl->c = n / L; pl->w_rows = w_rows; pl->w_cols = w_cols;
    pl->packing = packing; pl->level = level; pl->heads = heads > 0 ? heads : 1;
    pl->B = std::min(bsgs_B, pl->c);
    pl->G = (pl->c + pl->B - 1) / pl->B;
    if (i_count < 0) i_count = pl->B - i_first;
    if (i_first < 0 || i_first + i_count > pl->B) {
        blb_set_error("blb_matmul_plan_create_window: window [%d, %d) outside [0, B = %d)", i_first, i_first + i_count,
                      pl->B);
        delete pl;
        return BLB_E_INVALID_ARG;
    }
    pl->i_first = i_first;
    pl->i_count = i_count;
    if (packing == BLB_PACK_SPATIAL) {
        if (col_map) {
            pl->D_out = D_out;
            pl->col_map.assign(col_map, col_map + D_out);
            for (int v : pl->col_map)
                if (v >= w_cols) {
                    delete pl;
                    blb_set_error("col_map entry %d >= w_cols %d", v, w_cols);
                    return BLB_E_LAYOUT;
                }
        } else {
            pl->D_out = w_cols;
            pl->col_map.resize(w_cols);
            for (int i = 0; i < w_cols; i++) pl->col_map[i] = i;
        }
        pl->nblk_in = w_rows;
        pl->dh = 0;
    } else if (packing == BLB_PACK_DIAGONAL) {
        if (w_rows % pl->heads) {
            delete pl;
            blb_set_error("diagonal packing: w_rows %d not divisible by heads %d", w_rows, pl->heads);
            return BLB_E_LAYOUT;
        }
        pl->dh = w_rows / pl->heads;
        pl->nblk_in = w_rows;
        pl->D_out = w_cols;
        pl->col_map.resize(w_cols);
        for (int i = 0; i < w_cols; i++) pl->col_map[i] = i;
    } else {
        delete pl;
        blb_set_error("unknown packing");
        return BLB_E_LAYOUT;
    }
    pl->n_in = (pl->nblk_in + pl->c - 1) / pl->c;
    pl->n_out = (pl->D_out + pl->c - 1) / pl->c;
    pl->baby.assign(pl->n_in, {});
    pl->giant.assign(pl->n_out, {});
    pl->ent_start.push_back(0);
    std::vector<int> ent_o;
    std::vector<std::vector<char>> baby_used(pl->n_in, std::vector<char>(pl->B, 0));
    for (int bp = 0; bp < pl->n_out; bp++) {
        for (int g = 0; g < pl->G; g++) {
            int cnt = 0;
            for (int b = 0; b < pl->n_in; b++)
                for (int i = 0; i < pl->B; i++) {
                    const int t = g * pl->B + i;
                    if (t >= pl->c) continue;
                    if (!nz_entry(pl, b, bp, t)) continue;
                    cnt++;  // giant steps follow the whole plan (the owner rotates the summed acc)
                    if (i < pl->i_first || i >= pl->i_first + pl->i_count) continue;
                    pl->ent_b.push_back(b);
                    pl->ent_i.push_back(i);
                    ent_o.push_back(bp * pl->G + g);
                    baby_used[b][i] = 1;
                }
            if (cnt && g > 0) pl->giant[bp].push_back(g);
            pl->ent_start.push_back((int)pl->ent_b.size());
        }
    }
    std::map<int32_t, int> steps;
    for (int b = 0; b < pl->n_in; b++)
        for (int i = 1; i < pl->B; i++)
            if (baby_used[b][i]) {
                pl->baby[b].push_back(i);
                steps[i * L] = 1;
            }
    for (int bp = 0; bp < pl->n_out; bp++)
        for (int g : pl->giant[bp]) steps[g * pl->B * L] = 1;
    for (auto &kv : steps) pl->rot_steps.push_back(kv.first);
    // device copies
    const size_t ne = pl->ent_b.size();
    std::vector<int> bi(ne);
    for (size_t e = 0; e < ne; e++) bi[e] = pl->ent_b[e] * pl->B + pl->ent_i[e];
    const int n_og = pl->n_out * pl->G;
    pl->same_next.assign(n_og, 0);
    for (int o = 0; o + 1 < n_og; o++) {
        const int a0 = pl->ent_start[o], a1 = pl->ent_start[o + 1], b1 = pl->ent_start[o + 2];
        pl->same_next[o] = (a1 - a0 == b1 - a1) && std::equal(bi.begin() + a0, bi.begin() + a1, bi.begin() + a1);
    }
    cudaError_t err = cudaSuccess;
    err = cudaMalloc(&pl->d_ent, sizeof(int) * (2 * ne + 1));
    if (err == cudaSuccess) err = cudaMalloc(&pl->d_ent_start, sizeof(int) * pl->ent_start.size());
    if (err == cudaSuccess) err = cudaMalloc(&pl->d_col_map, sizeof(int32_t) * (pl->col_map.size() + 1));
    if (err == cudaSuccess && ne) err = cudaMemcpy(pl->d_ent, bi.data(), sizeof(int) * ne, cudaMemcpyHostToDevice);
    if (err == cudaSuccess && ne)
        err = cudaMemcpy(pl->d_ent + ne, ent_o.data(), sizeof(int) * ne, cudaMemcpyHostToDevice);
    if (err == cudaSuccess)
        err = cudaMemcpy(pl->d_ent_start, pl->ent_start.data(), sizeof(int) * pl->ent_start.size(),
                         cudaMemcpyHostToDevice);
    if (err == cudaSuccess)
        err = cudaMemcpy(pl->d_col_map, pl->col_map.data(), sizeof(int32_t) * pl->col_map.size(),
                         cudaMemcpyHostToDevice);
    if (err != cudaSuccess) {
        blb_set_error("plan upload: %s", cudaGetErrorString(err));
        blb_matmul_plan_destroy(pl);
        return BLB_E_CUDA;
    }
    *out = pl;
    return BLB_OK;
}

extern "C" void blb_matmul_plan_destroy(blb_matmul_plan *pl) {
    if (!pl) return;
    cudaFree(pl->d_ent);
    cudaFree(pl->d_ent_start);
    cudaFree(pl->d_col_map);
    delete pl;
}

extern "C" blb_status blb_matmul_plan_info(const blb_matmul_plan *pl, int *n_in, int *n_out, int *n_pt, int *n_baby,
                                           int *n_giant, int *B, int *G) {
    if (!pl) return BLB_E_INVALID_ARG;
    int nb = 0, ng = 0;
    for (auto &v : pl->baby) nb += (int)v.size();
    for (auto &v : pl->giant) ng += (int)v.size();
    if (n_in) *n_in = pl->n_in;
    if (n_out) *n_out = pl->n_out;
    if (n_pt) *n_pt = (int)pl->ent_b.size();
    if (n_baby) *n_baby = nb;
    if (n_giant) *n_giant = ng;
    if (B) *B = pl->B;
    if (G) *G = pl->G;
    return BLB_OK;
}

extern "C" blb_status blb_matmul_plan_rotations(const blb_matmul_plan *pl, int32_t *steps, int *n) {
    if (!pl || !n) return BLB_E_INVALID_ARG;
    const int need = (int)pl->rot_steps.size();
    if (steps) {
        if (*n < need) {
            blb_set_error("rotation buffer too small (%d < %d)", *n, need);
            return BLB_E_INVALID_ARG;
        }
        for (int i = 0; i < need; i++) steps[i] = pl->rot_steps[i];
    }
    *n = need;
    return BLB_OK;
}

static blb_status check_slice(const blb_matmul_plan *pl, int out_first, int out_count) {
    if (out_first < 0 || out_count < 0 || out_first + out_count > pl->n_out) {
        blb_set_error("output slice [%d, %d) outside [0, %d)", out_first, out_first + out_count, pl->n_out);
        return BLB_E_INVALID_ARG;
    }
    return BLB_OK;
}

// width-packed blocked plaintext layout of the plan's level (see the weight MAC above)
static PtLayout pt_layout(const blb_matmul_plan *pl) {
    const blb_params *P = pl->P;
    const int k = pl->level + 1;
    PtLayout lay{};
    long long off = 0;
    for (int l = 0; l < k; l++) {
        lay.w[l] = (P->mod[l] < (1ull << 40) && P->logN >= 9) ? 5 : 8;
        lay.loff[l] = off;
        off += (long long)lay.w[l] * P->N;
    }
    lay.bpp = off;
    return lay;
}

extern "C" blb_status blb_matmul_pt_bytes(const blb_matmul_plan *pl, int out_first, int out_count, size_t *bytes) {
    if (!pl || !bytes) return BLB_E_INVALID_ARG;
    BLB_TRY(check_slice(pl, out_first, out_count));
    const long long n = pl->ent_start[(out_first + out_count) * pl->G] - pl->ent_start[out_first * pl->G];
    *bytes = (size_t)n * (size_t)pt_layout(pl).bpp;
    return BLB_OK;
}

extern "C" blb_status blb_matmul_pt_count(const blb_matmul_plan *pl, int out_first, int out_count, int *n_pt) {
    if (!pl || !n_pt) return BLB_E_INVALID_ARG;
    BLB_TRY(check_slice(pl, out_first, out_count));
    *n_pt = pl->ent_start[(out_first + out_count) * pl->G] - pl->ent_start[out_first * pl->G];
    return BLB_OK;
}

extern "C" blb_status blb_matmul_encode_weights(const blb_matmul_plan *pl, const double *W, int out_first,
                                                int out_count, u64 *pt_dev, void *stream) {
    if (!pl || !W || !pt_dev) return BLB_E_INVALID_ARG;
    BLB_TRY(check_slice(pl, out_first, out_count));
    const blb_params *P = pl->P;
    cudaStream_t st = (cudaStream_t)stream;
    const int e0 = pl->ent_start[out_first * pl->G];
    const int e1 = pl->ent_start[(out_first + out_count) * pl->G];
    const int k = pl->level + 1;
    const size_t ne_total = pl->ent_b.size();
    double *dW = nullptr, *slots = nullptr, *buf = nullptr;
    int *flag = nullptr;
    const int chunk = 64;
    BLB_CUDA_TRY(cudaMallocAsync(&dW, sizeof(double) * (size_t)pl->w_rows * pl->w_cols, st));
    // W may be host or device memory (unified addressing): per-layer re-encode from device-resident weights
    BLB_CUDA_TRY(cudaMemcpyAsync(dW, W, sizeof(double) * (size_t)pl->w_rows * pl->w_cols, cudaMemcpyDefault, st));
    BLB_CUDA_TRY(cudaMallocAsync(&slots, sizeof(double) * (size_t)chunk * pl->n, st));
    BLB_CUDA_TRY(cudaMallocAsync(&buf, sizeof(double) * encode_scratch_doubles(P, chunk), st));
    BLB_CUDA_TRY(cudaMallocAsync(&flag, sizeof(int), st));
    BLB_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int), st));
    u64 *tmp = nullptr;
    BLB_CUDA_TRY(cudaMallocAsync(&tmp, sizeof(u64) * (size_t)chunk * k * P->N, st));
    PlanDev pd{pl->L, pl->n, pl->c, pl->B, pl->G, pl->w_rows, pl->w_cols, pl->nblk_in, pl->D_out, pl->packing,
               pl->heads, pl->dh};
    const double scale = (double)P->mod[pl->level];  // reading S6: plaintext scale = q_level
    blb_status s = BLB_OK;
    for (int e = e0; e < e1 && s == BLB_OK; e += chunk) {
        const int cnt = std::min(chunk, e1 - e);
        k_build_slots<<<dim3((pl->n + kTB - 1) / kTB, cnt), kTB, 0, st>>>(pd, pl->d_ent, pl->d_ent + ne_total, e, dW,
                                                                         pl->d_col_map, slots);
        BLB_COUNT_LAUNCH(1);
        s = launch_encode(P, slots, cnt, scale, pl->level, tmp, buf, flag, st);
        if (s == BLB_OK) {
            k_block_pts<<<dim3((P->N + kTB - 1) / kTB, k, cnt), kTB, 0, st>>>(
                tmp, reinterpret_cast<unsigned char *>(pt_dev), pl->d_ent_start, pl->d_ent + ne_total, e, e0, k, P->N,
                pt_layout(pl));
            BLB_COUNT_LAUNCH(1);
        }
    }
    int h_flag = 0;
    cudaMemcpyAsync(&h_flag, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(dW, st);
    cudaFreeAsync(tmp, st);
    cudaFreeAsync(slots, st);
    cudaFreeAsync(buf, st);
    cudaFreeAsync(flag, st);
    BLB_CUDA_TRY(cudaStreamSynchronize(st));
    if (s != BLB_OK) return s;
    if (h_flag) {
        blb_set_error("encode overflow: |scale * m_k| >= 2^52");
        return BLB_E_OVERFLOW;
    }
    return BLB_OK;
}

// Config 5 (12 layers on one GPU): the prime-independent half of the encode kept in compact form.
extern "C" blb_status blb_matmul_coeff_bytes(const blb_matmul_plan *pl, int out_first, int out_count, size_t *bytes) {
    if (!pl || !bytes) return BLB_E_INVALID_ARG;
    BLB_TRY(check_slice(pl, out_first, out_count));
    const size_t n = (size_t)(pl->ent_start[(out_first + out_count) * pl->G] - pl->ent_start[out_first * pl->G]);
    *bytes = n * 5 * (size_t)pl->P->N;
    return BLB_OK;
}

extern "C" blb_status blb_matmul_encode_coeffs(const blb_matmul_plan *pl, const double *W, int out_first, int out_count,
                                               void *coef_dev, void *stream) {
    if (!pl || !W || !coef_dev) return BLB_E_INVALID_ARG;
    BLB_TRY(check_slice(pl, out_first, out_count));
    const blb_params *P = pl->P;
    cudaStream_t st = (cudaStream_t)stream;
    const int e0 = pl->ent_start[out_first * pl->G];
    const int e1 = pl->ent_start[(out_first + out_count) * pl->G];
    const size_t ne_total = pl->ent_b.size();
    double *dW = nullptr, *slots = nullptr, *buf = nullptr;
    int *flag = nullptr;
    const int chunk = 64;
    BLB_CUDA_TRY(cudaMallocAsync(&dW, sizeof(double) * (size_t)pl->w_rows * pl->w_cols, st));
    BLB_CUDA_TRY(cudaMemcpyAsync(dW, W, sizeof(double) * (size_t)pl->w_rows * pl->w_cols, cudaMemcpyDefault, st));
    BLB_CUDA_TRY(cudaMallocAsync(&slots, sizeof(double) * (size_t)chunk * pl->n, st));
    BLB_CUDA_TRY(cudaMallocAsync(&buf, sizeof(double) * encode_scratch_doubles(P, chunk), st));
    BLB_CUDA_TRY(cudaMallocAsync(&flag, sizeof(int), st));
    BLB_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int), st));
    PlanDev pd{pl->L, pl->n, pl->c, pl->B, pl->G, pl->w_rows, pl->w_cols, pl->nblk_in, pl->D_out, pl->packing,
               pl->heads, pl->dh};
    const double scale = (double)P->mod[pl->level];  // reading S6: plaintext scale = q_level
    unsigned char *cb = reinterpret_cast<unsigned char *>(coef_dev);
    blb_status s = BLB_OK;
    for (int e = e0; e < e1 && s == BLB_OK; e += chunk) {
        const int cnt = std::min(chunk, e1 - e);
        k_build_slots<<<dim3((pl->n + kTB - 1) / kTB, cnt), kTB, 0, st>>>(pd, pl->d_ent, pl->d_ent + ne_total, e, dW,
                                                                         pl->d_col_map, slots);
        BLB_COUNT_LAUNCH(1);
        s = launch_encode_coef5(P, slots, cnt, scale, cb + (size_t)(e - e0) * 5 * P->N, buf, flag, st);
    }
    int h_flag = 0;
    cudaMemcpyAsync(&h_flag, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(dW, st);
    cudaFreeAsync(slots, st);
    cudaFreeAsync(buf, st);
    cudaFreeAsync(flag, st);
    BLB_CUDA_TRY(cudaStreamSynchronize(st));
    if (s != BLB_OK) return s;
    if (h_flag == 1) {
        blb_set_error("encode overflow: |scale * m_k| >= 2^52");
        return BLB_E_OVERFLOW;
    }
    if (h_flag == 2) {
        blb_set_error("blb_matmul_encode_coeffs: a coefficient needs more than 40 bits (use blb_matmul_encode_weights)");
        return BLB_E_OVERFLOW;
    }
    return BLB_OK;
}

extern "C" blb_status blb_matmul_coeffs_to_pts(const blb_matmul_plan *pl, const void *coef_dev, int out_first,
                                               int out_count, uint64_t *pt_dev, void *stream) {
    if (!pl || !coef_dev || !pt_dev) return BLB_E_INVALID_ARG;
    BLB_TRY(check_slice(pl, out_first, out_count));
    const blb_params *P = pl->P;
    cudaStream_t st = (cudaStream_t)stream;
    const int e0 = pl->ent_start[out_first * pl->G];
    const int e1 = pl->ent_start[(out_first + out_count) * pl->G];
    const size_t ne_total = pl->ent_b.size();
    const int k = pl->level + 1;
    const int chunk = 256;  // 256 plaintexts x k limbs per NTT batch
    u64 *tmp = nullptr;
    BLB_CUDA_TRY(cudaMallocAsync(&tmp, sizeof(u64) * (size_t)std::min(chunk, std::max(1, e1 - e0)) * k * P->N, st));
    const unsigned char *cb = reinterpret_cast<const unsigned char *>(coef_dev);
    blb_status s = BLB_OK;
    const PtLayout lay = pt_layout(pl);
    for (int e = e0; e < e1 && s == BLB_OK; e += chunk) {
        const int cnt = std::min(chunk, e1 - e);
        if (P->logN == 16) {
            // one fused launch pair: residues in the first NTT pass, packed layout in the last
            RowBatch rb{};
            rb.base = tmp; rb.poly_stride = (long long)k * P->N; rb.n_polys = cnt; rb.limbs = k; rb.limb0 = 0;
            for (int i = 0; i < k; i++) rb.prime[i] = i;
            NttFuse fz{};
            fz.pro = 3;
            fz.epi = 2;
            fz.coef = cb + (size_t)(e - e0) * 5 * P->N;
            fz.pk_dst = reinterpret_cast<unsigned char *>(pt_dev);
            fz.pk_ent_o = pl->d_ent + ne_total;
            fz.pk_ent_start = pl->d_ent_start;
            fz.pk_e0 = e;
            fz.pk_ebase = e0;
            fz.pk_bpp = lay.bpp;
            for (int i = 0; i < k; i++) { fz.pk_loff[i] = lay.loff[i]; fz.pk_w[i] = lay.w[i]; }
            s = launch_ntt_fused(P, rb, false, fz, st);
            continue;
        }
        s = launch_coef5_to_rns(P, cb + (size_t)(e - e0) * 5 * P->N, cnt, pl->level, tmp, st);
        if (s == BLB_OK) {
            k_block_pts<<<dim3((P->N + kTB - 1) / kTB, k, cnt), kTB, 0, st>>>(
                tmp, reinterpret_cast<unsigned char *>(pt_dev), pl->d_ent_start, pl->d_ent + ne_total, e, e0, k, P->N, lay);
            BLB_COUNT_LAUNCH(1);
        }
    }
    cudaFreeAsync(tmp, st);
    BLB_CHECK_LAUNCH();
    return s;
}

// workspace layout (u64 elements)
struct MatmulWs {
    size_t ext_in, coef, R, ks, acc, gext, gcoef, gks, rot, yext, resc, total;
};
static MatmulWs matmul_ws(const blb_matmul_plan *pl, int out_count) {
    const blb_params *P = pl->P;
    const size_t N = P->N, k = pl->level + 1, E = k + P->np, beta = blb_beta(P, pl->level);
    MatmulWs w{};
    size_t o = 0;
    w.ext_in = o; o += (size_t)pl->n_in * beta * E * N;
    w.coef = o; o += (size_t)kMaxJobs * k * N;
    w.R = o; o += (size_t)pl->n_in * pl->B * 2 * k * N;
    w.ks = o; o += keyswitch_scratch_elems(P, pl->level, kMaxJobs);
    w.acc = o; o += (size_t)out_count * pl->G * 2 * k * N;
    w.gext = o; o += (size_t)kMaxJobs * beta * E * N;
    w.gcoef = o; o += (size_t)kMaxJobs * k * N;
    w.gks = o; o += keyswitch_scratch_elems(P, pl->level, kMaxJobs);
    w.rot = o; o += (size_t)kMaxJobs * 2 * E * N;
    w.yext = o; o += (size_t)out_count * 2 * E * N;
    w.resc = o; o += (2 + 2 * k) * N;
    w.total = o;
    return w;
}

extern "C" size_t blb_matmul_workspace_bytes(const blb_matmul_plan *pl, int out_count) {
    if (!pl) return 0;
    return matmul_ws(pl, out_count).total * sizeof(u64) + 256;
}

static const u64 *mm_key(const blb_params *P, const blb_keys *keys, int32_t step) {
    const uint32_t g = blb_galois_element(P, step);
    for (size_t i = 0; i < keys->galois.size(); i++)
        if (keys->galois[i] == g) return keys->data[i];
    return nullptr;
}

static blb_status mm_check(const blb_matmul_plan *pl, const blb_keys *keys, const blb_ct *in, int n_in, bool baby,
                           bool giant) {
    const blb_params *P = pl->P;
    if (in) {
        if (n_in != pl->n_in) {
            blb_set_error("blb_ct_pt_matmul: %d inputs, plan needs %d", n_in, pl->n_in);
            return BLB_E_LAYOUT;
        }
        for (int b = 0; b < n_in; b++)
            if (in[b].level != pl->level || !in[b].data) {
                blb_set_error("input %d at level %d, plan level %d", b, in[b].level, pl->level);
                return BLB_E_LEVEL;
            }
    }
    for (int32_t s : pl->rot_steps) {
        const bool is_giant = s % (pl->B * pl->L) == 0 && s >= pl->B * pl->L;
        if ((is_giant ? giant : baby) && !mm_key(P, keys, s)) {
            blb_set_error("missing rotation key for step %d", s);
            return BLB_E_MISSING_KEY;
        }
    }
    return BLB_OK;
}

namespace {
// acc[o][p][l][x] mod q_l for cross-rank sums of residues (< 2^64: at most 8 ranks of residues < 2^61)
__global__ void k_reduce_acc(const u64 *src, u64 *dst, Primes pr, int k, int N, long long n_polys) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int l = blockIdx.y;
    if (x >= N) return;
    const ModConst &mc = pr.m[l];
    for (long long p = blockIdx.z; p < n_polys; p += gridDim.z) {
        const long long off = (p * k + l) * N + x;
        dst[off] = mod64(src[off], mc);
    }
}
}  // namespace

// Phase A (rows a2 + a3): ModUp of every input once (hoisting, C8), the baby-step rotations of the
// plan's window, and the MAC of the window's plaintexts into acc[o][g] for the outputs
// [out_first, out_first + out_count) (pt_dev holds that slice's plaintexts).
static blb_status mm_acc(const blb_matmul_plan *pl, const blb_keys *keys, const blb_ct *in, const u64 *pt_dev,
                         int out_first, int out_count, u64 *acc, u64 *W, const MatmulWs &w, cudaStream_t st,
                         bool do_mac = true) {
    const blb_params *P = pl->P;
    const int n_in = pl->n_in, level = pl->level, k = level + 1, N = P->N, E = k + P->np, beta = blb_beta(P, level);
    u64 *ext_in = W + w.ext_in, *coef = W + w.coef, *R = W + w.R, *ks = W + w.ks;
    const size_t ctN = (size_t)2 * k * N;
    u64 *ks_u = ks, *ks_conv = ks + (size_t)kMaxJobs * 2 * E * N;
    auto find_key = [&](int32_t step) { return mm_key(P, keys, step); };
    const bool has_baby = [&] {
        for (auto &v : pl->baby)
            if (!v.empty()) return true;
        return false;
    }();
    const bool win0 = pl->i_first == 0;  // R[b][0] = X_b is in this window
    // 1. ModUp of every input c1 (hoisted) and R[b][0] = X_b
    if (has_baby || win0) {
        std::vector<const u64 *> c1;
        for (int b = 0; b < n_in; b++) c1.push_back(in[b].data + (size_t)k * N);
        for (int b0 = 0; b0 < n_in && has_baby; b0 += kMaxJobs) {
            const int cnt = std::min(kMaxJobs, n_in - b0);
            BLB_TRY(launch_modup(P, level, c1.data() + b0, cnt, ext_in + (size_t)b0 * beta * E * N, coef, st));
        }
        for (int b = 0; b < n_in && win0; b++) {
            k_copy_ct_f64<<<(unsigned)((ctN + kTB - 1) / kTB), kTB, 0, st>>>(in[b].data, R + (size_t)b * pl->B * ctN,
                                                                            P->pr, k, P->logN);
            BLB_COUNT_LAUNCH(1);
        }
    }
    // 2. baby steps: R[b][i] = Rot_{iL}(X_b), batched
    {
        // i-major order: the inputs that use the same baby-step key are adjacent, so one
        // launch group loads each key once for all of them (launch_keyswitch groups by key)
        std::vector<KsJob> jobs;
        for (int i = 1; i < pl->B; i++)
            for (int b = 0; b < n_in; b++) {
                if (!std::binary_search(pl->baby[b].begin(), pl->baby[b].end(), i)) continue;
                KsJob J{};
                J.ext = ext_in + (size_t)b * beta * E * N;
                J.key = find_key(i * pl->L);
                J.c0 = in[b].data;
                J.out = R + ((size_t)b * pl->B + i) * ctN;
                J.galois = blb_galois_element(P, i * pl->L);
                J.add_mode = 1;
                J.out_f64 = 1;
                jobs.push_back(J);
            }
        for (size_t j0 = 0; j0 < jobs.size(); j0 += kMaxJobs) {
            const int cnt = (int)std::min<size_t>(kMaxJobs, jobs.size() - j0);
            BLB_TRY(launch_keyswitch(P, level, jobs.data() + j0, cnt, ks_u, ks_conv, st));
        }
    }
    // 3. MAC: acc[b', g] = sum over the window's entries (b, i) of P (.) R[b][i]
    if (!do_mac) return BLB_OK;  // (blb_ct_pt_matmul_batch: one MAC launch for all input sets)
    const int o0 = out_first * pl->G, n_o = out_count * pl->G;
    const int e_base = pl->ent_start[out_first * pl->G];
    const int n_entries = pl->ent_start[o0 + n_o] - pl->ent_start[o0];
    if (n_o > 0 && n_entries == 0) {
        BLB_CUDA_TRY(cudaMemsetAsync(acc, 0, sizeof(u64) * (size_t)n_o * ctN, st));
    } else if (n_o > 0) {
        const int n_tiles = N / (2 * kTB);
        const PtLayout lay = pt_layout(pl);
        const unsigned char *ptb = reinterpret_cast<const unsigned char *>(pt_dev);
        cudaEvent_t t0 = blb_timing_begin(st);
        // pairs of consecutive (b', g) with one entry list -> the two-output kernel (each R tile
        // staged once for both); plans whose pairs differ take one output per CTA.  An empty entry
        // list (possible in a window) yields a zero accumulator.
        bool grouped = true;
        for (int j = 0; j < n_o && grouped; j++)
            if (j % BLB_MAC_P != BLB_MAC_P - 1 && j + 1 < n_o && !pl->same_next[o0 + j]) grouped = false;
#ifndef BLB_MAC_Q0
#define BLB_MAC_Q0 1
#endif
        // the 8-byte limb with a prime >= 2^41 (q0) in its own kernel on the auxiliary stream
        int q0l = -1;
        if (BLB_MAC_Q0 && grouped && P->aux && BLB_MAC_P == 2)
            for (int l = 0; l < k && q0l < 0; l++)
                if (lay.w[l] == 8 && P->mod[l] >= (1ull << 41)) q0l = l;
        if (q0l >= 0) {
            cudaEvent_t ef = P->ev[P->ev_next];
            P->ev_next = (P->ev_next + 1) % 64;
            cudaEventRecord(ef, st);
            cudaStreamWaitEvent(P->aux, ef, 0);
            constexpr size_t qsm = (size_t)kQ0Stages * kQ0StageBytes + 2 * kQ0Stages * 8;
            blb_smem_optin(k_mac_q0, qsm);
            const unsigned gq = (unsigned)(((n_o + 1) / 2) * (size_t)(P->N / 512));
            k_mac_q0<<<gq, kQ0Cons + 32, qsm, P->aux>>>(ptb, R, acc, pl->d_ent, pl->d_ent_start, o0, e_base, n_o, k, q0l,
                                                        P->logN, P->pr, lay);
            BLB_COUNT_LAUNCH(1);
        }
        if (grouped)
            launch_mac4<BLB_MAC_P, BLB_MAC_STG, BLB_MAC_MINB, BLB_MAC_STGP>(ptb, R, acc, pl->d_ent, pl->d_ent_start, o0,
                                                                            e_base, n_o, k, P->logN, P->pr, n_tiles,
                                                                            lay, st, q0l);
        else
            launch_mac4<1, 4, 3>(ptb, R, acc, pl->d_ent, pl->d_ent_start, o0, e_base, n_o, k, P->logN, P->pr,
                                 n_tiles, lay, st);
        if (q0l >= 0) {
            cudaEvent_t ej = P->ev[P->ev_next];
            P->ev_next = (P->ev_next + 1) % 64;
            cudaEventRecord(ej, P->aux);
            cudaStreamWaitEvent(st, ej, 0);
        }
        BLB_COUNT_LAUNCH(1);
        BLB_COUNT(3, n_entries);
        blb_timing_end(0, t0, st, (double)n_entries * (double)lay.bpp);  // packed plaintext bytes
        BLB_CHECK_LAUNCH();
    }
    return BLB_OK;
}

// Phase B (rows a4 + a5): giant steps of the outputs [out_first, out_first + out_count) from their
// accumulators acc[t][g] (reading C11: lazy giant sum in Q_l u P, one fused ModDown + rescale per
// output, C17; outputs without giant steps are rescaled directly).
static blb_status mm_finish(const blb_matmul_plan *pl, const blb_keys *keys, const u64 *acc, int out_first,
                            int out_count, double scale, blb_ct *out, u64 *W, const MatmulWs &w, cudaStream_t st) {
    const blb_params *P = pl->P;
    const int level = pl->level, k = level + 1, N = P->N, E = k + P->np, beta = blb_beta(P, level);
    u64 *gext = W + w.gext, *rot = W + w.rot, *resc = W + w.resc, *gcoef = W + w.gcoef, *yext = W + w.yext;
    u64 *gks_conv = W + w.gks + (size_t)kMaxJobs * 2 * E * N;
    const size_t ctN = (size_t)2 * k * N;
    auto find_key = [&](int32_t step) { return mm_key(P, keys, step); };
    cudaStream_t sa = st;
    const int c0 = 0, cn = out_count;
    {
        // giant steps (reading C11, lazy ModDown): Y[b'] = lift(acc[b'][0]) + sum_g Rot_ext(acc[b'][g])
        // in Q_l u P, then ONE ModDown per output; g-major so outputs sharing a key are adjacent
        std::vector<int> yslot(cn, -1);
        int n_y = 0;
        for (int t = c0; t < c0 + cn; t++)
            if (!pl->giant[out_first + t].empty()) {
                yslot[t - c0] = n_y;
                BLB_TRY(launch_lift_ext(P, level, acc + (size_t)t * pl->G * ctN, yext + (size_t)n_y * 2 * E * N, sa));
                n_y++;
            }
        struct GJob {
            int t, g;
        };
        std::vector<GJob> gj;
        for (int g = 1; g < pl->G; g++)
            for (int t = c0; t < c0 + cn; t++)
                if (std::binary_search(pl->giant[out_first + t].begin(), pl->giant[out_first + t].end(), g))
                    gj.push_back({t, g});
        const int gb = kIndepBatch;
        for (size_t j0 = 0; j0 < gj.size(); j0 += gb) {
            const int cnt = (int)std::min<size_t>(gb, gj.size() - j0);
            std::vector<const u64 *> c1(cnt);
            std::vector<KsJob> jobs(cnt);
            AccJobs aj{};
            aj.n = cnt;
            for (int j = 0; j < cnt; j++) {
                const GJob &G = gj[j0 + j];
                const u64 *a = acc + ((size_t)G.t * pl->G + G.g) * ctN;
                c1[j] = a + (size_t)k * N;
                KsJob J{};
                J.ext = gext + (size_t)j * beta * E * N;
                J.key = find_key(G.g * pl->B * pl->L);
                J.c0 = a;
                J.out = rot + (size_t)j * 2 * E * N;
                J.galois = blb_galois_element(P, G.g * pl->B * pl->L);
                jobs[j] = J;
                aj.dst[j] = yext + (size_t)yslot[G.t - c0] * 2 * E * N;
                aj.src[j] = J.out;
            }
            BLB_TRY(launch_modup(P, level, c1.data(), cnt, gext, gcoef, sa));
            BLB_TRY(launch_keyswitch_ext(P, level, jobs.data(), cnt, sa));
            k_accumulate<<<dim3((N + kTB - 1) / kTB, E, 2), kTB, 0, sa>>>(aj, P->pr, E, N, k, P->K);
            BLB_COUNT_LAUNCH(1);
            BLB_CHECK_LAUNCH();
        }
        // ModDown + rescale as one exact rounding (reading C17); outputs without giant steps are
        // rescaled directly (round(P x / (q_l P)) = round(x / q_l), pinned in the oracle tests)
        std::vector<u64 *> youts;
        for (int t = c0; t < c0 + cn; t++) {
            if (yslot[t - c0] >= 0) youts.push_back(out[t].data);
            else BLB_TRY(launch_rescale(P, acc + (size_t)t * pl->G * ctN, level, 2, out[t].data, resc, sa));
            out[t].level = level - 1;
            out[t].scale = scale;  // Delta * q_level / q_level, exact (reading S6)
        }
        if (n_y > 0) BLB_TRY(launch_moddown_rescale(P, level, yext, n_y, youts.data(), gks_conv, sa));
    }
    return BLB_OK;
}

extern "C" blb_status blb_ct_pt_matmul(const blb_matmul_plan *pl, const blb_keys *keys, const blb_ct *in, int n_in,
                                       const u64 *pt_dev, int out_first, int out_count, blb_ct *out, void *ws,
                                       size_t ws_bytes, void *stream) {
    if (!pl || !keys || !in || !pt_dev || !out || !ws) {
        blb_set_error("blb_ct_pt_matmul: null argument");
        return BLB_E_INVALID_ARG;
    }
    BLB_TRY(check_slice(pl, out_first, out_count));
    if (pl->i_first != 0 || pl->i_count != pl->B) {
        blb_set_error("blb_ct_pt_matmul: a windowed plan needs blb_ct_pt_matmul_acc + blb_ct_pt_matmul_finish");
        return BLB_E_INVALID_ARG;
    }
    BLB_TRY(mm_check(pl, keys, in, n_in, true, true));
    for (int t = 0; t < out_count; t++)
        if (!out[t].data) return BLB_E_INVALID_ARG;
    const MatmulWs w = matmul_ws(pl, out_count);
    if (ws_bytes < w.total * sizeof(u64)) {
        blb_set_error("workspace too small: %zu < %zu", ws_bytes, w.total * sizeof(u64));
        return BLB_E_NOMEM;
    }
    u64 *W = (u64 *)ws;
    cudaStream_t st = (cudaStream_t)stream;
    BLB_TRY(mm_acc(pl, keys, in, pt_dev, out_first, out_count, W + w.acc, W, w, st));
    return mm_finish(pl, keys, W + w.acc, out_first, out_count, in[0].scale, out, W, w, st);
}

extern "C" blb_status blb_ct_pt_matmul_batch(const blb_matmul_plan *pl, const blb_keys *keys, const blb_ct *in,
                                             int n_in, int n_batch, const u64 *pt_dev, int out_first, int out_count,
                                             blb_ct *out, void *ws, size_t ws_bytes, void *stream) {
    if (!pl || !keys || !in || !pt_dev || !out || !ws || n_batch < 1) {
        blb_set_error("blb_ct_pt_matmul_batch: null argument or n_batch < 1");
        return BLB_E_INVALID_ARG;
    }
    BLB_TRY(check_slice(pl, out_first, out_count));
    if (pl->i_first != 0 || pl->i_count != pl->B) {
        blb_set_error("blb_ct_pt_matmul_batch: windowed plans are not supported");
        return BLB_E_INVALID_ARG;
    }
    for (int b = 0; b < n_batch; b++) BLB_TRY(mm_check(pl, keys, in + (size_t)b * n_in, n_in, true, true));
    for (int t = 0; t < n_batch * out_count; t++)
        if (!out[t].data) return BLB_E_INVALID_ARG;
    const MatmulWs w = matmul_ws(pl, out_count);
    if (ws_bytes < (size_t)n_batch * w.total * sizeof(u64)) {
        blb_set_error("workspace too small: %zu < %zu", ws_bytes, (size_t)n_batch * w.total * sizeof(u64));
        return BLB_E_NOMEM;
    }
    u64 *W = (u64 *)ws;
    cudaStream_t st = (cudaStream_t)stream;
    const blb_params *P = pl->P;
    // 1-2 per input set: ModUp and the baby-step rotations into its own R
    for (int b = 0; b < n_batch; b++) {
        u64 *Wb = W + (size_t)b * w.total;
        BLB_TRY(mm_acc(pl, keys, in + (size_t)b * n_in, pt_dev, out_first, out_count, Wb + w.acc, Wb, w, st, false));
    }
    // 3. one weight-stationary MAC for all input sets
    const int k = pl->level + 1, N = P->N;
    const int o0 = out_first * pl->G, n_o = out_count * pl->G;
    const int e_base = pl->ent_start[o0];
    const int n_entries = pl->ent_start[o0 + n_o] - e_base;
    if (n_o > 0 && n_entries == 0) {
        for (int b = 0; b < n_batch; b++)
            BLB_CUDA_TRY(cudaMemsetAsync(W + (size_t)b * w.total + w.acc, 0, sizeof(u64) * (size_t)n_o * 2 * k * N, st));
    } else if (n_o > 0) {
        const int n_tiles = N / (2 * kTB);
        const PtLayout lay = pt_layout(pl);
        constexpr size_t smem = macb_smem();
        blb_smem_optin(k_mac_tma4b, smem);
        cudaEvent_t t0 = blb_timing_begin(st);
        const size_t grid = (size_t)n_o * n_tiles * k * ((n_batch + kMbB - 1) / kMbB);
        k_mac_tma4b<<<(unsigned)grid, kTB + 32, smem, st>>>(reinterpret_cast<const unsigned char *>(pt_dev), W + w.R,
                                                            (long long)w.total, W + w.acc, (long long)w.total, n_batch,
                                                            pl->d_ent, pl->d_ent_start, o0, e_base, n_o, k, P->logN, P->pr,
                                                            lay);
        BLB_COUNT_LAUNCH(1);
        BLB_COUNT(3, (long long)n_entries * n_batch);
        blb_timing_end(0, t0, st, (double)n_entries * (double)lay.bpp);  // packed plaintext bytes (read once)
        BLB_CHECK_LAUNCH();
    }
    // 4-5 per input set: giant steps, fused ModDown + rescale
    for (int b = 0; b < n_batch; b++) {
        u64 *Wb = W + (size_t)b * w.total;
        BLB_TRY(mm_finish(pl, keys, Wb + w.acc, out_first, out_count, in[(size_t)b * n_in].scale,
                          out + (size_t)b * out_count, Wb, w, st));
    }
    return BLB_OK;
}

extern "C" blb_status blb_ct_pt_matmul_acc(const blb_matmul_plan *pl, const blb_keys *keys, const blb_ct *in,
                                           int n_in, const u64 *pt_dev, u64 *acc_out, void *ws, size_t ws_bytes,
                                           void *stream) {
    if (!pl || !keys || !in || !pt_dev || !acc_out || !ws) {
        blb_set_error("blb_ct_pt_matmul_acc: null argument");
        return BLB_E_INVALID_ARG;
    }
    BLB_TRY(mm_check(pl, keys, in, n_in, true, false));
    const MatmulWs w = matmul_ws(pl, 0);
    if (ws_bytes < w.total * sizeof(u64)) {
        blb_set_error("workspace too small: %zu < %zu", ws_bytes, w.total * sizeof(u64));
        return BLB_E_NOMEM;
    }
    return mm_acc(pl, keys, in, pt_dev, 0, pl->n_out, acc_out, (u64 *)ws, w, (cudaStream_t)stream);
}

extern "C" blb_status blb_ct_pt_matmul_finish(const blb_matmul_plan *pl, const blb_keys *keys, const u64 *acc_in,
                                              int out_first, int out_count, double scale, blb_ct *out, void *ws,
                                              size_t ws_bytes, void *stream) {
    if (!pl || !keys || (out_count > 0 && (!acc_in || !out)) || !ws) {
        blb_set_error("blb_ct_pt_matmul_finish: null argument");
        return BLB_E_INVALID_ARG;
    }
    BLB_TRY(check_slice(pl, out_first, out_count));
    BLB_TRY(mm_check(pl, keys, nullptr, 0, false, true));
    for (int t = 0; t < out_count; t++)
        if (!out[t].data) return BLB_E_INVALID_ARG;
    const MatmulWs w = matmul_ws(pl, out_count);
    if (ws_bytes < w.total * sizeof(u64)) {
        blb_set_error("workspace too small: %zu < %zu", ws_bytes, w.total * sizeof(u64));
        return BLB_E_NOMEM;
    }
    if (out_count == 0) return BLB_OK;
    u64 *W = (u64 *)ws;
    cudaStream_t st = (cudaStream_t)stream;
    const int k = pl->level + 1, N = pl->P->N;
    const long long n_polys = (long long)out_count * pl->G * 2;
    k_reduce_acc<<<dim3((N + kTB - 1) / kTB, k, (unsigned)std::min<long long>(n_polys, 1024)), kTB, 0, st>>>(
        acc_in, W + w.acc, pl->P->pr, k, N, n_polys);
    BLB_COUNT_LAUNCH(1);
    BLB_CHECK_LAUNCH();
    return mm_finish(pl, keys, W + w.acc, out_first, out_count, scale, out, W, w, st);
}
