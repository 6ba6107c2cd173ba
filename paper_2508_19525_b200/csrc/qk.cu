#include <array>
// qk.cu -- BLB's rotation-efficient ct-ct MatMul Q_h K_h^T for all heads (row a7).
//
// Sec. 5.1: Observations 1-2, the three steps, multi-head packing
// (MHP) and BSGS with the giant step deferred into step 3 (App. C.1,
// P:1203-1207); the masks follow DESIGN.md reading C13 (the paper's figures are
// elided).  With t = u*B + i:
//   K'_i  = sum_c Mnw_{c,i} (.) Rot_s(K) + Mw_{c,i} (.) Rot_{s-L}(K),  s = (c+i) mod L   (hoisted)
//   Q_u   = Mq_{u,hi} (.) Rot_{-uB}(Q) + Mq_{u,lo} (.) Rot_{L-uB}(Q)                     (hoisted)
//   S_ui  = rescale(relin(sum_j Q_u^(j) (x) K'_i^(j)))
//   T_ui  = Rot_{-i H_p L}(S_ui)
//   A_uwf = rescale(sum_i M3_{u,i,w,f} (.) T_ui);  out[(uB + wg) mod L / g] += Rot_{uB or uB-L}(A_uwf)
// GPU mapping: every mask stage is one launch of the MAC kernel (masks are
// plaintexts shared by all J ciphertexts), all rotations of one ciphertext
// share one ModUp, independent rotations / relinearisations run 32 key
// switches per launch group, the J-sum of the tensor products is one kernel
// with 128-bit lazy accumulation, rescales are batched over all ciphertexts
// of a stage.
#include <algorithm>
#include <map>
#include <set>
#include <type_traits>
#include "blb_internal.cuh"

extern "C" uint32_t blb_galois_element(const blb_params *P, int32_t step);

struct MaskDesc {
    int type;  // 0: K (c, i, wrap)  1: Q (u, low)  2: step 3 (u, i, w, f)
    int a, b, c, d;
};

struct blb_qk_plan {
    const blb_params *P;
    int L, H, Hp, dh, n, g, J, B, G, level;
    int iw0 = 0, iw1 = 0;                        // baby-index window [iw0, iw1) of this rank (section 8(e))
    std::vector<int32_t> k_rots, q_rots;         // non-zero left rotations (slots)
    std::vector<int> kw_slot;                    // kr indices (1 + k_rots index) the window's K' entries use
    std::vector<int> out_acc_start;              // CSR over outputs of the (output-sorted) accumulators
    std::vector<MaskDesc> m1, m3;                // stage-1 masks (level), stage-3 masks (level-2)
    // MAC entry lists (CSR): K' outputs o = i*J + j; Q outputs o = (u-1)*J + j; A outputs = accumulators
    std::vector<int> kp_start, kp_r, kp_pt, qp_start, qp_r, qp_pt, a_start, a_r, a_pt;
    std::vector<int> aw_start, aw_r, aw_pt;      // step-3 entries of the window's i only
    struct Acc {
        int u, w, f, out, rot;
    };
    std::vector<Acc> accs;
    std::vector<int32_t> steps;
    int *d_ent = nullptr;  // all entry arrays, device
    size_t off_kp_start, off_kp_r, off_kp_pt, off_qp_start, off_qp_r, off_qp_pt, off_a_start, off_a_r, off_a_pt;
    size_t off_aw_start, off_aw_r, off_aw_pt;
    MaskDesc *d_m1 = nullptr, *d_m3 = nullptr;
};

namespace {
constexpr int kTB = 256;

struct QKDev {
    int L, Hp, g, B, n;
};
__global__ void k_mask_slots(const MaskDesc *descs, int m0, QKDev q, double *slots) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    const int e = blockIdx.y;
    if (s >= q.n) return;
    const MaskDesc D = descs[m0 + e];
    const int blk = s / q.L, p = s - blk * q.L, c = blk / q.Hp;
    bool v = false;
    if (D.type == 0) {
        const int sh = (D.a + D.b) % q.L;
        v = (c == D.a) && (D.c ? (p + sh >= q.L) : (p + sh < q.L));
    } else if (D.type == 1) {
        const int a = D.a * q.B;
        v = D.b ? (p < a) : (p >= a);
    } else {
        const int i = D.b;
        const int cc = ((c - i) % q.g + q.g) % q.g;
        const int w = (cc + i) / q.g;
        const int a = D.a * q.B;
        v = (w == D.c) && (D.d == 0 ? (p >= a) : (p < a));
    }
    slots[(long long)e * q.n + s] = v ? 1.0 : 0.0;
}

// the J-sum in chunks of 4: the 16 loads of a chunk are issued before its first multiply (a runtime-J
// loop exposed one load latency per j); missing j of the last chunk contribute 0 * 0
#define TSUM_LOOP                                                                  \
    for (int j0 = 0; j0 < J; j0 += 4) {                                            \
        u64 a0[4], a1[4], b0[4], b1[4];                                            \
        _Pragma("unroll") for (int jj = 0; jj < 4; jj++) {                         \
            a0[jj] = a1[jj] = b0[jj] = b1[jj] = 0;                                 \
            if (j0 + jj < J) {                                                     \
                const u64 *a = Qp + (long long)(u * J + j0 + jj) * 2 * kN + lx;    \
                const u64 *b = Kp + (long long)(i * J + j0 + jj) * 2 * kN + lx;    \
                a0[jj] = a[0]; a1[jj] = a[kN]; b0[jj] = b[0]; b1[jj] = b[kN];      \
            }                                                                      \
        }                                                                          \
        _Pragma("unroll") for (int jj = 0; jj < 4; jj++) {                         \
            d0.mac(a0[jj], b0[jj]);                                                \
            d1.mac(a0[jj], b1[jj]);                                                \
            d1.mac(a1[jj], b0[jj]);                                                \
            d2.mac(a1[jj], b1[jj]);                                                \
        }                                                                          \
    }
// D[o][0..2] = sum_j (a0 b0, a0 b1 + a1 b0, a1 b1) with a = Qp[u*J + j], b = Kp[i*J + j], o = u*B + i.
// 1-D grid with the output o fastest: the CTAs in flight cover all (u, i) of a few (tile, limb)
// slices, so each Q_u / K'_i tile is read from DRAM once and reused through L2 (B and G times).
// Window form: local outputs o = u * Bw + (i - iw0) for i in [iw0, iw0 + Bw), written at u * B + i.
__global__ void k_tensor_sum(const u64 *Qp, const u64 *Kp, u64 *D, Primes pr, int J, int B, int k, int N,
                             int n_o, int iw0, int Bw) {
    int bid = blockIdx.x;
    const int ol = bid % n_o;
    bid /= n_o;
    const int l = bid % k;
    const int x = (bid / k) * blockDim.x + threadIdx.x;
    if (x >= N) return;
    const int u = ol / Bw, i = iw0 + (ol - u * Bw);
    const int o = u * B + i;
    const long long kN = (long long)k * N, lx = (long long)l * N + x;
    const ModConst &mc = pr.m[l];
    u64 *out = D + (long long)o * 3 * kN + lx;
    if (mc.q < (1ull << 41)) {
        Acc41 d0, d1, d2;
        d0.zero(); d1.zero(); d2.zero();
        TSUM_LOOP
        out[0] = d0.reduce(mc);
        out[kN] = d1.reduce(mc);
        out[2 * kN] = d2.reduce(mc);
        return;
    }
    Acc128 d0, d1, d2;
    d0.zero(); d1.zero(); d2.zero();
    TSUM_LOOP
    out[0] = d0.reduce(mc);
    out[kN] = d1.reduce(mc);
    out[2 * kN] = d2.reduce(mc);
}
#undef TSUM_LOOP

// 2 x 2 register-blocked J-sum: a thread owns one coefficient of the four outputs (u0 + du, i0 + di),
// so each Q_u / K'_i word it loads feeds two outputs (half the L2 -> SM traffic of k_tensor_sum, which
// is what bounds it: the whole J-sum is ~1.5 GB of DRAM but 8.6 GB of L2 reads one output at a time).
// Grid: (block (u0/2, i0/2) fastest, limb, x-tile).
// SMALL (q < 2^41): every product on the grid-split FP64 accumulator (AccG, 4 FP64 ops per product,
// each loaded word converted to a double once).  Otherwise Acc128 throughout.
template <bool SMALL>
__device__ __forceinline__ void tsum22_body(const u64 *Qp, const u64 *Kp, u64 *D, int J, int B, long long kN,
                                            long long lx, int u0, int i0, const ModConst &mc) {
    if constexpr (SMALL) {
        const double qd = (double)mc.q, qinv = 1.0 / qd;
        AccG d0[2][2], d1[2][2], d2[2][2];  // 2 J <= 512 products per accumulator
#pragma unroll
        for (int a = 0; a < 2; a++)
#pragma unroll
            for (int b = 0; b < 2; b++) { d0[a][b].zero(); d1[a][b].zero(); d2[a][b].zero(); }
        for (int j = 0; j < J; j++) {
            double q0[2], q1[2], k0[2], k1[2];
#pragma unroll
            for (int a = 0; a < 2; a++) {
                const u64 *qa = Qp + (long long)((u0 + a) * J + j) * 2 * kN + lx;
                const u64 *kb = Kp + (long long)((i0 + a) * J + j) * 2 * kN + lx;
                q0[a] = AccF64::u2d(qa[0]); q1[a] = AccF64::u2d(qa[kN]);
                k0[a] = AccF64::u2d(kb[0]); k1[a] = AccF64::u2d(kb[kN]);
            }
#pragma unroll
            for (int a = 0; a < 2; a++)
#pragma unroll
                for (int b = 0; b < 2; b++) {
                    d0[a][b].macd(q0[a], k0[b]);
                    d2[a][b].macd(q1[a], k1[b]);
                    d1[a][b].macd(q0[a], k1[b]);
                    d1[a][b].macd(q1[a], k0[b]);
                }
        }
#pragma unroll
        for (int a = 0; a < 2; a++)
#pragma unroll
            for (int b = 0; b < 2; b++) {
                u64 *out = D + (long long)((u0 + a) * B + i0 + b) * 3 * kN + lx;
                out[0] = d0[a][b].reduce(qd, qinv);
                out[kN] = d1[a][b].reduce(qd, qinv);
                out[2 * kN] = d2[a][b].reduce(qd, qinv);
            }
    } else {
    Acc128 d0[2][2], d1[2][2], d2[2][2];
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
        for (int b = 0; b < 2; b++) { d0[a][b].zero(); d1[a][b].zero(); d2[a][b].zero(); }
    for (int j = 0; j < J; j++) {
        u64 q0[2], q1[2], k0[2], k1[2];
#pragma unroll
        for (int a = 0; a < 2; a++) {
            const u64 *qa = Qp + (long long)((u0 + a) * J + j) * 2 * kN + lx;
            const u64 *kb = Kp + (long long)((i0 + a) * J + j) * 2 * kN + lx;
            q0[a] = qa[0]; q1[a] = qa[kN]; k0[a] = kb[0]; k1[a] = kb[kN];
        }
#pragma unroll
        for (int a = 0; a < 2; a++)
#pragma unroll
            for (int b = 0; b < 2; b++) {
                d0[a][b].mac(q0[a], k0[b]);
                d2[a][b].mac(q1[a], k1[b]);
                d1[a][b].mac(q0[a], k1[b]);
                d1[a][b].mac(q1[a], k0[b]);
            }
    }
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
        for (int b = 0; b < 2; b++) {
            u64 *out = D + (long long)((u0 + a) * B + i0 + b) * 3 * kN + lx;
            out[0] = d0[a][b].reduce(mc);
            out[kN] = d1[a][b].reduce(mc);
            out[2 * kN] = d2[a][b].reduce(mc);
        }
    }
}
__global__ void __launch_bounds__(kTB, 2) k_tensor_sum22(const u64 *Qp, const u64 *Kp, u64 *D, Primes pr, int J, int G,
                                                      int B, int k, int N, int iw0, int Bw) {
    const int nb = (G / 2) * (Bw / 2);
    int bid = blockIdx.x;
    const int ob = bid % nb;
    bid /= nb;
    const int l = bid % k;
    const int x = (bid / k) * blockDim.x + threadIdx.x;
    if (x >= N) return;
    const int u0 = 2 * (ob / (Bw / 2)), i0 = iw0 + 2 * (ob % (Bw / 2));
    const long long kN = (long long)k * N, lx = (long long)l * N + x;
    const ModConst &mc = pr.m[l];
    // AccG holds <= 512 products (2 J per accumulator here); Acc128 <= 64 products of 61-bit residues
    if (mc.q < (1ull << 41)) tsum22_body<true>(Qp, Kp, D, J, B, kN, lx, u0, i0, mc);
    else tsum22_body<false>(Qp, Kp, D, J, B, kN, lx, u0, i0, mc);
}

// dst[p][i][x] = src[p][i][x] for i < k_dst (src has k_src limbs per poly): exact level drop / copy
__global__ void k_copy_limbs(const u64 *src, u64 *dst, int k_src, int k_dst, int N) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y, p = blockIdx.z;
    if (x >= N) return;
    dst[((long long)p * k_dst + i) * N + x] = src[((long long)p * k_src + i) * N + x];
}

struct SumList {
    int n;
    const u64 *src[64];
};
// out = sum of the listed ciphertexts ([2][k][N] each; limbs l >= kq are special primes K + l - kq)
__global__ void k_sum_list(SumList sl, u64 *out, Primes pr, int k, int N, int kq, int K) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int l = blockIdx.y, p = blockIdx.z;
    if (x >= N) return;
    const long long off = ((long long)p * k + l) * N + x;
    const u64 q = pr.m[l < kq ? l : K + (l - kq)].q;
    u64 acc = 0;
    for (int t = 0; t < sl.n; t++) acc = addmod(acc, sl.src[t][off], q);
    out[off] = acc;
}
inline dim3 gx(int N, int y, int z) { return dim3((N + kTB - 1) / kTB, y, z); }
}  // namespace

// ---------------------------------------------------------------- plan
static int wrap_class(int cprime, int i, int g) {
    const int c = ((cprime - i) % g + g) % g;
    return (c + i) / g;
}

extern "C" void blb_qk_plan_destroy(blb_qk_plan *pl) {
    if (!pl) return;
    cudaFree(pl->d_ent);
    cudaFree(pl->d_m1);
    cudaFree(pl->d_m3);
    delete pl;
}

extern "C" blb_status blb_qk_plan_create(const blb_params *P, int L, int heads, int d_h, int bsgs_B, int level,
                                         blb_qk_plan **out) {
    return blb_qk_plan_create_window(P, L, heads, d_h, bsgs_B, level, 0, -1, out);
}

extern "C" blb_status blb_qk_plan_create_window(const blb_params *P, int L, int heads, int d_h, int bsgs_B, int level,
                                                int i_first, int i_count, blb_qk_plan **out) {
    if (!P || !out || L <= 0 || heads <= 0 || d_h <= 0) return BLB_E_INVALID_ARG;
    const int n = P->N / 2;
    int Hp = 1;
    while (Hp < heads) Hp <<= 1;
    if (n % (L * Hp)) {
        blb_set_error("MHP needs L * H_p | N/2 (L=%d, H_p=%d, n=%d)", L, Hp, n);
        return BLB_E_LAYOUT;
    }
    const int g = n / (L * Hp);
    const int B = bsgs_B > 0 ? bsgs_B : g;
    if (B % g || L % B) {
        blb_set_error("ct-ct BSGS needs g | B | L (g=%d, B=%d, L=%d)", g, B, L);
        return BLB_E_LAYOUT;
    }
    if (level < 3 || level >= P->K) {
        blb_set_error("ct-ct MatMul consumes 3 levels: input level %d must be in [3, %d)", level, P->K);
        return BLB_E_LEVEL;
    }
    if (i_count < 0) i_count = B - i_first;
    if (i_first < 0 || i_count < 1 || i_first + i_count > B) {
        blb_set_error("blb_qk_plan_create_window: window [%d, %d) outside [0, B = %d)", i_first, i_first + i_count, B);
        return BLB_E_INVALID_ARG;
    }
    auto *pl = new blb_qk_plan();
    pl->P = P; pl->L = L; pl->H = heads; pl->Hp = Hp; pl->dh = d_h; pl->n = n; pl->g = g;
    pl->J = (d_h + g - 1) / g; pl->B = B; pl->G = L / B; pl->level = level;
    pl->iw0 = i_first; pl->iw1 = i_first + i_count;
    std::set<int32_t> ks, qs;
    for (int c = 0; c < g; c++)
        for (int i = 0; i < B; i++) {
            const int s = (c + i) % L;
            if (s) { ks.insert(s); ks.insert(s - L); }
        }
    for (int u = 1; u < pl->G; u++) { qs.insert(-u * B); qs.insert(L - u * B); }
    pl->k_rots.assign(ks.begin(), ks.end());
    pl->q_rots.assign(qs.begin(), qs.end());
    const int NKR = 1 + (int)pl->k_rots.size();
    auto kr_index = [&](int32_t r) -> int {
        if (r == 0) return 0;
        return 1 + (int)(std::lower_bound(pl->k_rots.begin(), pl->k_rots.end(), r) - pl->k_rots.begin());
    };
    const int NQR = (int)pl->q_rots.size();
    auto qr_index = [&](int32_t r) -> int {
        return (int)(std::lower_bound(pl->q_rots.begin(), pl->q_rots.end(), r) - pl->q_rots.begin());
    };
    // stage-1 masks: K (c, i, wrap), then Q (u, low)
    std::map<std::tuple<int, int, int>, int> kmask;
    for (int i = 0; i < B; i++)
        for (int c = 0; c < g; c++) {
            const int s = (c + i) % L;
            for (int wrap = 0; wrap < (s ? 2 : 1); wrap++) {
                kmask[{c, i, wrap}] = (int)pl->m1.size();
                pl->m1.push_back({0, c, i, wrap, 0});
            }
        }
    std::map<std::pair<int, int>, int> qmask;
    for (int u = 1; u < pl->G; u++)
        for (int low = 0; low < 2; low++) {
            qmask[{u, low}] = (int)pl->m1.size();
            pl->m1.push_back({1, u, low, 0, 0});
        }
    // K' MAC: output o = i*J + j, entries over c (and wrap), R = Kr[j][kr_index(r)]
    pl->kp_start.push_back(0);
    for (int i = 0; i < B; i++)
        for (int j = 0; j < pl->J; j++) {
            for (int c = 0; c < g; c++) {
                const int s = (c + i) % L;
                for (int wrap = 0; wrap < (s ? 2 : 1); wrap++) {
                    const int r = wrap ? s - L : s;
                    pl->kp_r.push_back(j * NKR + kr_index(r));
                    pl->kp_pt.push_back(kmask[{c, i, wrap}]);
                }
            }
            pl->kp_start.push_back((int)pl->kp_r.size());
        }
    // Q MAC: output o = (u-1)*J + j, two entries
    pl->qp_start.push_back(0);
    for (int u = 1; u < pl->G; u++)
        for (int j = 0; j < pl->J; j++) {
            const int a = u * B;
            pl->qp_r.push_back(j * NQR + qr_index(-a));
            pl->qp_pt.push_back(qmask[{u, 0}]);
            pl->qp_r.push_back(j * NQR + qr_index(L - a));
            pl->qp_pt.push_back(qmask[{u, 1}]);
            pl->qp_start.push_back((int)pl->qp_r.size());
        }
    // K rotations the window's K' entries use (every j uses the same ones)
    {
        std::set<int> used;
        for (int o = pl->iw0 * pl->J; o < pl->iw1 * pl->J; o++)
            for (int e = pl->kp_start[o]; e < pl->kp_start[o + 1]; e++) used.insert(pl->kp_r[e] % NKR);
        used.erase(0);  // the lift
        pl->kw_slot.assign(used.begin(), used.end());
    }
    // step 3: accumulators (u, w, f) with a non-zero mask
    const int wmax = (g - 1 + B - 1) / g;
    pl->a_start.push_back(0);
    pl->aw_start.push_back(0);
    for (int u = 0; u < pl->G; u++)
        for (int w = 0; w <= wmax; w++)
            for (int f = 0; f < 2; f++) {
                const int a = u * B;
                std::vector<int> terms;
                for (int i = 0; i < B; i++) {
                    bool any_block = false;
                    for (int cp = 0; cp < g && !any_block; cp++) any_block = wrap_class(cp, i, g) == w;
                    const bool any_pos = f == 0 ? (a < L) : (a > 0);
                    if (any_block && any_pos) terms.push_back(i);
                }
                if (terms.empty()) continue;
                for (int i : terms) {
                    pl->a_r.push_back(u * B + i);
                    pl->a_pt.push_back((int)pl->m3.size());
                    if (i >= pl->iw0 && i < pl->iw1) {
                        pl->aw_r.push_back(u * B + i);
                        pl->aw_pt.push_back((int)pl->m3.size());
                    }
                    pl->m3.push_back({2, u, i, w, f});
                }
                pl->a_start.push_back((int)pl->a_r.size());
                pl->aw_start.push_back((int)pl->aw_r.size());
                const int rot = f == 0 ? u * B : u * B - L;
                pl->accs.push_back({u, w, f, ((u * B + w * g) % L) / g, rot});
            }
    // accumulators sorted by output (stable; each accumulator is independent and the per-output
    // sum is an exact modular sum, so the order is bit-neutral): the accumulators of outputs
    // [o0, o1) are the contiguous slots [out_acc_start[o0], out_acc_start[o1])
    {
        const int NA = (int)pl->accs.size(), n_out = L / g;
        std::vector<int> perm(NA);
        for (int a = 0; a < NA; a++) perm[a] = a;
        std::stable_sort(perm.begin(), perm.end(), [&](int x, int y) { return pl->accs[x].out < pl->accs[y].out; });
        auto regroup = [&](std::vector<int> &st_, std::vector<int> &r_, std::vector<int> &pt_) {
            std::vector<int> s2{0}, r2, p2;
            for (int a : perm) {
                for (int e = st_[a]; e < st_[a + 1]; e++) { r2.push_back(r_[e]); p2.push_back(pt_[e]); }
                s2.push_back((int)r2.size());
            }
            st_.swap(s2); r_.swap(r2); pt_.swap(p2);
        };
        regroup(pl->a_start, pl->a_r, pl->a_pt);
        regroup(pl->aw_start, pl->aw_r, pl->aw_pt);
        std::vector<blb_qk_plan::Acc> acc2;
        for (int a : perm) acc2.push_back(pl->accs[a]);
        pl->accs.swap(acc2);
        pl->out_acc_start.assign(n_out + 1, 0);
        for (int a = 0; a < NA; a++) pl->out_acc_start[pl->accs[a].out + 1]++;
        for (int o = 0; o < n_out; o++) pl->out_acc_start[o + 1] += pl->out_acc_start[o];
    }
    // rotation key set
    std::set<int32_t> st(pl->k_rots.begin(), pl->k_rots.end());
    st.insert(pl->q_rots.begin(), pl->q_rots.end());
    for (int i = 1; i < B; i++)
        if ((i * Hp * L) % n) st.insert(-i * Hp * L);  // a multiple of n slots is the identity (lift, no key)
    for (auto &A : pl->accs)
        if (((A.rot % n) + n) % n) st.insert(A.rot);
    pl->steps.assign(st.begin(), st.end());
    // device copies
    std::vector<int> all;
    auto put = [&](const std::vector<int> &v) {
        const size_t o = all.size();
        all.insert(all.end(), v.begin(), v.end());
        return o;
    };
    pl->off_kp_start = put(pl->kp_start); pl->off_kp_r = put(pl->kp_r); pl->off_kp_pt = put(pl->kp_pt);
    pl->off_qp_start = put(pl->qp_start); pl->off_qp_r = put(pl->qp_r); pl->off_qp_pt = put(pl->qp_pt);
    pl->off_a_start = put(pl->a_start); pl->off_a_r = put(pl->a_r); pl->off_a_pt = put(pl->a_pt);
    pl->off_aw_start = put(pl->aw_start); pl->off_aw_r = put(pl->aw_r); pl->off_aw_pt = put(pl->aw_pt);
    cudaError_t e = cudaMalloc(&pl->d_ent, sizeof(int) * std::max<size_t>(all.size(), 1));
    if (e == cudaSuccess) e = cudaMemcpy(pl->d_ent, all.data(), sizeof(int) * all.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&pl->d_m1, sizeof(MaskDesc) * pl->m1.size());
    if (e == cudaSuccess)
        e = cudaMemcpy(pl->d_m1, pl->m1.data(), sizeof(MaskDesc) * pl->m1.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&pl->d_m3, sizeof(MaskDesc) * pl->m3.size());
    if (e == cudaSuccess)
        e = cudaMemcpy(pl->d_m3, pl->m3.data(), sizeof(MaskDesc) * pl->m3.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        blb_set_error("qk plan upload: %s", cudaGetErrorString(e));
        blb_qk_plan_destroy(pl);
        return BLB_E_CUDA;
    }
    *out = pl;
    return BLB_OK;
}

extern "C" blb_status blb_qk_plan_info(const blb_qk_plan *pl, int *J, int *n_out, int *g, int *B, int *G,
                                       int *n_rotations, int *n_masks) {
    if (!pl) return BLB_E_INVALID_ARG;
    if (J) *J = pl->J;
    if (n_out) *n_out = pl->L / pl->g;
    if (g) *g = pl->g;
    if (B) *B = pl->B;
    if (G) *G = pl->G;
    if (n_rotations) {
        int nf = 0;
        for (auto &A : pl->accs)
            if (((A.rot % pl->n) + pl->n) % pl->n) nf++;
        int n3 = 0;  // step-3 rotations by i H_p L slots that are not the identity
        for (int i = 1; i < pl->B; i++) n3 += ((i * pl->Hp * pl->L) % pl->n) != 0;
        *n_rotations = pl->J * (int)(pl->k_rots.size() + pl->q_rots.size()) + pl->G * n3 + nf;
    }
    if (n_masks) *n_masks = (int)(pl->m1.size() + pl->m3.size());
    return BLB_OK;
}

extern "C" blb_status blb_qk_plan_rotations(const blb_qk_plan *pl, int32_t *steps, int *n) {
    if (!pl || !n) return BLB_E_INVALID_ARG;
    const int need = (int)pl->steps.size();
    if (steps) {
        if (*n < need) return BLB_E_INVALID_ARG;
        for (int i = 0; i < need; i++) steps[i] = pl->steps[i];
    }
    *n = need;
    return BLB_OK;
}

static size_t qk_mask_elems(const blb_qk_plan *pl) {
    const size_t N = pl->P->N;
    // stage-1 masks over the extended basis Q_l u P (double hoisting), stage-3 masks over Q_{l-2}
    return pl->m1.size() * (size_t)(pl->level + 1 + pl->P->np) * N + pl->m3.size() * (size_t)(pl->level - 1 + pl->P->np) * N;
}
extern "C" size_t blb_qk_mask_bytes(const blb_qk_plan *pl) { return pl ? qk_mask_elems(pl) * sizeof(u64) : 0; }

namespace {
// the limbs of extended-basis plaintexts whose prime is < 2^41 -> double bits (the mask MACs' format)
__global__ void k_ext_to_f64(u64 *buf, long long n_polys, int E, int kq, int K, int N, Primes pr) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int l = blockIdx.y;
    if (x >= N || pr.m[l < kq ? l : K + (l - kq)].q >= (1ull << 41)) return;
    for (long long p = blockIdx.z; p < n_polys; p += gridDim.z) {
        const long long off = (p * E + l) * N + x;
        buf[off] = (u64)__double_as_longlong((double)buf[off]);
    }
}
}  // namespace

extern "C" blb_status blb_qk_encode_masks(const blb_qk_plan *pl, uint64_t *masks, void *stream) {
    if (!pl || !masks) return BLB_E_INVALID_ARG;
    const blb_params *P = pl->P;
    cudaStream_t st = (cudaStream_t)stream;
    const int chunk = 64;
    double *slots = nullptr, *buf = nullptr;
    int *flag = nullptr;
    BLB_CUDA_TRY(cudaMallocAsync(&slots, sizeof(double) * (size_t)chunk * pl->n, st));
    BLB_CUDA_TRY(cudaMallocAsync(&buf, sizeof(double) * encode_scratch_doubles(P, chunk), st));
    BLB_CUDA_TRY(cudaMallocAsync(&flag, sizeof(int), st));
    BLB_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int), st));
    QKDev qd{pl->L, pl->Hp, pl->g, pl->B, pl->n};
    blb_status s = BLB_OK;
    // stage 1 at level l (scale q_l), stage 3 at level l-2 (scale q_{l-2}): the primes the next rescales drop
    for (int stage = 0; stage < 2 && s == BLB_OK; stage++) {
        const MaskDesc *dm = stage == 0 ? pl->d_m1 : pl->d_m3;
        const int cnt_all = (int)(stage == 0 ? pl->m1.size() : pl->m3.size());
        const int lvl = stage == 0 ? pl->level : pl->level - 2;
        const int npx = P->np;  // both stages act on extended-basis (Q u P) rotations (C13)
        u64 *base = masks + (stage == 0 ? 0 : pl->m1.size() * (size_t)(pl->level + 1 + P->np) * P->N);
        for (int m0 = 0; m0 < cnt_all && s == BLB_OK; m0 += chunk) {
            const int cnt = std::min(chunk, cnt_all - m0);
            k_mask_slots<<<dim3((pl->n + kTB - 1) / kTB, cnt), kTB, 0, st>>>(dm, m0, qd, slots);
            BLB_COUNT_LAUNCH(1);
            s = launch_encode(P, slots, cnt, (double)P->mod[lvl], lvl, base + (size_t)m0 * (lvl + 1 + npx) * P->N, buf,
                              flag, st, npx);
        }
        // opaque mask format: limbs below 2^41 as doubles, read by the FP64 accumulators of the mask MACs
        if (cnt_all > 0 && s == BLB_OK) {
            k_ext_to_f64<<<dim3((P->N + kTB - 1) / kTB, lvl + 1 + npx, (unsigned)std::min(cnt_all, 1024)), kTB, 0, st>>>(
                base, cnt_all, lvl + 1 + npx, lvl + 1, P->K, P->N, P->pr);
            BLB_COUNT_LAUNCH(1);
        }
    }
    cudaFreeAsync(slots, st);
    cudaFreeAsync(buf, st);
    cudaFreeAsync(flag, st);
    BLB_CUDA_TRY(cudaStreamSynchronize(st));
    return s;
}

// workspace layout
struct QKWs {
    size_t kr, qr, kacc, kp, qacc, qp, d, s, sr, t, aacc, ar, arot, oext, ext, coef, ks, resc, total;
};
static QKWs qk_ws(const blb_qk_plan *pl) {
    const blb_params *P = pl->P;
    const size_t N = P->N, k = pl->level + 1, k1 = k - 1, k2 = k - 2, k3 = k - 3;
    const size_t np = P->np, E = k + np, E1 = k1 + np, E2 = k2 + np, E3 = k3 + np, beta = blb_beta(P, pl->level);
    const size_t J = pl->J, B = pl->B, G = pl->G, NA = pl->accs.size();
    const size_t NKR = 1 + pl->k_rots.size(), NQR = pl->q_rots.size();
    QKWs w{};
    size_t o = 0;
    // stage 1 in the extended basis (E limbs), ModDown to k limbs, rescale to k1
    w.kr = o; o += J * NKR * 2 * E * N;
    w.qr = o; o += J * std::max<size_t>(NQR, 1) * 2 * E * N;
    w.kacc = o; o += B * J * 2 * E * N;
    w.kp = o; o += B * J * 2 * k1 * N;
    w.qacc = o; o += (G > 1 ? (G - 1) : 1) * J * 2 * E * N;
    w.qp = o; o += G * J * 2 * k1 * N;
    w.d = o; o += G * B * 3 * k1 * N;
    w.s = o; o += G * B * 2 * E1 * N;      // relinearised products in Q u P (C17)
    w.sr = o; o += G * B * 2 * k2 * N;
    w.t = o; o += G * B * 2 * E2 * N;      // step-3 rotations in Q u P (double hoisting)
    w.aacc = o; o += NA * 2 * E2 * N;
    w.ar = o; o += NA * 2 * k3 * N;
    w.arot = o; o += NA * 2 * E3 * N;      // final rotations in Q u P
    w.oext = o; o += (size_t)(pl->L / pl->g) * 2 * E3 * N;
    w.ext = o; o += (size_t)kMaxJobs * beta * E * N;
    w.coef = o; o += (size_t)kMaxJobs * k * N;
    w.ks = o; o += keyswitch_scratch_elems(P, pl->level, kMaxJobs);
    const size_t maxct = std::max({B * J, G * J, G * B, NA});
    w.resc = o; o += 2 * maxct * (1 + k) * N;
    w.total = o;
    return w;
}
extern "C" size_t blb_qk_workspace_bytes(const blb_qk_plan *pl) { return pl ? qk_ws(pl).total * sizeof(u64) + 256 : 0; }

static const u64 *key_for(const blb_keys *K, uint32_t g) {
    for (size_t i = 0; i < K->galois.size(); i++)
        if (K->galois[i] == g) return K->data[i];
    return nullptr;
}

// rotations of independent inputs (each its own ModUp) kept in Q u P: out[t] [2][E][N]
static blb_status rotate_independent_ext(const blb_params *P, const blb_keys *keys, int level,
                                         const std::vector<const u64 *> &in, const std::vector<int32_t> &steps,
                                         const std::vector<u64 *> &out, u64 *ext, u64 *coef, cudaStream_t st,
                                         bool f64) {
    const int k = level + 1, N = P->N, E = k + P->np, beta = blb_beta(P, level);
    const int ib = kIndepBatch;
    for (size_t t0 = 0; t0 < in.size(); t0 += ib) {
        const int cnt = (int)std::min<size_t>(ib, in.size() - t0);
        std::vector<const u64 *> c1(cnt);
        std::vector<KsJob> jobs(cnt);
        for (int t = 0; t < cnt; t++) {
            c1[t] = in[t0 + t] + (size_t)k * N;
            const uint32_t g = blb_galois_element(P, steps[t0 + t]);
            KsJob J{};
            J.ext = ext + (size_t)t * beta * E * N;
            J.key = key_for(keys, g);
            J.c0 = in[t0 + t];
            J.out = out[t0 + t];
            J.galois = g;
            J.out_f64 = f64 ? 1 : 0;
            jobs[t] = J;
        }
        BLB_TRY(launch_modup(P, level, c1.data(), cnt, ext, coef, st));
        BLB_TRY(launch_keyswitch_ext(P, level, jobs.data(), cnt, st));
    }
    return BLB_OK;
}

static blb_status qk_check(const blb_qk_plan *pl, const blb_keys *keys, const blb_ct *Q, const blb_ct *K, int J) {
    const blb_params *P = pl->P;
    if (Q) {
        if (J != pl->J) {
            blb_set_error("blb_ct_ct_qk: %d ciphertexts per operand, plan needs J = %d", J, pl->J);
            return BLB_E_LAYOUT;
        }
        for (int j = 0; j < J; j++)
            if (Q[j].level != pl->level || K[j].level != pl->level || !Q[j].data || !K[j].data) {
                blb_set_error("blb_ct_ct_qk: operands must be at the plan level %d", pl->level);
                return BLB_E_LEVEL;
            }
    }
    for (int32_t s : pl->steps)  // a step that is a multiple of n is the identity: no key (B > g)
        if (blb_galois_element(P, s) != 1 && !key_for(keys, blb_galois_element(P, s))) {
            blb_set_error("missing rotation key for step %d", s);
            return BLB_E_MISSING_KEY;
        }
    if (!key_for(keys, 0)) {
        blb_set_error("missing relinearisation key");
        return BLB_E_MISSING_KEY;
    }
    return BLB_OK;
}

namespace {
// x mod the prime of limb l (limbs l >= kq of an extended-basis ciphertext are p_{l - kq})
__global__ void k_reduce_ext(const u64 *src, u64 *dst, Primes pr, int E, int kq, int K, int N, long long n_polys) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int l = blockIdx.y;
    if (x >= N) return;
    const ModConst &mc = pr.m[l < kq ? l : K + (l - kq)];
    for (long long p = blockIdx.z; p < n_polys; p += gridDim.z) {
        const long long off = (p * E + l) * N + x;
        dst[off] = mod64(src[off], mc);
    }
}
}  // namespace

// Phase A: stages 1-3 of reading C13 for the plan's baby-index window [iw0, iw1) -- the window's
// K'_i, every Q_u, the products S_{u,i} (relinearised, rescaled), the step-3 rotations T_{u,i} and
// the step-3 mask MAC into the (output-sorted) accumulators A_{u,w,f} over Q_{l-2} u P, before their
// ModDown + rescale: acc_out [NA][2][E2][N].  Windows of the ranks partition [0, B): the A's of all
// windows sum exactly to those of the whole plan.
static blb_status qk_acc(const blb_qk_plan *pl, const blb_keys *keys, const blb_ct *Q, const blb_ct *K,
                         const uint64_t *masks, u64 *acc_out, u64 *W, const QKWs &w, cudaStream_t st) {
    const blb_params *P = pl->P;
    const int J = pl->J;
    const int lvl = pl->level, k = lvl + 1, k1 = k - 1, k2 = k - 2, N = P->N;
    const int B = pl->B, G = pl->G, NA = (int)pl->accs.size();
    const int iw0 = pl->iw0, Bw = pl->iw1 - pl->iw0;
    const u64 *rlk = key_for(keys, 0);
    const int *E = pl->d_ent;
    const size_t ct_k1 = (size_t)2 * k1 * N, ct_k2 = (size_t)2 * k2 * N;
    const int NKR = 1 + (int)pl->k_rots.size(), NQR = (int)pl->q_rots.size();
    const u64 *m1 = masks, *m3 = masks + pl->m1.size() * (size_t)(k + P->np) * N;

    // 1. baby side, double-hoisted (reading C13): one ModUp per K^(j), the rotations stay in
    //    Q_l u P (no ModDown), the masks are multiplied there, ONE ModDown per K'_i, then rescale
    const int Ex = k + P->np;
    const size_t ct_e = (size_t)2 * Ex * N;
    u64 *conv = W + w.ks;  // ModDown intermediate (kMaxJobs x [2][k][N] fits the key-switch scratch)
    // hoisted rotations of all J ciphertexts of one operand: one ModUp launch for the J inputs, then
    // the jobs step-major (the J rotations by one step are adjacent and share their key: the key
    // switch reads each key once per step instead of once per ciphertext); rotation t of input j is
    // written to base + j * j_stride + slot[t] * ct_e
    auto rotate_ext_J = [&](const blb_ct *cts, const std::vector<int32_t> &steps, const std::vector<int> &slot,
                            u64 *base, size_t j_stride) -> blb_status {
        if (steps.empty()) return BLB_OK;
        const int beta = blb_beta(P, lvl);
        std::vector<const u64 *> c1(J);
        for (int j = 0; j < J; j++) c1[j] = cts[j].data + (size_t)k * N;
        BLB_TRY(launch_modup(P, lvl, c1.data(), J, W + w.ext, W + w.coef, st));
        std::vector<KsJob> jobs;
        for (size_t t = 0; t < steps.size(); t++) {
            const uint32_t g = blb_galois_element(P, steps[t]);
            for (int j = 0; j < J; j++) {
                KsJob Jb{};
                Jb.ext = W + w.ext + (size_t)j * beta * Ex * N;
                Jb.key = key_for(keys, g);
                Jb.c0 = cts[j].data;
                Jb.out = base + j * j_stride + slot[t] * ct_e;
                Jb.galois = g;
                Jb.out_f64 = 1;  // read by the mask MAC (k_mac_j) as doubles
                jobs.push_back(Jb);
            }
        }
        for (size_t t0 = 0; t0 < jobs.size(); t0 += kMaxJobs) {
            const int cnt = (int)std::min<size_t>(kMaxJobs, jobs.size() - t0);
            BLB_TRY(launch_keyswitch_ext(P, lvl, jobs.data() + t0, cnt, st));
        }
        return BLB_OK;
    };
    {
        std::vector<int32_t> ksteps;
        for (int sl : pl->kw_slot) ksteps.push_back(pl->k_rots[sl - 1]);
        for (int j = 0; j < J; j++)
            BLB_TRY(launch_lift_ext(P, lvl, K[j].data, W + w.kr + (size_t)j * NKR * ct_e, st, true));
        BLB_TRY(rotate_ext_J(K, ksteps, pl->kw_slot, W + w.kr, (size_t)NKR * ct_e));
    }
    // K' MAC of the window's outputs o = i*J + j, i in [iw0, iw1) (outputs i*J + j share their masks)
    {
        const int o0 = iw0 * J;
        u64 *kacc = W + w.kacc + (size_t)o0 * ct_e;
        BLB_TRY(launch_mac(P, m1, W + w.kr, kacc, E + pl->off_kp_r, E + pl->off_kp_pt, E + pl->off_kp_start, o0, 0,
                           Bw * J, pl->kp_start[(iw0 + Bw) * J] - pl->kp_start[o0], Ex, st, k, J));
        BLB_TRY(launch_moddown_rescale(P, lvl, kacc, Bw * J, W + w.kp + (size_t)o0 * ct_k1, conv, st));  // C17
    }
    // 2. giant side: Q_0 = level drop, Q_u = ModDown(MAC(masks, Rot_ext(Q))), rescale
    if (NQR) {
        std::vector<int> qslot(NQR);
        for (int t = 0; t < NQR; t++) qslot[t] = t;
        BLB_TRY(rotate_ext_J(Q, pl->q_rots, qslot, W + w.qr, (size_t)NQR * ct_e));
    }
    for (int j = 0; j < J; j++) {
        k_copy_limbs<<<gx(N, k1, 2), kTB, 0, st>>>(Q[j].data, W + w.qp + (size_t)j * ct_k1, k, k1, N);
        BLB_COUNT_LAUNCH(1);
    }
    if (G > 1) {
        BLB_TRY(launch_mac(P, m1, W + w.qr, W + w.qacc, E + pl->off_qp_r, E + pl->off_qp_pt, E + pl->off_qp_start, 0, 0,
                           (G - 1) * J, (int)pl->qp_r.size(), Ex, st, k, J));
        BLB_TRY(launch_moddown_rescale(P, lvl, W + w.qacc, (G - 1) * J, W + w.qp + (size_t)J * ct_k1, conv, st));
    }
    // 3. products summed over j for (u, i in the window), relinearisation (one per (u, i)), rescale
    cudaEvent_t tt0 = blb_timing_begin(st);
    if (G % 2 == 0 && Bw % 2 == 0 && 2 * J <= 64) {
        const unsigned g22 = (unsigned)((size_t)((N + kTB - 1) / kTB) * k1 * (G / 2) * (Bw / 2));
        k_tensor_sum22<<<g22, kTB, 0, st>>>(W + w.qp, W + w.kp, W + w.d, P->pr, J, G, B, k1, N, iw0, Bw);
    } else {
        k_tensor_sum<<<(unsigned)((size_t)((N + kTB - 1) / kTB) * k1 * G * Bw), kTB, 0, st>>>(
            W + w.qp, W + w.kp, W + w.d, P->pr, J, B, k1, N, G * Bw, iw0, Bw);
    }
    // algorithmic bytes: the Q_u and K'_i operands once + the three-component products written
    blb_timing_end(4, tt0, st, ((double)(G + Bw) * J * 2 + (double)G * Bw * 3) * k1 * N * 8.0);
    BLB_COUNT_LAUNCH(1);
    BLB_COUNT(3, (size_t)G * Bw * J);
    BLB_CHECK_LAUNCH();
    // relinearisation kept in Q u P: (P d0 + u0, P d1 + u1), then ModDown + rescale (C17); the
    // window's (u, i) are stored contiguously in w.s (local index u * Bw + i - iw0)
    const int E1 = k1 + P->np, E2 = k2 + P->np;
    std::vector<u64 *> sr_out;
    {
        const int beta1 = blb_beta(P, lvl - 1);
        const int rb = kIndepBatch;
        const int n_ui = G * Bw;
        for (int o0 = 0; o0 < n_ui; o0 += rb) {
            const int cnt = std::min(rb, n_ui - o0);
            std::vector<const u64 *> d2(cnt);
            std::vector<KsJob> jobs(cnt);
            for (int t = 0; t < cnt; t++) {
                const int ol = o0 + t, u = ol / Bw, i = iw0 + ol % Bw;
                const u64 *D = W + w.d + (size_t)(u * B + i) * 3 * k1 * N;
                d2[t] = D + (size_t)2 * k1 * N;
                KsJob Jb{};
                Jb.ext = W + w.ext + (size_t)t * beta1 * E1 * N;
                Jb.key = rlk;
                Jb.c0 = D;
                Jb.c1_add = D + (size_t)k1 * N;
                Jb.out = W + w.s + (size_t)ol * 2 * E1 * N;
                Jb.galois = 1;
                jobs[t] = Jb;
            }
            BLB_TRY(launch_modup(P, lvl - 1, d2.data(), cnt, W + w.ext, W + w.coef, st));
            BLB_TRY(launch_keyswitch_ext(P, lvl - 1, jobs.data(), cnt, st));
        }
        for (int ol = 0; ol < n_ui; ol++) {
            const int u = ol / Bw, i = iw0 + ol % Bw;
            sr_out.push_back(W + w.sr + (size_t)(u * B + i) * ct_k2);
        }
        for (int o0 = 0; o0 < n_ui; o0 += kMaxJobs) {
            const int cnt = std::min(kMaxJobs, n_ui - o0);
            BLB_TRY(launch_moddown_rescale(P, lvl - 1, W + w.s + (size_t)o0 * 2 * E1 * N, cnt, sr_out.data() + o0,
                                           conv, st));
        }
    }
    // 4. step 3: T_ui = Rot_{-i H_p L}(S_ui) kept in Q u P (double hoisting); i = 0 is the lift
    {
        std::vector<const u64 *> in;
        std::vector<int32_t> steps;
        std::vector<u64 *> outp;
        for (int i = iw0; i < iw0 + Bw; i++)  // i-major: the G rotations by the same step share a key
            for (int u = 0; u < G; u++) {
                const size_t o = (size_t)(u * B + i);
                u64 *dst = W + w.t + o * 2 * E2 * N;
                // i = 0, and i H_p L a multiple of n (B > g), rotate by the identity: the lift
                if ((i * pl->Hp * pl->L) % pl->n == 0) {
                    BLB_TRY(launch_lift_ext(P, lvl - 2, W + w.sr + o * ct_k2, dst, st, true));
                    continue;
                }
                in.push_back(W + w.sr + o * ct_k2);
                steps.push_back(-i * pl->Hp * pl->L);
                outp.push_back(dst);
            }
        BLB_TRY(rotate_independent_ext(P, keys, lvl - 2, in, steps, outp, W + w.ext, W + w.coef, st, true));
    }
    // 5. step-3 masks of the window (MAC into the accumulators, Q_{l-2} u P)
    BLB_TRY(launch_mac(P, m3, W + w.t, acc_out, E + pl->off_aw_r, E + pl->off_aw_pt, E + pl->off_aw_start, 0, 0, NA,
                       (int)pl->aw_r.size(), E2, st, k2));
    return BLB_OK;
}

// Phase B: outputs [o0, o0 + n_o) from the (cross-rank summed) accumulators acc of their slots
// [out_acc_start[o0], out_acc_start[o0 + n_o)): (reduce mod the primes of Q_{l-2} u P), ModDown +
// rescale (C17), the deferred giant rotations kept in Q u P, summed per output, one ModDown each.
static blb_status qk_finish(const blb_qk_plan *pl, const blb_keys *keys, const u64 *acc, bool reduce, int o0, int n_o,
                            double sQ, double sK, blb_ct *out, u64 *W, const QKWs &w, cudaStream_t st) {
    const blb_params *P = pl->P;
    const int lvl = pl->level, k = lvl + 1, k2 = k - 2, k3 = k - 3, N = P->N;
    const int E2 = k2 + P->np, E3 = k3 + P->np;
    const size_t ct_k3 = (size_t)2 * k3 * N;
    u64 *conv = W + w.ks;
    const int a0 = pl->out_acc_start[o0], a1 = pl->out_acc_start[o0 + n_o], na = a1 - a0;
    u64 *aacc = W + w.aacc + (size_t)a0 * 2 * E2 * N;
    if (reduce && na > 0) {
        const long long n_polys = (long long)na * 2;
        k_reduce_ext<<<dim3((N + kTB - 1) / kTB, E2, (unsigned)std::min<long long>(n_polys, 1024)), kTB, 0, st>>>(
            acc, aacc, P->pr, E2, k2, P->K, N, n_polys);
        BLB_COUNT_LAUNCH(1);
        BLB_CHECK_LAUNCH();
    } else if (acc != aacc && na > 0) {
        BLB_CUDA_TRY(cudaMemcpyAsync(aacc, acc, sizeof(u64) * (size_t)na * 2 * E2 * N, cudaMemcpyDeviceToDevice, st));
    }
    if (na > 0) BLB_TRY(launch_moddown_rescale(P, lvl - 2, aacc, na, W + w.ar + (size_t)a0 * ct_k3, conv, st));  // C17
    // deferred giant rotations kept in Q u P, summed per output, one ModDown per output
    {
        std::vector<const u64 *> in;
        std::vector<int32_t> steps;
        std::vector<u64 *> outp;
        for (int a = a0; a < a1; a++) {
            const int r = pl->accs[a].rot;
            u64 *dst = W + w.arot + (size_t)a * 2 * E3 * N;
            if (((r % pl->n) + pl->n) % pl->n == 0) {
                BLB_TRY(launch_lift_ext(P, lvl - 3, W + w.ar + (size_t)a * ct_k3, dst, st));
                continue;
            }
            in.push_back(W + w.ar + (size_t)a * ct_k3);
            steps.push_back(r);
            outp.push_back(dst);
        }
        BLB_TRY(rotate_independent_ext(P, keys, lvl - 3, in, steps, outp, W + w.ext, W + w.coef, st, false));
    }
    std::vector<u64 *> outs(n_o);
    for (int t = 0; t < n_o; t++) {
        const int o = o0 + t;
        if (!out[t].data) return BLB_E_INVALID_ARG;
        outs[t] = out[t].data;
        SumList sl{};
        for (int a = pl->out_acc_start[o]; a < pl->out_acc_start[o + 1]; a++) {
            if (sl.n >= 64) return BLB_E_LAYOUT;
            sl.src[sl.n++] = W + w.arot + (size_t)a * 2 * E3 * N;
        }
        k_sum_list<<<gx(N, E3, 2), kTB, 0, st>>>(sl, W + w.oext + (size_t)t * 2 * E3 * N, P->pr, E3, N, k3, P->K);
        BLB_COUNT_LAUNCH(1);
        out[t].level = lvl - 3;
        // scale bookkeeping in the same floating-point order as the oracle: the masks
        // (scale q_l, q_{l-2}) cancel in their rescales, the product rescale divides by q_{l-1}
        const double ql = (double)P->mod[lvl], ql1 = (double)P->mod[lvl - 1], ql2 = (double)P->mod[lvl - 2];
        int first_u = 0;
        for (auto &A : pl->accs)
            if (A.out == o) { first_u = A.u; break; }
        const double sq = first_u == 0 ? sQ : (sQ * ql) / ql;
        const double sk = (sK * ql) / ql;
        out[t].scale = (((sq * sk) / ql1) * ql2) / ql2;
    }
    if (n_o > 0) BLB_TRY(launch_moddown(P, lvl - 3, W + w.oext, n_o, outs.data(), conv, st));
    BLB_CHECK_LAUNCH();
    return BLB_OK;
}

extern "C" blb_status blb_ct_ct_qk(const blb_qk_plan *pl, const blb_keys *keys, const blb_ct *Q, const blb_ct *K, int J,
                                   const uint64_t *masks, blb_ct *out, void *ws, size_t ws_bytes, void *stream) {
    if (!pl || !keys || !Q || !K || !masks || !out || !ws) return BLB_E_INVALID_ARG;
    if (pl->iw0 != 0 || pl->iw1 != pl->B) {
        blb_set_error("blb_ct_ct_qk: a windowed plan needs blb_ct_ct_qk_acc + blb_ct_ct_qk_finish");
        return BLB_E_INVALID_ARG;
    }
    BLB_TRY(qk_check(pl, keys, Q, K, J));
    const QKWs w = qk_ws(pl);
    if (ws_bytes < w.total * sizeof(u64)) {
        blb_set_error("workspace too small: %zu < %zu", ws_bytes, w.total * sizeof(u64));
        return BLB_E_NOMEM;
    }
    cudaStream_t st = (cudaStream_t)stream;
    u64 *W = (u64 *)ws;
    BLB_TRY(qk_acc(pl, keys, Q, K, masks, W + w.aacc, W, w, st));
    return qk_finish(pl, keys, W + w.aacc, false, 0, pl->L / pl->g, Q[0].scale, K[0].scale, out, W, w, st);
}

extern "C" size_t blb_qk_acc_bytes(const blb_qk_plan *pl) {
    if (!pl) return 0;
    return pl->accs.size() * 2 * (size_t)(pl->level - 1 + pl->P->np) * pl->P->N * sizeof(u64);
}

extern "C" blb_status blb_qk_acc_range(const blb_qk_plan *pl, int out_first, int out_count, int *slot_first,
                                       int *slot_count) {
    if (!pl || !slot_first || !slot_count) return BLB_E_INVALID_ARG;
    const int n_out = pl->L / pl->g;
    if (out_first < 0 || out_count < 0 || out_first + out_count > n_out) return BLB_E_INVALID_ARG;
    *slot_first = pl->out_acc_start[out_first];
    *slot_count = pl->out_acc_start[out_first + out_count] - *slot_first;
    return BLB_OK;
}

extern "C" blb_status blb_ct_ct_qk_acc(const blb_qk_plan *pl, const blb_keys *keys, const blb_ct *Q, const blb_ct *K,
                                       int J, const uint64_t *masks, uint64_t *acc_out, void *ws, size_t ws_bytes,
                                       void *stream) {
    if (!pl || !keys || !Q || !K || !masks || !acc_out || !ws) return BLB_E_INVALID_ARG;
    BLB_TRY(qk_check(pl, keys, Q, K, J));
    const QKWs w = qk_ws(pl);
    if (ws_bytes < w.total * sizeof(u64)) {
        blb_set_error("workspace too small: %zu < %zu", ws_bytes, w.total * sizeof(u64));
        return BLB_E_NOMEM;
    }
    return qk_acc(pl, keys, Q, K, masks, acc_out, (u64 *)ws, w, (cudaStream_t)stream);
}

extern "C" blb_status blb_ct_ct_qk_finish(const blb_qk_plan *pl, const blb_keys *keys, const uint64_t *acc_in,
                                          int out_first, int out_count, double scale_q, double scale_k, blb_ct *out,
                                          void *ws, size_t ws_bytes, void *stream) {
    const int n_out = pl ? pl->L / pl->g : 0;
    if (!pl || !keys || !ws || (out_count > 0 && (!acc_in || !out))) return BLB_E_INVALID_ARG;
    if (out_first < 0 || out_count < 0 || out_first + out_count > n_out) {
        blb_set_error("blb_ct_ct_qk_finish: outputs [%d, %d) outside [0, %d)", out_first, out_first + out_count, n_out);
        return BLB_E_INVALID_ARG;
    }
    BLB_TRY(qk_check(pl, keys, nullptr, nullptr, 0));
    const QKWs w = qk_ws(pl);
    if (ws_bytes < w.total * sizeof(u64)) {
        blb_set_error("workspace too small: %zu < %zu", ws_bytes, w.total * sizeof(u64));
        return BLB_E_NOMEM;
    }
    if (out_count == 0) return BLB_OK;
    return qk_finish(pl, keys, acc_in, true, out_first, out_count, scale_q, scale_k, out, (u64 *)ws, w,
                     (cudaStream_t)stream);
}
