// peaks.cu -- measured arithmetic-pipe peaks of the device the library runs on (SURVEY 8(d)
// "integer-pipe fraction against an IMAD/ALU microbenchmark peak measured on the box").
//
// The hot path is exact modular integer arithmetic: the 60-bit NTT / MAC rows are bound by the
// fma-heavy pipe (IMAD, IMAD.WIDE, IMAD.HI), the 40-bit rows by the FP64 pipe (DFMA / DADD /
// DMUL).  MEASURED_PEAKS.json has HBM and bf16 figures only, so the bench measures these two
// denominators itself: every thread runs kChains independent dependency chains of one
// instruction kind (enough to cover the pipe latency), grids of 8 CTAs per SM, CUDA events.
#include <algorithm>
#include "blb_internal.cuh"

namespace {
constexpr int kChains = 8;
constexpr int kIters = 4096;

// 32-bit IMAD (mad.lo.u32): the fma-heavy pipe's integer multiply-add
__global__ void __launch_bounds__(256) k_peak_imad(uint32_t *out, uint32_t seed) {
    uint32_t a[kChains];
#pragma unroll
    for (int c = 0; c < kChains; c++) a[c] = seed + threadIdx.x * 7u + c;
    const uint32_t m = seed | 1u, b = seed * 3u + 1u;
    for (int i = 0; i < kIters; i++) {
#pragma unroll
        for (int c = 0; c < kChains; c++) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[c]) : "r"(m), "r"(b));
    }
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < kChains; c++) s ^= a[c];
    if (s == 0x12345678u) out[threadIdx.x] = s;  // keep the chains live
}

// FP64 fused multiply-add
__global__ void __launch_bounds__(256) k_peak_dfma(double *out, double seed) {
    double a[kChains];
#pragma unroll
    for (int c = 0; c < kChains; c++) a[c] = seed + threadIdx.x * 1e-9 + c;
    const double m = 0.999999, b = 1e-7;
    for (int i = 0; i < kIters; i++) {
#pragma unroll
        for (int c = 0; c < kChains; c++) a[c] = __fma_rn(a[c], m, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < kChains; c++) s += a[c];
    if (s == 12345.0) out[threadIdx.x] = s;
}
}  // namespace

// ops/s of each pipe (one IMAD or one DFMA = one op), best of `reps` timed launches on `stream`
extern "C" blb_status blb_measure_pipe_peaks(int device, double *imad_per_s, double *dfma_per_s, void *stream) {
    if (!imad_per_s || !dfma_per_s) return BLB_E_INVALID_ARG;
    BLB_CUDA_TRY(cudaSetDevice(device));
    int sms = 0;
    BLB_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    cudaStream_t st = (cudaStream_t)stream;
    void *buf = nullptr;
    BLB_CUDA_TRY(cudaMalloc(&buf, 256 * sizeof(double)));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = sms * 8;
    const double ops = (double)grid * 256 * kChains * kIters;
    double best_i = 0, best_d = 0;
    for (int r = 0; r < 4; r++) {
        float ms = 0;
        cudaEventRecord(e0, st);
        k_peak_imad<<<grid, 256, 0, st>>>((uint32_t *)buf, 12345u + r);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0) best_i = std::max(best_i, ops / (ms * 1e-3));
        cudaEventRecord(e0, st);
        k_peak_dfma<<<grid, 256, 0, st>>>((double *)buf, 1.0 + r);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0) best_d = std::max(best_d, ops / (ms * 1e-3));
    }
    BLB_COUNT_LAUNCH(8);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(buf);
    BLB_CHECK_LAUNCH();
    *imad_per_s = best_i;
    *dfma_per_s = best_d;
    return BLB_OK;
}
