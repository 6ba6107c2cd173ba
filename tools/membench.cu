// membench.cu -- HBM streaming microbenchmark for the MAC access pattern (standalone tool).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench tools/membench.cu
// Modes: 0 = plain 16-byte streaming read of P bytes;
//        1 = MAC pattern, plaintext loads only (blocked layout, 4 KB per CTA-entry);
//        2 = MAC pattern, R loads only (L2-resident working set);
//        3 = MAC pattern, both (no arithmetic beyond an xor);
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;

__global__ void k_stream(const ulonglong2 *p, size_t n, u64 *out) {
    u64 acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        ulonglong2 v = p[i];
        acc ^= v.x ^ v.y;
    }
    if (acc == 0x1234567) out[0] = acc;
}

// grid: n_o * n_tiles * k CTAs of 256 threads; n_e entries per output
__global__ void k_pattern(const u64 *pt, const u64 *R, int n_o, int n_e, int k, int N, int mode, u64 *out) {
    const int n_tiles = N / 512;
    int bid = blockIdx.x;
    const int o = bid % n_o; bid /= n_o;
    const int tile = bid % n_tiles;
    const int l = bid / n_tiles;
    const long long kN = (long long)k * N;
    const long long lx = (long long)l * N + tile * 512 + 2 * threadIdx.x;
    const u64 *pp = pt + (long long)o * n_e * kN + (long long)l * n_e * N + (long long)tile * n_e * 512 + 2 * threadIdx.x;
    u64 acc = 0;
    for (int e = 0; e < n_e; e += 4) {
        ulonglong2 pv[4], r0[4], r1[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int bi = (e + u) % 96;
            if (mode != 2) pv[u] = *reinterpret_cast<const ulonglong2 *>(pp + (long long)(e + u) * 512);
            else pv[u] = make_ulonglong2(0, 0);
            if (mode >= 2) {
                r0[u] = *reinterpret_cast<const ulonglong2 *>(R + (long long)bi * 2 * kN + lx);
                r1[u] = *reinterpret_cast<const ulonglong2 *>(R + ((long long)bi * 2 + 1) * kN + lx);
            } else {
                r0[u] = make_ulonglong2(0, 0);
                r1[u] = r0[u];
            }
        }
#pragma unroll
        for (int u = 0; u < 4; u++) acc ^= pv[u].x ^ pv[u].y ^ r0[u].x ^ r0[u].y ^ r1[u].x ^ r1[u].y;
    }
    if (acc == 0x1234567) out[0] = acc;
}

int main() {
    const int N = 1 << 16, k = 5, n_e = 96, n_o = 88;
    const size_t pt_words = (size_t)n_o * n_e * k * N;  // 22 GB
    const size_t r_words = (size_t)96 * 2 * k * N;
    u64 *pt, *R, *out;
    cudaMalloc(&pt, pt_words * 8);
    cudaMalloc(&R, r_words * 8);
    cudaMalloc(&out, 8);
    cudaMemset(pt, 1, pt_words * 8);
    cudaMemset(R, 2, r_words * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(a);
        k_stream<<<148 * 8, 256>>>((const ulonglong2 *)pt, pt_words / 2, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("stream-read: %.3f ms  %.1f GB/s\n", ms, pt_words * 8 / (ms * 1e-3) / 1e9);
    }
    for (int mode = 1; mode <= 3; mode++) {
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(a);
            k_pattern<<<n_o * (N / 512) * k, 256>>>(pt, R, n_o, n_e, k, N, mode, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("pattern mode %d: %.3f ms  pt-equivalent %.1f GB/s\n", mode, ms, pt_words * 8 / (ms * 1e-3) / 1e9);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
