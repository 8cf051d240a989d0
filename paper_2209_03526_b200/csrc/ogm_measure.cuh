// ogm_measure.cuh -- roofline denominators measured on the running device.
//
// The FSS walk is bound by the ALU pipe (PRMT/LOP3 address and XOR work for
// the table lookups), so its roofline denominator is the LOP3 issue rate of
// the whole GPU, measured here rather than taken from a datasheet.
#pragma once

#include "ogm_common.cuh"
#include "ogm_host.cuh"

namespace ogm {

constexpr int kPeakChains = 8;
constexpr int kPeakUnroll = 16;

__device__ __forceinline__ uint32_t lop3_xor3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// Each thread runs kPeakChains independent LOP3 chains; one lop3 = 1 int op.
__global__ void int_peak_kernel(uint32_t* out, int iters, uint32_t seed) {
    uint32_t a[kPeakChains];
#pragma unroll
    for (int c = 0; c < kPeakChains; c++) a[c] = seed * (threadIdx.x + 1) + c * 0x9e3779b9u;
    const uint32_t k1 = seed ^ 0x5bd1e995u, k2 = seed + blockIdx.x;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int u = 0; u < kPeakUnroll; u++) {
#pragma unroll
            for (int c = 0; c < kPeakChains; c++) a[c] = lop3_xor3(a[c], k1, k2 + u);
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int c = 0; c < kPeakChains; c++) r ^= a[c];
    if (r == 0x12345678u) out[blockIdx.x] = r;  // keep the chains live
}

}  // namespace ogm

extern "C" int ogm_measure_int_peak(double* ops_per_sec, double* seconds) {
    OGM_ENSURE_INIT();
    const int blocks = ogm::sm_count() * 4, threads = 512, iters = 4096;
    uint32_t* out = nullptr;
    cudaEvent_t e0, e1;
    OGM_CUDA_TRY(cudaMalloc(&out, blocks * 4));
    OGM_CUDA_TRY(cudaEventCreate(&e0));
    OGM_CUDA_TRY(cudaEventCreate(&e1));
    ogm::int_peak_kernel<<<blocks, threads>>>(out, iters / 8, 1u);  // warm-up
    OGM_CUDA_TRY(cudaEventRecord(e0));
    ogm::int_peak_kernel<<<blocks, threads>>>(out, iters, 3u);
    OGM_CUDA_TRY(cudaEventRecord(e1));
    OGM_CUDA_TRY(cudaEventSynchronize(e1));
    float ms = 0;
    OGM_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    const double ops = (double)blocks * threads * iters * ogm::kPeakUnroll * ogm::kPeakChains;
    *seconds = ms * 1e-3;
    *ops_per_sec = ops / (*seconds);
    return OGM_OK;
}
