// Random 4-byte reads from a 2 MB table: LSU loads through L1/L2 against the
// table spread over a 16-CTA cluster's shared memory (128 KB per CTA) read
// through DSMEM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 dsmem_bench.cu -o dsmem_bench
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <vector>
namespace cg = cooperative_groups;

constexpr int kWords = 1 << 19;          // 2 MB table
constexpr int kCl = 16;                   // CTAs per cluster
constexpr int kSlice = kWords / kCl;      // 32K words = 128 KB per CTA

__global__ void lsu_kernel(const uint32_t* __restrict__ tab, const int32_t* __restrict__ idx, int64_t n, uint32_t* out) {
    uint32_t acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) acc ^= __ldcg(tab + __ldcs(idx + i));
    if (acc == 0x12345678u) out[0] = acc;
}

__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(1024) dsmem_kernel(const uint32_t* __restrict__ tab,
                                                                                   const int32_t* __restrict__ idx,
                                                                                   int64_t n, uint32_t* out) {
    extern __shared__ uint32_t slice[];
    cg::cluster_group cl = cg::this_cluster();
    const int r = (int)cl.block_rank();
    for (int w = threadIdx.x; w < kSlice; w += blockDim.x) slice[w] = tab[r * kSlice + w];
    cl.sync();
    uint32_t acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int32_t j = __ldcs(idx + i);
        const uint32_t* p = cl.map_shared_rank(slice, j / kSlice);
        acc ^= p[j % kSlice];
    }
    cl.sync();   // no CTA leaves while others still read its slice
    if (acc == 0x12345678u) out[0] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t n = (int64_t)1 << 25;
    uint32_t *tab, *out;
    int32_t* idx;
    cudaMalloc(&tab, (size_t)kWords * 4);
    cudaMalloc(&idx, n * 4);
    cudaMalloc(&out, 64);
    cudaMemset(tab, 1, (size_t)kWords * 4);
    std::vector<int32_t> h(n);
    uint64_t x = 88172645463325252ull;
    for (int64_t i = 0; i < n; i++) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = (int32_t)(x % kWords); }
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(dsmem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSlice * 4);
    cudaFuncSetAttribute(dsmem_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float ms;
    for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(a);
        lsu_kernel<<<sms * 8, 256>>>(tab, idx, n, out);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        if (rep) printf("LSU   %.3f ms = %.2f reads/clk/SM\n", ms, n / (ms * 1e-3) / sms / 1.965e9);
    }
    int ncl = sms / kCl;   // whole clusters that fit
    for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(a);
        dsmem_kernel<<<ncl * kCl, 1024, kSlice * 4>>>(tab, idx, n, out);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        cudaError_t e = cudaGetLastError();
        if (rep) printf("DSMEM %.3f ms = %.2f reads/clk/SM (%d CTAs in clusters of %d; per SM used: %.2f) %s\n", ms,
                        n / (ms * 1e-3) / sms / 1.965e9, ncl * kCl, kCl, n / (ms * 1e-3) / (ncl * kCl) / 1.965e9,
                        cudaGetErrorString(e));
    }
    return 0;
}
