// Random 16-byte row reads from an L2-resident table: LSU loads (one
// uncoalesced sector per row) against TMA tile::gather4 (four rows per
// instruction, issued by one thread per warp into shared memory).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lcuda gather4_bench.cu -o gather4_bench
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <vector>

__global__ void lsu_kernel(const uint4* __restrict__ tab, const int32_t* __restrict__ idx, int64_t n, uint4* out) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint4 v = __ldcg(tab + __ldcs(idx + i));
        acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ void mbar_init(uint64_t* b, int c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)),
                 "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(
            (uint32_t)__cvta_generic_to_shared(b)),
        "r"(phase));
}

// each warp: a ring of D slots of 4 rows; lane 0 issues gather4 for slot s, waits D slots later
template <int D>
__global__ void __launch_bounds__(256) tma_kernel(const __grid_constant__ CUtensorMap tm, const int32_t* __restrict__ idx,
                                                  int64_t n, uint4* out) {
    __shared__ __align__(128) uint4 ring[8][D][8];   // 128-B slots (tensor TMA destinations)
    __shared__ uint64_t bar[8][D];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0)
        for (int s = 0; s < D; s++) mbar_init(&bar[w][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int64_t groups = n / 4;
    const int64_t gw = (int64_t)gridDim.x * 8;
    uint4 acc = make_uint4(0, 0, 0, 0);
    uint32_t phase[D];
    for (int s = 0; s < D; s++) phase[s] = 0;
    int64_t g = (int64_t)blockIdx.x * 8 + w;
    // prologue
    if (lane == 0)
        for (int s = 0; s < D && g + (int64_t)s * gw < groups; s++) {
            const int64_t gg = g + (int64_t)s * gw;
            const int r0 = idx[4 * gg], r1 = idx[4 * gg + 1], r2 = idx[4 * gg + 2], r3 = idx[4 * gg + 3];
            mbar_expect(&bar[w][s], 64);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"((uint32_t)__cvta_generic_to_shared(&ring[w][s][0])),
                "l"(&tm), "r"((uint32_t)__cvta_generic_to_shared(&bar[w][s])), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
                : "memory");
        }
    for (int64_t k = 0;; k++) {
        const int s = (int)(k % D);
        const int64_t gg = g + k * gw;
        if (gg >= groups) break;
        mbar_wait(&bar[w][s], phase[s]);
        phase[s] ^= 1;
        if (lane < 4) {
            const uint4 v = ring[w][s][lane];
            acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
        }
        __syncwarp();
        const int64_t nx = gg + (int64_t)D * gw;
        if (lane == 0 && nx < groups) {
            const int r0 = idx[4 * nx], r1 = idx[4 * nx + 1], r2 = idx[4 * nx + 2], r3 = idx[4 * nx + 3];
            mbar_expect(&bar[w][s], 64);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"((uint32_t)__cvta_generic_to_shared(&ring[w][s][0])),
                "l"(&tm), "r"((uint32_t)__cvta_generic_to_shared(&bar[w][s])), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
                : "memory");
        }
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int64_t rows : {(int64_t)1 << 21, (int64_t)1 << 24}) {
        const int64_t n = (int64_t)1 << 25;   // random reads per launch
        uint4* tab;
        int32_t* idx;
        uint4* out;
        cudaMalloc(&tab, rows * 16);
        cudaMalloc(&idx, n * 4);
        cudaMalloc(&out, 64);
        cudaMemset(tab, 1, rows * 16);
        std::vector<int32_t> h(n);
        uint64_t x = 88172645463325252ull;
        for (int64_t i = 0; i < n; i++) {
            x ^= x << 13; x ^= x >> 7; x ^= x << 17;
            h[i] = (int32_t)(x % rows);
        }
        cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
        EncodeFn enc = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
        CUtensorMap tm;
        cuuint64_t dims[2] = {4, (cuuint64_t)rows};
        cuuint64_t strides[1] = {16};
        cuuint32_t box[2] = {4, 1};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, tab, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float ms;
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(a);
            lsu_kernel<<<sms * 8, 256>>>(tab, idx, n, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("rows %lld: LSU   %.3f ms = %.2f rows/clk/SM\n", (long long)rows, ms, n / (ms * 1e-3) / sms / 1.965e9);
        }
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(a);
            tma_kernel<8><<<sms * 4, 256>>>(tm, idx, n, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            cudaError_t e = cudaGetLastError();
            if (rep) printf("rows %lld: TMA g4 %.3f ms = %.2f rows/clk/SM (%s)\n", (long long)rows, ms, n / (ms * 1e-3) / sms / 1.965e9,
                            cudaGetErrorString(e));
        }
        cudaFree(tab); cudaFree(idx); cudaFree(out);
    }
    return 0;
}
