// Microbenchmark (not product code): what bounds a random 16-B row gather on
// B200?  (1) source-size sweep at a fixed access count: is a random gather
// from an L2-resident source faster?  (2) windowed gathers over a 4 GiB
// table: output swept in order, sources random inside a sliding window.
// (3) one smem-staged radix partition pass (coalesced runs out) at several
// fan-outs: the building block of a multi-pass permutation.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o exp_l2_gather exp_l2_gather.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

__global__ void make_idx(int32_t* idx, int64_t n, int64_t src_rows, int64_t win, uint32_t salt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t h = hash32((uint32_t)i * 2654435761u ^ salt);
        if (win > 0) {
            int64_t base = (i * src_rows / n) / win * win;
            idx[i] = (int32_t)(base + h % win);
        } else idx[i] = (int32_t)(h % src_rows);
    }
}

__global__ void gather4(const int32_t* __restrict__ idx, const uint4* __restrict__ src, int64_t n, uint4* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        __stcs(out + i, __ldcg(src + __ldcs(idx + i)));
}

// Partition pass: tile of T rows -> F buckets; bucket of row = hash; the
// CTA counts, scans, scatters into smem in bucket order, then writes each
// bucket run to out[bucket_base + cursor] (cursors: global atomics per
// bucket, so run placement is approximate -- bandwidth study only).
template <int T, int F>
__global__ void __launch_bounds__(512) partition_pass(const uint4* __restrict__ src, int64_t n, uint4* __restrict__ out,
                                                      int64_t bucket_cap, unsigned long long* cursors) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint4* tile = (uint4*)smem;
    int* cnt = (int*)(tile + T);
    int* off = cnt + F;
    int* gbase = off + F;
    uint16_t* bk = (uint16_t*)(gbase + F);
    for (int64_t t0 = (int64_t)blockIdx.x * T; t0 < n; t0 += (int64_t)gridDim.x * T) {
        for (int b = threadIdx.x; b < F; b += blockDim.x) cnt[b] = 0;
        __syncthreads();
        int rank[T / 512];
        uint4 v[T / 512];
#pragma unroll
        for (int k = 0; k < T / 512; k++) {
            int e = k * 512 + threadIdx.x;
            v[k] = __ldcs(src + t0 + e);
            int b = hash32((uint32_t)(t0 + e)) % F;
            bk[e] = (uint16_t)b;
            rank[k] = atomicAdd(&cnt[b], 1);
        }
        __syncthreads();
        if (threadIdx.x == 0) {  // tiny serial scan (F <= 2048)
            int s = 0;
            for (int b = 0; b < F; b++) { off[b] = s; s += cnt[b]; }
        }
        __syncthreads();
        for (int b = threadIdx.x; b < F; b += blockDim.x)
            gbase[b] = (int)(atomicAdd(&cursors[b], (unsigned long long)cnt[b]) % bucket_cap) + 0;
#pragma unroll
        for (int k = 0; k < T / 512; k++) {
            int e = k * 512 + threadIdx.x;
            tile[off[bk[e]] + rank[k]] = v[k];
        }
        __syncthreads();
        // write runs: slot s belongs to bucket b (binary search over off)
        for (int s = threadIdx.x; s < T; s += blockDim.x) {
            int lo = 0, hi = F - 1;
            while (lo < hi) { int mid = (lo + hi + 1) >> 1; if (off[mid] <= s) lo = mid; else hi = mid - 1; }
            int64_t dst = (int64_t)lo * bucket_cap + (gbase[lo] + (s - off[lo])) % bucket_cap;
            __stcs(out + dst, tile[s]);
        }
        __syncthreads();
    }
}

// Local permutation: bucket of B rows in smem, out[b*B + i] = tile[q[i]]
template <int B>
__global__ void __launch_bounds__(512) local_perm(const uint4* __restrict__ src, int64_t n, uint4* __restrict__ out) {
    extern __shared__ __align__(16) uint4 tl[];
    for (int64_t t0 = (int64_t)blockIdx.x * B; t0 < n; t0 += (int64_t)gridDim.x * B) {
        for (int e = threadIdx.x; e < B; e += blockDim.x) tl[e] = __ldcs(src + t0 + e);
        __syncthreads();
        for (int e = threadIdx.x; e < B; e += blockDim.x) __stcs(out + t0 + e, tl[hash32(e + (uint32_t)t0) % B]);
        __syncthreads();
    }
}

__global__ void copy4(const uint4* __restrict__ s, int64_t n, uint4* __restrict__ d) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        __stcs(d + i, __ldcs(s + i));
}

template <class F>
float timeit(F f, int reps = 5) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    f(); f();
    std::vector<float> ts;
    for (int r = 0; r < reps; r++) {
        cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    return ts[reps / 2];
}

int main() {
    const int64_t BIG = 1ll << 28;  // rows (4 GiB table)
    uint4 *src, *out; int32_t* idx; unsigned long long* cur;
    CK(cudaMalloc(&src, BIG * 16)); CK(cudaMalloc(&out, BIG * 16)); CK(cudaMalloc(&idx, BIG * 4));
    CK(cudaMalloc(&cur, 4096 * 8));
    CK(cudaMemset(src, 1, BIG * 16));
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int G = sms * 8;
    float tc = timeit([&] { copy4<<<G, 256>>>(src, BIG, out); });
    printf("copy 2^28 x 16B: %.3f ms  %.0f GB/s (r+w)\n", tc, 2.0 * BIG * 16 / tc / 1e6);
    const int64_t N = 1ll << 26;  // accesses for the source-size sweep
    printf("\n[1] random 16-B gather, %lld accesses, source size sweep\n", (long long)N);
    for (int lg = 16; lg <= 28; lg += 2) {
        int64_t srows = 1ll << lg;
        make_idx<<<G, 256>>>(idx, N, srows, 0, 77);
        float t = timeit([&] { gather4<<<G, 256>>>(idx, src, N, out); });
        printf("  src %8.1f MB: %.3f ms  %.1f G rows/s\n", srows * 16 / 1e6, t, N / t / 1e6);
    }
    printf("\n[2] windowed gather over 2^28 rows (out in order; src random within window)\n");
    for (int64_t wmb : {1, 4, 16, 32, 64, 0}) {
        int64_t win = wmb * (1 << 20) / 16;
        make_idx<<<G, 256>>>(idx, BIG, BIG, wmb ? win : 0, 99);
        float t = timeit([&] { gather4<<<G, 256>>>(idx, src, BIG, out); });
        printf("  window %3lld MB: %.3f ms  %.1f G rows/s\n", (long long)wmb, t, BIG / t / 1e6);
    }
    printf("\n[3] smem partition pass over 2^28 rows (tile T rows -> F buckets, coalesced runs)\n");
    auto run_part = [&](auto kern, int T, int F) {
        size_t sm = (size_t)T * 16 + 3 * F * 4 + T * 2;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        int occ; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 512, sm);
        float t = timeit([&] {
            cudaMemsetAsync(cur, 0, 4096 * 8);
            kern<<<sms * occ, 512, sm>>>(src, BIG, out, BIG / F + BIG / F / 8, cur);
        });
        CK(cudaGetLastError());
        printf("  T=%5d F=%5d occ=%d: %.3f ms  %.0f GB/s (r+w)\n", T, F, occ, t, 2.0 * BIG * 16 / t / 1e6);
    };
    run_part(partition_pass<4096, 64>, 4096, 64);
    run_part(partition_pass<4096, 256>, 4096, 256);
    run_part(partition_pass<8192, 256>, 8192, 256);
    run_part(partition_pass<8192, 1024>, 8192, 1024);
    run_part(partition_pass<8192, 2048>, 8192, 2048);
    printf("\n[4] smem local permutation pass over 2^28 rows\n");
    auto run_lp = [&](auto kern, int B) {
        size_t sm = (size_t)B * 16;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        int occ; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 512, sm);
        float t = timeit([&] { kern<<<sms * occ, 512, sm>>>(src, BIG, out); });
        CK(cudaGetLastError());
        printf("  B=%5d occ=%d: %.3f ms  %.0f GB/s (r+w)\n", B, occ, t, 2.0 * BIG * 16 / t / 1e6);
    };
    run_lp(local_perm<4096>, 4096);
    run_lp(local_perm<8192>, 8192);
    run_lp(local_perm<12288>, 12288);
    return 0;
}
