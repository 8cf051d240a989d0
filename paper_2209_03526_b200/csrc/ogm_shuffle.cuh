// ogm_shuffle.cuh -- seeded permutation (src/prf.py:95-105) and the 3-party
// secret-shared shuffle (src/shuffle.py:80-144) for sm_100a.
#pragma once

#include "ogm_aes.cuh"
#include "ogm_common.cuh"
#include "ogm_host.cuh"

namespace ogm {

// ---------------------------------------------------------------------------
// Bit-exact Fisher-Yates on the device.
//
// The reference runs   for i = n-1 .. 1:  j = draw[n-1-i] mod (i+1);
// swap(perm[i], perm[j])   (src/prf.py:100-104), with draws the u64 LE words
// of prf_stream(key, "SHPI", table_id, 8(n-1)).  Iteration i touches only the
// locations i and H[i] <= i, and must run after every earlier (larger) i'
// that touches one of them.  Deterministic reservations (Shun, Gu, Blelloch,
// Fineman, Gibbons, SODA'15) execute it in parallel rounds:
//   reserve: every live i does atomicMax(R[i], i), atomicMax(R[H[i]], i)
//   commit:  i swaps iff it holds both reservations, else it stays live
//   reset:   R[i] = R[H[i]] = -1 for every live i of the round
// Two committers of one round touch disjoint locations and every committer
// has all its predecessors done, so the result equals the sequential loop.
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(kAesThreads) perm_draws_kernel(
    AesKeySched key, uint32_t label_be, uint64_t index, int64_t n, int32_t* __restrict__ H,
    int32_t* __restrict__ live, int32_t* __restrict__ perm, int32_t* __restrict__ R) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    aes_fill_tables(smem_raw);
    __syncthreads();
    const AesTab T(smem_raw);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t x = tid; x < n; x += stride) {
        perm[x] = (int32_t)x;
        R[x] = -1;
    }
    const int64_t ndraw = n - 1;
    const int64_t nblk = (ndraw + 1) >> 1;  // two u64 draws per AES block
    for (int64_t b = tid; b < nblk; b += stride) {
        const uint4 ks = aes128_enc(T, ctr_block(label_be, index, (uint64_t)b), ParamKey{key.rk});
        const uint64_t d[2] = {((uint64_t)ks.y << 32) | ks.x, ((uint64_t)ks.w << 32) | ks.z};
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int64_t q = 2 * b + h;
            if (q >= ndraw) break;
            const int64_t i = n - 1 - q;
            H[i] = (int32_t)(d[h] % (uint64_t)(i + 1));
            live[q] = (int32_t)i;
        }
    }
}

__global__ void perm_reserve_kernel(const int32_t* __restrict__ live, const int32_t* __restrict__ cnt,
                                    const int32_t* __restrict__ H, int32_t* __restrict__ R) {
    const int32_t c = *cnt;
    for (int32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < c; t += gridDim.x * blockDim.x) {
        const int32_t i = live[t];
        atomicMax(&R[i], i);
        atomicMax(&R[H[i]], i);
    }
}

__global__ void perm_commit_kernel(const int32_t* __restrict__ live, const int32_t* __restrict__ cnt,
                                   const int32_t* __restrict__ H, const int32_t* __restrict__ R,
                                   int32_t* __restrict__ perm, int32_t* __restrict__ next,
                                   int32_t* __restrict__ next_cnt) {
    const int32_t c = *cnt;
    for (int32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < c; t += gridDim.x * blockDim.x) {
        const int32_t i = live[t];
        const int32_t h = H[i];
        if (R[i] == i && R[h] == i) {
            const int32_t a = perm[i];
            perm[i] = perm[h];
            perm[h] = a;
        } else {
            next[atomicAdd(next_cnt, 1)] = i;
        }
    }
}

__global__ void perm_reset_kernel(const int32_t* __restrict__ live, const int32_t* __restrict__ cnt,
                                  const int32_t* __restrict__ H, int32_t* __restrict__ R) {
    const int32_t c = *cnt;
    for (int32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < c; t += gridDim.x * blockDim.x) {
        const int32_t i = live[t];
        R[i] = -1;
        R[H[i]] = -1;
    }
}

int shuffle_init() {
    OGM_CUDA_TRY(allow_big_smem(perm_draws_kernel, kAesTableBytes));
    return OGM_OK;
}

static int64_t perm_ws_bytes(int64_t n) { return 4 * n * 4 + 256; }

static int seeded_permutation_impl(const uint8_t* key, const uint8_t* label, uint64_t index, int64_t n,
                                   int32_t* perm, void* workspace, cudaStream_t st) {
    if (n == 0) return OGM_OK;
    uint8_t* ws = (uint8_t*)workspace;
    int32_t* cnts = (int32_t*)ws;  // [0], [1]: live counts of the two lists; [2]: host-read scratch
    int32_t* H = (int32_t*)(ws + 256);
    int32_t* R = H + n;
    int32_t* live[2] = {R + n, R + 2 * n};
    AesKeySched ks = make_sched(key);
    const int32_t init_cnt = (int32_t)(n - 1);
    OGM_CUDA_TRY(cudaMemcpyAsync(&cnts[0], &init_cnt, 4, cudaMemcpyHostToDevice, st));
    OGM_CUDA_TRY(cudaMemsetAsync(&cnts[1], 0, 4, st));
    perm_draws_kernel<<<aes_grid(n), kAesThreads, kAesTableBytes, st>>>(ks, label_be(label), index, n, H,
                                                                        live[0], perm, R);
    OGM_LAUNCH_CHECK();
    if (n < 2) return OGM_OK;
    const int grid = sm_count() * 8, threads = 256;
    int cur = 0;
    int32_t remaining = init_cnt;
    int rounds = 0;
    while (remaining > 0) {
        // a few rounds per host round-trip; empty rounds are cheap no-ops
        for (int r = 0; r < 4; r++, rounds++) {
            perm_reserve_kernel<<<grid, threads, 0, st>>>(live[cur], &cnts[cur], H, R);
            perm_commit_kernel<<<grid, threads, 0, st>>>(live[cur], &cnts[cur], H, R, perm, live[cur ^ 1],
                                                         &cnts[cur ^ 1]);
            perm_reset_kernel<<<grid, threads, 0, st>>>(live[cur], &cnts[cur], H, R);
            OGM_LAUNCH_CHECK();
            OGM_CUDA_TRY(cudaMemsetAsync(&cnts[cur], 0, 4, st));
            cur ^= 1;
        }
        OGM_CUDA_TRY(cudaMemcpyAsync(&remaining, &cnts[cur], 4, cudaMemcpyDeviceToHost, st));
        OGM_CUDA_TRY(cudaStreamSynchronize(st));
        if (rounds > 100000) {
            set_error("permutation did not converge");
            return OGM_ERR_CUDA;
        }
    }
    return OGM_OK;
}

}  // namespace ogm

extern "C" {

int64_t ogm_perm_workspace_bytes(int64_t n) { return ogm::perm_ws_bytes(n < 0 ? 0 : n); }

int ogm_seeded_permutation(const uint8_t* key, const uint8_t* label, uint64_t index, int64_t n,
                           int32_t* perm, void* workspace, void* stream) {
    OGM_CHECK_ARG(key && label, OGM_ERR_ARG, "permutation key and label are required");
    OGM_CHECK_ARG(n >= 0 && n < ((int64_t)1 << 31), OGM_ERR_ARG, "permutation size %lld out of range",
                  (long long)n);
    OGM_CHECK_ARG(n == 0 || workspace, OGM_ERR_ARG, "permutation workspace is required");
    OGM_ENSURE_INIT();
    return ogm::seeded_permutation_impl(key, label, index, n, perm, workspace, ogm::as_stream(stream));
}

}  // extern "C"
