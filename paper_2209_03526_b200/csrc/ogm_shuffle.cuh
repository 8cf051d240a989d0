// ogm_shuffle.cuh -- seeded permutation (src/prf.py:95-105) and the 3-party
// secret-shared shuffle (src/shuffle.py:80-144) for sm_100a.
#pragma once

#include <cub/cub.cuh>

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


// ---------------------------------------------------------------------------
// One step of the 3-party shuffle (src/shuffle.py:106-143), as a gather:
//
//   k2 = P2 ? P2[i] : i          k1 = P1 ? P1[k2] : k2
//   out[i] = M1[k1] ^ M2[k1] ^ T1[k1] ^ T2[k2] ^ M3[i] ^ R[i]
//
// with every term optional.  T1/T2/R are blinding tables: either
// precomputed matrices (offline phase) or generated on the fly from
// AES-CTR (label, table id), row r = stream words [r*W, r*W + W) with the
// row tail masked to `width` (src/shuffle.py:69-73).  `_apply(p, M) = M[p]`
// (src/shuffle.py:76-77), so nested applications compose as index lookups:
//   P1: x1 = pi31(pi12(a^b^T12) ^ T31):  P2=pi31, P1=pi12, M1=a, M2=b, T1=T12, T2=T31
//   P2: y1 = pi12(b^T12):                 P1=pi12, M1=b, T1=T12
//   P2: c1 = pi23(x1^T23) ^ R2:           P1=pi23, M1=x1, T1=T23, R=R2
//   P3: R3 = c1 ^ pi23(pi31(y1^T31)^T23) ^ R1:
//                                          P2=pi23, P1=pi31, M1=y1, T1=T31, T2=T23, M3=c1, R=R1
// A thread owns a 4-word chunk of one output row.
// ---------------------------------------------------------------------------
struct GatherTerm {
    AesKeySched key;
    const uint32_t* mat;  // precomputed table (row-major, W words) or null
    uint32_t label_be;
    uint64_t index;
    int on;  // 0 absent, 1 online PRF, 2 matrix
};

struct GatherArgs {
    const int32_t* P1;
    const int32_t* P2;
    const uint32_t* M1;
    const uint32_t* M2;
    const uint32_t* M3;
    GatherTerm t1, t2, r;
    uint32_t* out;
    int64_t rows, W, width;
    int64_t row0;   // global index of local row 0 (PRF term at i uses i + row0)
    int64_t pitch;  // words per row in memory (>= W; zero padding past W)
};

__device__ __forceinline__ void prf_row_chunk(const AesTab& T, const GatherTerm& g, int64_t row, int64_t W,
                                              int64_t c, int nw, uint32_t v[4]) {
    const uint64_t g0 = (uint64_t)row * (uint64_t)W + 4 * (uint64_t)c;
    const uint64_t b0 = g0 >> 2;
    const int off = (int)(g0 & 3);
    const uint4 k0 = aes128_enc(T, ctr_block(g.label_be, g.index, b0), ParamKey{g.key.rk});
    uint32_t w8[8] = {k0.x, k0.y, k0.z, k0.w, 0, 0, 0, 0};
    if (off + nw > 4) {
        const uint4 k1 = aes128_enc(T, ctr_block(g.label_be, g.index, b0 + 1), ParamKey{g.key.rk});
        w8[4] = k1.x; w8[5] = k1.y; w8[6] = k1.z; w8[7] = k1.w;
    }
#pragma unroll
    for (int j = 0; j < 4; j++) v[j] = w8[(off + j) & 7];
}

template <bool ONLINE>
__device__ __forceinline__ void gather_chunk(const AesTab& T, const GatherArgs& a, int64_t i, int64_t c,
                                             uint32_t tail, bool vec) {
    // words [4c, 4c+nw) of row i; with a 16-B pitch the padding words ride
    // along as zeros and every access is 128-bit
    const int nw = (int)min((int64_t)4, a.W - 4 * c);  // words inside the logical row (may be <= 0)
    const int64_t k2 = a.P2 ? (int64_t)__ldg(a.P2 + i) : i;
    const int64_t k1 = a.P1 ? (int64_t)__ldg(a.P1 + k2) : k2;
    uint32_t acc[4] = {0, 0, 0, 0};
    const GatherTerm* terms[3] = {&a.t1, &a.t2, &a.r};
    const int64_t trow[3] = {k1, k2, i + a.row0};
#pragma unroll
    for (int q = 0; q < 3; q++) {
        const GatherTerm& g = *terms[q];
        if (g.on == 0 || nw <= 0) continue;
        uint32_t v[4] = {0, 0, 0, 0};
        if (ONLINE && g.on == 1) {
            prf_row_chunk(T, g, trow[q], a.W, c, nw, v);
            if (4 * c + nw == a.W) v[nw - 1] &= tail;
#pragma unroll
            for (int j = 0; j < 4; j++)
                if (j >= nw) v[j] = 0;
        } else {
            const uint32_t* src = g.mat + (q == 2 ? i : trow[q]) * a.pitch + 4 * c;
            if (vec) {
                const uint4 x = *reinterpret_cast<const uint4*>(src);
                v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
            } else {
                for (int j = 0; j < nw; j++) v[j] = src[j];
            }
        }
#pragma unroll
        for (int j = 0; j < 4; j++) acc[j] ^= v[j];
    }
    const uint32_t* m1 = a.M1 ? a.M1 + k1 * a.pitch + 4 * c : nullptr;
    const uint32_t* m2 = a.M2 ? a.M2 + k1 * a.pitch + 4 * c : nullptr;
    const uint32_t* m3 = a.M3 ? a.M3 + i * a.pitch + 4 * c : nullptr;
    uint32_t* o = a.out + i * a.pitch + 4 * c;
    if (vec) {
        uint4 x = make_uint4(acc[0], acc[1], acc[2], acc[3]);
        if (m1) x = xor4(x, *reinterpret_cast<const uint4*>(m1));
        if (m2) x = xor4(x, *reinterpret_cast<const uint4*>(m2));
        if (m3) x = xor4(x, *reinterpret_cast<const uint4*>(m3));
        *reinterpret_cast<uint4*>(o) = x;
    } else {
        for (int j = 0; j < nw; j++) {
            uint32_t x = acc[j];
            if (m1) x ^= m1[j];
            if (m2) x ^= m2[j];
            if (m3) x ^= m3[j];
            o[j] = x;
        }
    }
}

template <bool ONLINE>
__global__ void __launch_bounds__(kAesThreads) shuffle_gather_kernel(const GatherArgs a) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    if (ONLINE) {
        aes_fill_tables(smem_raw);
        __syncthreads();
    }
    const AesTab T(smem_raw);
    // 128-bit path when rows are 16-B pitched and every base is aligned
    const bool vec = (a.pitch & 3) == 0 &&
                     ((((uintptr_t)a.M1) | ((uintptr_t)a.M2) | ((uintptr_t)a.M3) | ((uintptr_t)a.out) |
                       ((uintptr_t)a.t1.mat) | ((uintptr_t)a.t2.mat) | ((uintptr_t)a.r.mat)) & 15) == 0;
    const int64_t nch = vec ? (a.pitch >> 2) : ((a.W + 3) >> 2);
    const uint32_t tail = (a.width & 31) ? ((1u << (a.width & 31)) - 1u) : 0xffffffffu;
    if (nch >= 64) {
        // wide rows: a CTA walks rows, its threads walk the row's 4-word chunks
        for (int64_t i = blockIdx.x; i < a.rows; i += gridDim.x)
            for (int64_t c = threadIdx.x; c < nch; c += blockDim.x) gather_chunk<ONLINE>(T, a, i, c, tail, vec);
    } else {
        const int64_t total = a.rows * nch;
        const int64_t stride = (int64_t)gridDim.x * blockDim.x;
        for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
            const int64_t i = t / nch;
            gather_chunk<ONLINE>(T, a, i, t - i * nch, tail, vec);
        }
    }
}

// The same step when every term is a precomputed matrix (the online phase
// after ShuffleOffline, and the wide-row material build): no AES tables, so
// a lean kernel with high occupancy for the random 16-byte row reads of
// narrow tables, and a row-per-CTA streaming loop for wide rows.
__device__ __forceinline__ uint4 ld_term(const uint32_t* m, int64_t row, int64_t pitch, int64_t c) {
    return m ? __ldcs(reinterpret_cast<const uint4*>(m + row * pitch) + c) : make_uint4(0, 0, 0, 0);
}

__global__ void __launch_bounds__(256) gather_matrix_rows_kernel(const GatherArgs a, int64_t nch) {
    const uint32_t* T1 = a.t1.on ? a.t1.mat : nullptr;
    const uint32_t* T2 = a.t2.on ? a.t2.mat : nullptr;
    const uint32_t* R = a.r.on ? a.r.mat : nullptr;
    {
        // wide rows: row indices and bases once per row, then 128-bit streams;
        // every load of two groups is issued before either store
        const int bd = blockDim.x;
        for (int64_t i = blockIdx.x; i < a.rows; i += gridDim.x) {
            const int64_t k2 = a.P2 ? (int64_t)__ldg(a.P2 + i) : i;
            const int64_t k1 = a.P1 ? (int64_t)__ldg(a.P1 + k2) : k2;
            uint4* o = reinterpret_cast<uint4*>(a.out + i * a.pitch);
            for (int64_t c0 = threadIdx.x; c0 < nch; c0 += 2 * bd) {
                const int64_t c1 = c0 + bd;
                const bool v1 = c1 < nch;
                uint4 x0 = xor4(xor4(ld_term(a.M1, k1, a.pitch, c0), ld_term(a.M2, k1, a.pitch, c0)),
                                xor4(ld_term(a.M3, i, a.pitch, c0), ld_term(T1, k1, a.pitch, c0)));
                x0 = xor4(x0, xor4(ld_term(T2, k2, a.pitch, c0), ld_term(R, i, a.pitch, c0)));
                uint4 x1 = make_uint4(0, 0, 0, 0);
                if (v1) {
                    x1 = xor4(xor4(ld_term(a.M1, k1, a.pitch, c1), ld_term(a.M2, k1, a.pitch, c1)),
                              xor4(ld_term(a.M3, i, a.pitch, c1), ld_term(T1, k1, a.pitch, c1)));
                    x1 = xor4(x1, xor4(ld_term(T2, k2, a.pitch, c1), ld_term(R, i, a.pitch, c1)));
                }
                o[c0] = x0;
                if (v1) o[c1] = x1;
            }
        }
    }
}

__global__ void __launch_bounds__(256) gather_matrix_kernel(const GatherArgs a, int64_t nch, int vec) {
    const uint32_t* T1 = a.t1.on ? a.t1.mat : nullptr;
    const uint32_t* T2 = a.t2.on ? a.t2.mat : nullptr;
    const uint32_t* R = a.r.on ? a.r.mat : nullptr;
    const int64_t total = a.rows * nch;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
        const int64_t i = t / nch, c = t - i * nch;
        const int64_t k2 = a.P2 ? (int64_t)__ldg(a.P2 + i) : i;
        const int64_t k1 = a.P1 ? (int64_t)__ldg(a.P1 + k2) : k2;
        if (vec) {
            uint4 x = xor4(xor4(ld_term(a.M1, k1, a.pitch, c), ld_term(a.M2, k1, a.pitch, c)),
                           xor4(ld_term(a.M3, i, a.pitch, c), ld_term(T1, k1, a.pitch, c)));
            x = xor4(x, xor4(ld_term(T2, k2, a.pitch, c), ld_term(R, i, a.pitch, c)));
            reinterpret_cast<uint4*>(a.out + i * a.pitch)[c] = x;
        } else {
            const int nw = (int)min((int64_t)4, a.W - 4 * c);
            for (int j = 0; j < nw; j++) {
                const int64_t w = 4 * c + j;
                uint32_t x = 0;
                if (a.M1) x ^= a.M1[k1 * a.pitch + w];
                if (a.M2) x ^= a.M2[k1 * a.pitch + w];
                if (a.M3) x ^= a.M3[i * a.pitch + w];
                if (T1) x ^= T1[k1 * a.pitch + w];
                if (T2) x ^= T2[k2 * a.pitch + w];
                if (R) x ^= R[i * a.pitch + w];
                a.out[i * a.pitch + w] = x;
            }
        }
    }
}

// out[i] = inner[outer[i]]: the composition a party precomputes offline for
// the two permutations it knows (pi12 o pi31 at P1, pi31 o pi23 at P3).
__global__ void perm_compose_kernel(const int32_t* __restrict__ outer, const int32_t* __restrict__ inner,
                                    int64_t n, int32_t* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = __ldg(inner + __ldg(outer + i));
}

// ---------------------------------------------------------------------------
// Planned two-pass gather for a permutation known ahead of the data.
//
// A party's online shuffle step is out[i] = M[k(i)] ^ (terms at i), with k a
// permutation the party fixed offline (src/shuffle.py:106-143).  A direct
// gather reads one random 16-byte row per output row; HBM serves that at
// ~1/4 of streaming bandwidth.  Since k is data-independent, the offline
// phase plans two streaming passes instead:
//
//   pass 1 (bucket scatter):  inter[pos1[j]] = M1[j] ^ M2[j]   (j sequential)
//       pos1 puts every source row into the bucket of its destination tile,
//       in increasing j within the bucket, so each bucket fills front to back
//       and its open lines merge in L2 before they are written back;
//   pass 2 (tile gather):     out[i] = tile[q2[i]] ^ R[i] ^ M3[i]
//       one CTA stages a bucket (<= 96 KB) in shared memory and emits its
//       tile in order: coalesced reads and writes.
// ---------------------------------------------------------------------------
__global__ void invert_perm_kernel(const int32_t* __restrict__ k, int64_t n, int32_t* __restrict__ inv) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) inv[k[i]] = (int32_t)i;
}

__global__ void tile_keys_kernel(const int32_t* __restrict__ inv, int64_t n, int64_t T, int32_t* __restrict__ key,
                                 int32_t* __restrict__ val) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
        key[j] = (int32_t)(inv[j] / T);
        val[j] = (int32_t)j;
    }
}

__global__ void scatter_pos_kernel(const int32_t* __restrict__ sorted_j, int64_t n, int32_t* __restrict__ pos1) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) pos1[sorted_j[p]] = (int32_t)p;
}

__global__ void local_q_kernel(const int32_t* __restrict__ k, const int32_t* __restrict__ pos1, int64_t n, int64_t T,
                               int32_t* __restrict__ q2) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        q2[i] = (int32_t)(pos1[k[i]] - (i / T) * T);
}

__global__ void bucket_scatter_kernel(const int32_t* __restrict__ pos1, const uint32_t* __restrict__ m1,
                                      const uint32_t* __restrict__ m2, int64_t rows, int64_t W,
                                      uint32_t* __restrict__ inter) {
    const int64_t total = rows * W;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
        const int64_t j = t / W, w = t - j * W;
        uint32_t v = __ldcs(m1 + t);
        if (m2) v ^= __ldcs(m2 + t);
        inter[(int64_t)__ldcs(pos1 + j) * W + w] = v;
    }
}

__global__ void __launch_bounds__(512) tile_gather_kernel(const int32_t* __restrict__ q2,
                                                          const uint32_t* __restrict__ inter,
                                                          const uint32_t* __restrict__ r,
                                                          const uint32_t* __restrict__ m3, int64_t rows, int64_t W,
                                                          int64_t T, uint32_t* __restrict__ out) {
    extern __shared__ __align__(16) uint32_t tile[];
    const int64_t ntiles = (rows + T - 1) / T;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t r0 = t * T;
        const int64_t nr = min(T, rows - r0);
        const int64_t nw = nr * W;
        const uint32_t* src = inter + r0 * W;
        __syncthreads();
        for (int64_t e = threadIdx.x; e < nw; e += blockDim.x) tile[e] = __ldcs(src + e);
        __syncthreads();
        for (int64_t e = threadIdx.x; e < nw; e += blockDim.x) {
            const int64_t li = e / W, w = e - li * W;
            const int64_t g = (r0 + li) * W + w;
            uint32_t v = tile[(int64_t)__ldcs(q2 + r0 + li) * W + w];
            if (r) v ^= __ldcs(r + g);
            if (m3) v ^= __ldcs(m3 + g);
            out[g] = v;
        }
    }
}


// 128-bit rows (the C5 shape): one thread per row, uint4 traffic only.
// Pass 2 with L2-sized windows (tile rows x row bytes > the shared-memory
// tile): a window's rows are read at random, but the grid sweeps output rows
// in order, so the live window (~32 MB) stays L2-resident and HBM sees each
// of its lines once; the streamed terms are evict-first.
__global__ void window_gather4_kernel(const int32_t* __restrict__ q2, const uint4* __restrict__ inter,
                                      const uint4* __restrict__ r, const uint4* __restrict__ m3, int64_t rows,
                                      int64_t T, uint4* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += stride) {
        const int64_t src = (i / T) * T + __ldcs(q2 + i);
        uint4 v = __ldcg(inter + src);
        if (r) v = xor4(v, __ldcs(r + i));
        if (m3) v = xor4(v, __ldcs(m3 + i));
        __stcs(out + i, v);
    }
}

__global__ void window_gather_kernel(const int32_t* __restrict__ q2, const uint32_t* __restrict__ inter,
                                     const uint32_t* __restrict__ r, const uint32_t* __restrict__ m3, int64_t rows,
                                     int64_t W, int64_t T, uint32_t* __restrict__ out) {
    const int64_t total = rows * W;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
        const int64_t i = t / W, w = t - i * W;
        const int64_t src = (i / T) * T + __ldcs(q2 + i);
        uint32_t v = __ldcg(inter + src * W + w);
        if (r) v ^= __ldcs(r + t);
        if (m3) v ^= __ldcs(m3 + t);
        __stcs(out + t, v);
    }
}

__global__ void bucket_scatter4_kernel(const int32_t* __restrict__ pos1, const uint4* __restrict__ m1,
                                       const uint4* __restrict__ m2, int64_t rows, uint4* __restrict__ inter) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < rows; j += stride) {
        uint4 v = __ldcs(m1 + j);
        if (m2) v = xor4(v, __ldcs(m2 + j));
        inter[__ldcs(pos1 + j)] = v;
    }
}

__global__ void __launch_bounds__(512) tile_gather4_kernel(const int32_t* __restrict__ q2,
                                                           const uint4* __restrict__ inter,
                                                           const uint4* __restrict__ r, const uint4* __restrict__ m3,
                                                           int64_t rows, int T, uint4* __restrict__ out) {
    extern __shared__ __align__(16) uint4 tile4[];
    const int64_t ntiles = (rows + T - 1) / T;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t r0 = t * T;
        const int nr = (int)min((int64_t)T, rows - r0);
        __syncthreads();
        for (int e = threadIdx.x; e < nr; e += blockDim.x) tile4[e] = __ldcs(inter + r0 + e);
        __syncthreads();
        for (int e = threadIdx.x; e < nr; e += blockDim.x) {
            uint4 v = tile4[__ldcs(q2 + r0 + e)];
            if (r) v = xor4(v, __ldcs(r + r0 + e));
            if (m3) v = xor4(v, __ldcs(m3 + r0 + e));
            out[r0 + e] = v;
        }
    }
}

constexpr int64_t kTileBytes = 96 * 1024;


// All reservation rounds in ONE CTA (small permutations: no host round
// trips).  Same reserve / commit / reset phases as the multi-kernel loop,
// separated by __syncthreads (which orders global memory inside the block).
constexpr int64_t kPermBlockMax = 1 << 16;

__global__ void __launch_bounds__(1024) perm_rounds_block_kernel(const int32_t* __restrict__ H, int32_t* R,
                                                                 int32_t* perm, int32_t* liveA, int32_t* liveB,
                                                                 int32_t n_live) {
    __shared__ int32_t cnt_next;
    int32_t* cur = liveA;
    int32_t* nxt = liveB;
    int32_t c = n_live;
    while (c > 0) {
        for (int32_t t = threadIdx.x; t < c; t += blockDim.x) {
            const int32_t i = cur[t];
            atomicMax(&R[i], i);
            atomicMax(&R[H[i]], i);
        }
        if (threadIdx.x == 0) cnt_next = 0;
        __syncthreads();
        for (int32_t t = threadIdx.x; t < c; t += blockDim.x) {
            const int32_t i = cur[t];
            const int32_t h = H[i];
            if (R[i] == i && R[h] == i) {
                const int32_t a = perm[i];
                perm[i] = perm[h];
                perm[h] = a;
            } else {
                nxt[atomicAdd(&cnt_next, 1)] = i;
            }
        }
        __syncthreads();
        for (int32_t t = threadIdx.x; t < c; t += blockDim.x) {
            const int32_t i = cur[t];
            R[i] = -1;
            R[H[i]] = -1;
        }
        __syncthreads();
        c = cnt_next;
        int32_t* tmp = cur;
        cur = nxt;
        nxt = tmp;
        __syncthreads();
    }
}

int shuffle_init() {
    OGM_CUDA_TRY(allow_big_smem(perm_draws_kernel, kAesTableBytes));
    OGM_CUDA_TRY(allow_big_smem(shuffle_gather_kernel<true>, kAesTableBytes));
    OGM_CUDA_TRY(allow_big_smem(tile_gather_kernel, (int)kTileBytes));
    OGM_CUDA_TRY(allow_big_smem(tile_gather4_kernel, (int)kTileBytes));
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
    if (n <= kPermBlockMax) {
        perm_rounds_block_kernel<<<1, 1024, 0, st>>>(H, R, perm, live[0], live[1], init_cnt);
        OGM_LAUNCH_CHECK();
        return OGM_OK;
    }
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

int ogm_perm_compose(int64_t n, const int32_t* outer, const int32_t* inner, int32_t* out, void* stream) {
    OGM_CHECK_ARG(n >= 0, OGM_ERR_ARG, "negative length");
    if (n == 0) return OGM_OK;
    int64_t g = (n + 255) / 256;
    const int64_t cap = (int64_t)ogm::sm_count() * 16;
    if (g > cap) g = cap;
    ogm::perm_compose_kernel<<<(int)g, 256, 0, ogm::as_stream(stream)>>>(outer, inner, n, out);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

static int set_term(ogm::GatherTerm& g, const uint8_t* key, const uint8_t* label, uint64_t index,
                    const uint32_t* mat) {
    if (mat) {
        g.on = 2;
        g.mat = mat;
    } else if (key) {
        OGM_CHECK_ARG(label, OGM_ERR_ARG, "PRF table label is required");
        g.on = 1;
        g.key = ogm::make_sched(key);
        g.label_be = ogm::label_be(label);
        g.index = index;
    }
    return OGM_OK;
}

int ogm_shuffle_gather(int64_t rows, int64_t words, int64_t width_bits, const int32_t* perm_outer,
                       const int32_t* perm_inner, const uint32_t* m1, const uint32_t* m2, const uint32_t* m3,
                       const uint8_t* t1_key, const uint8_t* t1_label, uint64_t t1_index, const uint32_t* t1_mat,
                       const uint8_t* t2_key, const uint8_t* t2_label, uint64_t t2_index, const uint32_t* t2_mat,
                       const uint8_t* r_key, const uint8_t* r_label, uint64_t r_index, const uint32_t* r_mat,
                       int64_t prf_row0, int64_t pitch, uint32_t* out, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(rows >= 0 && words >= 0 && width_bits >= 0 && (width_bits + 31) / 32 == words, OGM_ERR_ARG,
                  "table shares must have %lld words per row for width %lld", (long long)((width_bits + 31) / 32),
                  (long long)width_bits);
    OGM_CHECK_ARG(out, OGM_ERR_ARG, "output is required");
    if (rows == 0 || words == 0) return OGM_OK;
    OGM_ENSURE_INIT();
    GatherArgs a{};
    a.P1 = perm_inner;
    a.P2 = perm_outer;
    a.M1 = m1;
    a.M2 = m2;
    a.M3 = m3;
    int rc = set_term(a.t1, t1_key, t1_label, t1_index, t1_mat);
    if (!rc) rc = set_term(a.t2, t2_key, t2_label, t2_index, t2_mat);
    if (!rc) rc = set_term(a.r, r_key, r_label, r_index, r_mat);
    if (rc) return rc;
    a.out = out;
    a.rows = rows;
    a.W = words;
    a.width = width_bits;
    a.row0 = prf_row0;
    a.pitch = pitch > 0 ? pitch : words;
    OGM_CHECK_ARG(a.pitch >= words, OGM_ERR_ARG, "pitch %lld below %lld words", (long long)a.pitch, (long long)words);
    const bool online = a.t1.on == 1 || a.t2.on == 1 || a.r.on == 1;
    const int64_t work = rows * ((a.pitch + 3) / 4);
    cudaStream_t st = as_stream(stream);
    if (online) {
        shuffle_gather_kernel<true><<<aes_grid(work), kAesThreads, kAesTableBytes, st>>>(a);
    } else {
        const bool vec = (a.pitch & 3) == 0 &&
                         ((((uintptr_t)a.M1) | ((uintptr_t)a.M2) | ((uintptr_t)a.M3) | ((uintptr_t)a.out) |
                           ((uintptr_t)a.t1.mat) | ((uintptr_t)a.t2.mat) | ((uintptr_t)a.r.mat)) & 15) == 0;
        const int64_t nch = vec ? (a.pitch >> 2) : ((a.W + 3) >> 2);
        const int64_t cap = (int64_t)sm_count() * 8;
        int64_t g = (vec && nch >= 64) ? rows : (rows * nch + 255) / 256;
        if (g > cap) g = cap;
        if (vec && nch >= 64)
            gather_matrix_rows_kernel<<<(int)(g < 1 ? 1 : g), 256, 0, st>>>(a, nch);
        else
            gather_matrix_kernel<<<(int)(g < 1 ? 1 : g), 256, 0, st>>>(a, nch, vec ? 1 : 0);
    }
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

int64_t ogm_gather_tile_rows(int64_t words) {
    if (words <= 0) return 0;
    return ogm::kTileBytes / (4 * words);
}

int64_t ogm_gather_plan_workspace_bytes(int64_t n) {
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp, (int32_t*)nullptr, (int32_t*)nullptr, (int32_t*)nullptr,
                                    (int32_t*)nullptr, (int)(n > 0 ? n : 1));
    return (int64_t)temp + 5 * 4 * n + 1024;
}

int ogm_gather_plan(int64_t n, const int32_t* idx, int64_t tile_rows, int32_t* pos1, int32_t* q2, void* workspace,
                    int64_t workspace_bytes, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(n >= 0 && n < ((int64_t)1 << 31), OGM_ERR_ARG, "plan size out of range");
    OGM_CHECK_ARG(tile_rows >= 1, OGM_ERR_ARG, "tile_rows must be positive");
    if (n == 0) return OGM_OK;
    cudaStream_t st = as_stream(stream);
    uint8_t* ws = (uint8_t*)workspace;
    int32_t* inv = (int32_t*)ws;
    int32_t* key = inv + n;
    int32_t* val = key + n;
    int32_t* skey = val + n;
    int32_t* sval = skey + n;
    void* temp = (void*)(((uintptr_t)(sval + n) + 255) & ~(uintptr_t)255);
    size_t temp_bytes = (size_t)(workspace_bytes - ((uint8_t*)temp - ws));
    const int g = grid_for(n);
    invert_perm_kernel<<<g, 256, 0, st>>>(idx, n, inv);
    tile_keys_kernel<<<g, 256, 0, st>>>(inv, n, tile_rows, key, val);
    int end_bit = 1;
    while (((n - 1) / tile_rows) >> end_bit) end_bit++;
    OGM_CUDA_TRY(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, key, skey, val, sval, (int)n, 0, end_bit, st));
    scatter_pos_kernel<<<g, 256, 0, st>>>(sval, n, pos1);
    local_q_kernel<<<g, 256, 0, st>>>(idx, pos1, n, tile_rows, q2);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

int ogm_gather_planned(int64_t rows, int64_t words, int64_t tile_rows, const int32_t* pos1, const int32_t* q2,
                       const uint32_t* m1, const uint32_t* m2, const uint32_t* m3, const uint32_t* r_mat,
                       uint32_t* inter, uint32_t* out, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(rows >= 0 && words >= 1 && tile_rows >= 1, OGM_ERR_ARG, "bad planned-gather shape");
    OGM_CHECK_ARG(m1 && inter && out, OGM_ERR_ARG, "m1, inter and out are required");
    if (rows == 0) return OGM_OK;
    OGM_ENSURE_INIT();
    cudaStream_t st = as_stream(stream);
    const int64_t ntiles = (rows + tile_rows - 1) / tile_rows;
    int64_t g = ntiles;
    const int64_t cap = (int64_t)sm_count() * 2;
    if (g > cap) g = cap;
    const bool aligned = ((((uintptr_t)m1) | ((uintptr_t)m2) | ((uintptr_t)m3) | ((uintptr_t)r_mat) |
                           ((uintptr_t)inter) | ((uintptr_t)out)) & 15) == 0;
    const bool window = tile_rows * words * 4 > kTileBytes;  // L2-window pass 2 instead of smem tiles
    if (window) {
        if (words == 4 && aligned) {
            bucket_scatter4_kernel<<<grid_for(rows), 256, 0, st>>>(pos1, (const uint4*)m1, (const uint4*)m2, rows,
                                                                   (uint4*)inter);
            window_gather4_kernel<<<grid_for(rows), 256, 0, st>>>(q2, (const uint4*)inter, (const uint4*)r_mat,
                                                                  (const uint4*)m3, rows, tile_rows, (uint4*)out);
        } else {
            bucket_scatter_kernel<<<grid_for(rows * words), 256, 0, st>>>(pos1, m1, m2, rows, words, inter);
            window_gather_kernel<<<grid_for(rows * words), 256, 0, st>>>(q2, inter, r_mat, m3, rows, words,
                                                                         tile_rows, out);
        }
    } else if (words == 4 && aligned) {
        bucket_scatter4_kernel<<<grid_for(rows), 256, 0, st>>>(pos1, (const uint4*)m1, (const uint4*)m2, rows,
                                                               (uint4*)inter);
        tile_gather4_kernel<<<(int)g, 512, (size_t)(tile_rows * 16), st>>>(
            q2, (const uint4*)inter, (const uint4*)r_mat, (const uint4*)m3, rows, (int)tile_rows, (uint4*)out);
    } else {
        bucket_scatter_kernel<<<grid_for(rows * words), 256, 0, st>>>(pos1, m1, m2, rows, words, inter);
        tile_gather_kernel<<<(int)g, 512, (size_t)(tile_rows * words * 4), st>>>(q2, inter, r_mat, m3, rows,
                                                                               words, tile_rows, out);
    }
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

}  // extern "C"
