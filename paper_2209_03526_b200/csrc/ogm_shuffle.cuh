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

template <class TAB>
__device__ __forceinline__ void perm_draws_body(const TAB& T, const AesKeySched& key, uint32_t label_be,
                                                uint64_t index, int64_t n, int32_t* __restrict__ H,
                                                int32_t* __restrict__ live, int32_t* __restrict__ perm,
                                                int32_t* __restrict__ R) {
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

template <class TAB = AesTab>
__global__ void __launch_bounds__(kAesThreads) perm_draws_kernel(
    const __grid_constant__ AesKeySched key, uint32_t label_be, uint64_t index, int64_t n, int32_t* __restrict__ H,
    int32_t* __restrict__ live, int32_t* __restrict__ perm, int32_t* __restrict__ R, int32_t* __restrict__ cnts) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    TAB::fill(smem_raw);
    __syncthreads();
    const TAB T(smem_raw);
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // live counts of the multi-launch rounds (no pageable H2D copy)
        cnts[0] = (int32_t)(n - 1);
        cnts[1] = 0;
    }
    perm_draws_body(T, key, label_be, index, n, H, live, perm, R);
}

// The three permutations of one shuffle (same label, index and size,
// different pairwise keys) in one launch each for draws and rounds
// (small tables: the trio executor's shuffles).
struct PermJob {
    AesKeySched key;
    int32_t *H, *R, *live0, *live1, *perm;
};
struct PermJobs3 {
    PermJob j[3];
};

template <class TAB>
__global__ void __launch_bounds__(kAesThreads) perm_draws3_kernel(const __grid_constant__ PermJobs3 jobs, uint32_t label_be,
                                                                  uint64_t index, int64_t n) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    TAB::fill(smem_raw);
    __syncthreads();
    const TAB T(smem_raw);
    const PermJob& j = jobs.j[blockIdx.y];
    perm_draws_body(T, j.key, label_be, index, n, j.H, j.live0, j.perm, j.R);
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

template <class TAB>
__device__ __forceinline__ void prf_row_chunk(const TAB& T, const GatherTerm& g, int64_t row, int64_t W,
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

template <bool ONLINE, class TAB>
__device__ __forceinline__ void gather_chunk(const TAB& T, const GatherArgs& a, int64_t i, int64_t c,
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

template <bool ONLINE, class TAB>
__device__ __forceinline__ void gather_body(const TAB& T, const GatherArgs& a) {
    // 128-bit path when rows are 16-B pitched and every base is aligned
    const bool vec = (a.pitch & 3) == 0 &&
                     ((((uintptr_t)a.M1) | ((uintptr_t)a.M2) | ((uintptr_t)a.M3) | ((uintptr_t)a.out) |
                       ((uintptr_t)a.t1.mat) | ((uintptr_t)a.t2.mat) | ((uintptr_t)a.r.mat)) & 15) == 0;
    const int64_t nch = vec ? (a.pitch >> 2) : ((a.W + 3) >> 2);
    const uint32_t tail = (a.width & 31) ? ((1u << (a.width & 31)) - 1u) : 0xffffffffu;
    if (nch >= 64) {
        // wide rows: a CTA walks rows, its threads walk the row's 4-word chunks
        for (int64_t i = blockIdx.x; i < a.rows; i += gridDim.x)
            for (int64_t c = threadIdx.x; c < nch; c += blockDim.x) gather_chunk<ONLINE, TAB>(T, a, i, c, tail, vec);
    } else {
        const int64_t total = a.rows * nch;
        const int64_t stride = (int64_t)gridDim.x * blockDim.x;
        for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
            const int64_t i = t / nch;
            gather_chunk<ONLINE, TAB>(T, a, i, t - i * nch, tail, vec);
        }
    }
}

template <bool ONLINE, class TAB = AesTab>
__global__ void __launch_bounds__(kAesThreads) shuffle_gather_kernel(const __grid_constant__ GatherArgs a) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    if (ONLINE) {
        TAB::fill(smem_raw);
        __syncthreads();
    }
    const TAB T(smem_raw);
    gather_body<ONLINE, TAB>(T, a);
}

// Up to kMultiGather independent gathers of the same shape in ONE launch
// (blockIdx.y picks one): the trio shuffle's blinding tables of a small
// table, which are otherwise six tiny launches that each mostly fill AES
// tables.
constexpr int kMultiGather = 6;
struct GatherArgsN {
    GatherArgs g[kMultiGather];
};

template <class TAB>
__global__ void __launch_bounds__(kAesThreads) shuffle_gather_multi_kernel(const __grid_constant__ GatherArgsN m) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    TAB::fill(smem_raw);
    __syncthreads();
    const TAB T(smem_raw);
    gather_body<true, TAB>(T, m.g[blockIdx.y]);
}

// The same step when every term is a precomputed matrix (the online phase
// after ShuffleOffline, and the wide-row material build): no AES tables, so
// a lean kernel with high occupancy for the random 16-byte row reads of
// narrow tables, and a row-per-CTA streaming loop for wide rows.
__device__ __forceinline__ uint4 ld_term(const uint32_t* m, int64_t row, int64_t pitch, int64_t c) {
    return m ? __ldcs(reinterpret_cast<const uint4*>(m + row * pitch) + c) : make_uint4(0, 0, 0, 0);
}
// gathered (random-row) terms keep normal L2 caching: a planned gather's
// window must stay resident while its lines are reused
__device__ __forceinline__ uint4 ld_rand(const uint32_t* m, int64_t row, int64_t pitch, int64_t c) {
    return m ? __ldcg(reinterpret_cast<const uint4*>(m + row * pitch) + c) : make_uint4(0, 0, 0, 0);
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
        const int64_t k2 = a.P2 ? (int64_t)__ldcs(a.P2 + i) : i;
        const int64_t k1 = a.P1 ? (int64_t)(a.P2 ? __ldg(a.P1 + k2) : __ldcs(a.P1 + k2)) : k2;
        if (vec) {
            uint4 x = xor4(xor4(ld_rand(a.M1, k1, a.pitch, c), ld_rand(a.M2, k1, a.pitch, c)),
                           xor4(ld_term(a.M3, i, a.pitch, c), ld_rand(T1, k1, a.pitch, c)));
            x = xor4(x, xor4(ld_rand(T2, k2, a.pitch, c), ld_term(R, i, a.pitch, c)));
            __stcs(reinterpret_cast<uint4*>(a.out + i * a.pitch) + c, x);  // evict-first: keep L2 for the window
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

// k1 = pi12 o pi31 and k3 = pi31 o pi23 of one small shuffle in one launch
__global__ void perm_compose2_kernel(const int32_t* __restrict__ o0, const int32_t* __restrict__ i0,
                                     int32_t* __restrict__ r0, const int32_t* __restrict__ o1,
                                     const int32_t* __restrict__ i1, int32_t* __restrict__ r1, int64_t n) {
    const int32_t* outer = blockIdx.y ? o1 : o0;
    const int32_t* inner = blockIdx.y ? i1 : i0;
    int32_t* out = blockIdx.y ? r1 : r0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = __ldg(inner + __ldg(outer + i));
}

// ---------------------------------------------------------------------------
// Planned two-pass gather for a permutation known ahead of the data.
//
// A party's online shuffle step is out[i] = M[idx[i]] ^ (terms at i), with
// idx a permutation the party fixed offline (src/shuffle.py:106-143).  On
// B200 a random 16-byte row read from a table much larger than L2 costs a
// full DRAM access with its own row activation: ~33 G rows/s however narrow
// the row (profiles/r01_c5_gather_variants.md).  Random reads confined to a
// CONTIGUOUS window of <= 16 MB run at ~150-160 G rows/s (the window's DRAM
// pages stay open / L2-resident), while the same reads over scattered 4 KB
// runs do not (profiles/r01_c5_plan.md).  Since idx is data-independent, the
// offline phase factors the gather into two passes that only ever touch
// HBM sequentially or inside one contiguous window:
//
//   I-layout: output window d = [d*Wr, (d+1)*Wr) owns I-region d, holding the
//             rows its outputs need, ordered by source row; P(j) = position
//             of source row j in I.
//   pass 1 (partition): a CTA stages a tile of T consecutive source rows in
//             shared memory (TMA bulk copies, double-buffered), then writes
//             I[gdst[k]] = tile[srow[k]] for slots k in order: slots are the
//             tile's rows grouped by destination region (source order inside
//             a group), so the writes form one contiguous run per region.
//   pass 2 (window gather): out[i] = I[q2[i]] ^ R[i] ^ M3[i], q2[i] =
//             P(idx[i]) lies in region d(i): random reads inside one
//             contiguous window, sequential writes.
// ---------------------------------------------------------------------------
constexpr int64_t kWindowBytes = 8 << 20;      // pass-2 window (contiguous I-region)
constexpr int64_t kPartSmemBytes = 64 << 10;   // pass-1 tile (3 CTAs per SM)
constexpr int64_t kMaxDynSmem = 200 << 10;

// L2 scrub between the passes of a large planned gather.  Pass 1 leaves L2
// holding its (partly written, evict-first) run lines; with those resident,
// pass 2's window does not stay in L2 and every random read goes to DRAM
// (2^28 rows: 2.3 -> 5.6 ms, DRAM reads 9.7 -> 28.6 GB).  Writing one L2's
// worth of full lines in between (a memset, ~40 us) restores the fast window
// pass (profiles/r01_c5_plan.md, scripts/exp_plan11.py).  Only worth it when
// the table is far larger than L2.
constexpr int64_t kScrubMinBytes = (int64_t)2 << 30;

static void* scrub_buffer(int64_t* bytes) {
    static std::mutex mu;
    static void* buf[64] = {};
    static int64_t len[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> g(mu);
    if (!buf[dev]) {
        int l2 = 0;
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
        int64_t want = l2 > 0 ? (int64_t)l2 : ((int64_t)126 << 20);
        if (cudaMalloc(&buf[dev], (size_t)want) != cudaSuccess) {
            cudaGetLastError();
            buf[dev] = nullptr;
            return nullptr;
        }
        len[dev] = want;
    }
    *bytes = len[dev];
    return buf[dev];
}

// chunk counters for the ordered streaming passes, one small buffer per
// (device, stream): calls on one stream reuse it in stream order, calls on
// different streams never share it
static unsigned long long* flat_counters(cudaStream_t st) {
    static std::mutex mu;
    static std::vector<std::pair<std::pair<int, cudaStream_t>, void*>> bufs;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    for (auto& e : bufs)
        if (e.first.first == dev && e.first.second == st) return (unsigned long long*)e.second;
    void* p = nullptr;
    if (cudaMalloc(&p, 256) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    bufs.push_back({{dev, st}, p});
    return (unsigned long long*)p;
}

__device__ __forceinline__ uint4 xorU(uint4 a, uint4 b) { return xor4(a, b); }
__device__ __forceinline__ uint32_t xorU(uint32_t a, uint32_t b) { return a ^ b; }

__global__ void plan_inv_kernel(const int32_t* __restrict__ idx, int64_t n, int32_t* __restrict__ inv) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) inv[__ldg(idx + i)] = (int32_t)i;
}

// ---- plan construction without a global sort ------------------------------
// The I-layout is a stable sort of the sources by destination window, and
// the pass-1 slots a stable sort of each tile's sources by window.  Window d
// receives exactly Wr sources (idx is a permutation), so source j's I row is
// P(j) = d*Wr + (its rank among window d's sources) -- a sum over earlier
// tiles of the (tile, window) counts plus its rank inside its tile.  So: one
// shared-memory sort per tile (by (window, tile row): the slot order, run
// starts and counts), a per-window scan of the counts over the tiles, then
// P, gdst and q2 elementwise.  Hand-written, no library sort.
constexpr int kPlanSortMax = 16384;   // tile rows sorted in shared memory (64-bit keys, 128 KB)

// one CTA per tile (grid-stride): bitonic sort of key = window << 32 | tile row
__global__ void __launch_bounds__(1024) plan_tile_sort_kernel(const int32_t* __restrict__ inv, int64_t n, int64_t T,
                                                              int Tp, int64_t Wr, int64_t nwin,
                                                              uint16_t* __restrict__ srow,
                                                              int32_t* __restrict__ rstart,
                                                              int32_t* __restrict__ rend) {
    extern __shared__ __align__(16) unsigned long long pk[];
    const int64_t ntiles = (n + T - 1) / T;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int nt = (int)min(T, n - t * T);
        for (int e = threadIdx.x; e < Tp; e += blockDim.x)
            pk[e] = e < nt ? ((unsigned long long)(__ldg(inv + t * T + e) / Wr) << 32) | (unsigned)e : ~0ull;
        __syncthreads();
        for (int size = 2; size <= Tp; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int i = threadIdx.x; i < (Tp >> 1); i += blockDim.x) {
                    const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                    const unsigned long long a = pk[lo], b = pk[hi];
                    if ((a > b) == ((lo & size) == 0)) {
                        pk[lo] = b;
                        pk[hi] = a;
                    }
                }
                __syncthreads();
            }
        }
        for (int k = threadIdx.x; k < nt; k += blockDim.x) {
            const unsigned long long key = pk[k];
            const int64_t d = (int64_t)(key >> 32);
            srow[t * T + k] = (uint16_t)(key & 0xffffu);
            if (k == 0 || (pk[k - 1] >> 32) != (unsigned long long)d) rstart[t * nwin + d] = k;
            if (k == nt - 1 || (pk[k + 1] >> 32) != (unsigned long long)d) rend[t * nwin + d] = k + 1;
        }
        __syncthreads();   // the tile's keys are rewritten next
    }
}

// per-window scan of the (tile, window) counts over the tiles, in chunks of
// kPlanScanChunk tiles: chunk sums, then their scan (+ d * Wr), then the
// chunks' own scans -- leaving base[t][d] = the I row of run (t, d)'s first slot
constexpr int kPlanScanChunk = 256;

__global__ void plan_chunk_sums_kernel(const int32_t* __restrict__ rstart, const int32_t* __restrict__ rend,
                                       int64_t ntiles, int64_t nwin, int64_t* __restrict__ csum) {
    const int64_t nch = (ntiles + kPlanScanChunk - 1) / kPlanScanChunk;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < nch * nwin; x += stride) {
        const int64_t c = x / nwin, d = x - c * nwin;
        int64_t s = 0;
        const int64_t t1 = min(ntiles, (c + 1) * kPlanScanChunk);
        for (int64_t t = c * kPlanScanChunk; t < t1; t++) s += rend[t * nwin + d] - rstart[t * nwin + d];
        csum[x] = s;
    }
}

__global__ void plan_chunk_scan_kernel(int64_t nch, int64_t nwin, int64_t Wr, int64_t* __restrict__ csum) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; d < nwin; d += stride) {
        int64_t run = d * Wr;
        for (int64_t c = 0; c < nch; c++) {
            const int64_t v = csum[c * nwin + d];
            csum[c * nwin + d] = run;
            run += v;
        }
    }
}

// rend[t][d] becomes base[t][d] (the count is read first)
__global__ void plan_chunk_bases_kernel(const int32_t* __restrict__ rstart, int32_t* __restrict__ rend,
                                        int64_t ntiles, int64_t nwin, const int64_t* __restrict__ csum) {
    const int64_t nch = (ntiles + kPlanScanChunk - 1) / kPlanScanChunk;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < nch * nwin; x += stride) {
        const int64_t c = x / nwin, d = x - c * nwin;
        int64_t run = csum[x];
        const int64_t t1 = min(ntiles, (c + 1) * kPlanScanChunk);
        for (int64_t t = c * kPlanScanChunk; t < t1; t++) {
            const int64_t cnt = rend[t * nwin + d] - rstart[t * nwin + d];
            rend[t * nwin + d] = (int32_t)run;
            run += cnt;
        }
    }
}

// slot s of tile t holds tile row srow[s] (source j); its I row:
// gdst[s] = base[t][d] + (s's offset in its run); P[j] = gdst[s]
__global__ void plan_slots_kernel(const int32_t* __restrict__ inv, const uint16_t* __restrict__ srow, int64_t n,
                                  int64_t T, int64_t Wr, int64_t nwin, const int32_t* __restrict__ rstart,
                                  const int32_t* __restrict__ base, int32_t* __restrict__ gdst,
                                  int32_t* __restrict__ P) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += stride) {
        const int64_t t = s / T, k = s - t * T;
        const int64_t j = t * T + __ldg(srow + s);
        const int64_t d = __ldg(inv + j) / Wr;
        const int32_t g = (int32_t)(__ldg(base + t * nwin + d) + (k - __ldg(rstart + t * nwin + d)));
        gdst[s] = g;
        P[j] = g;
    }
}

__global__ void plan_q2_kernel(const int32_t* __restrict__ idx, const int32_t* __restrict__ P, int64_t n,
                               int32_t* __restrict__ q2) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) q2[i] = __ldg(P + __ldg(idx + i));
}

// ---- run tables: pass-1 destinations without a per-row index --------------
// Pass 1's slots are a tile's rows grouped by destination window, source
// order inside, and I-region d holds window d's rows in source order; so the
// slots of one (tile, window) run write consecutive I rows: gdst[s] =
// off[t][d] + s for every global slot s of run d of tile t.  A plan's run
// table -- per tile, the slot where each run starts (u16) and its offset
// (i32) -- replaces the TMA partition's 4-B-per-row gdst read with 0.05
// B/row at 2^24 rows (32 windows) and 0.75 B/row at 2^28 (512), staged with
// the tile and searched in shared memory (partitions 2-3% faster).  Per-tile
// strides are padded to 16 B for the bulk copies.  (The hand-over passes do
// not use it: a per-row search on a streaming pass's store address measured
// 10-40% slower than reading gdst; they run in I-row order instead.)
struct RunTable {
    const uint16_t* start;   // [ntiles][run_sstride(nwin)]: run d starts at slot start[d] (empty runs: the next start)
    const int32_t* off;      // [ntiles][run_ostride(nwin)]
    int nwin;
};
__host__ __device__ constexpr int run_sstride(int nwin) { return (nwin + 1 + 7) & ~7; }
__host__ __device__ constexpr int run_ostride(int nwin) { return (nwin + 3) & ~3; }

// the run holding tile slot k: the largest d < nwin with start[d] <= k
// (start[0] = 0; a fixed number of steps, so warps stay converged)
// the four plans' run tables from the C ABI's arrays (all null: none)
static inline bool run_tables(const uint16_t* const* start, const int32_t* const* off, const int64_t* nwin,
                              RunTable* rt) {
    if (!start) return false;
    for (int k = 0; k < 4; k++) rt[k] = RunTable{start[k], off ? off[k] : nullptr, nwin ? (int)nwin[k] : 0};
    return true;
}

template <bool LDG>
__device__ __forceinline__ int run_of(const uint16_t* __restrict__ start, int nwin, int k) {
    int d = 0;
    for (int step = 1 << (31 - __clz(nwin)); step; step >>= 1) {
        const int e = d + step;
        if (e < nwin && (int)(LDG ? __ldg(start + e) : start[e]) <= k) d = e;
    }
    return d;
}

__global__ void plan_runs_kernel(const int32_t* __restrict__ gdst, int64_t n, int64_t T, int64_t Wr, int nwin,
                                 uint16_t* __restrict__ start, int32_t* __restrict__ off) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int sst = run_sstride(nwin), ost = run_ostride(nwin);
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
        const int64_t t = k / T, kl = k - t * T;
        const int32_t g = __ldg(gdst + k);
        const int d = (int)(g / Wr);
        if (kl == 0 || __ldg(gdst + k - 1) / Wr != d) {
            start[t * sst + d] = (uint16_t)kl;
            off[t * ost + d] = (int32_t)(g - k);
        }
    }
}

// empty runs start where the next run starts; start[nwin] = the tile's row count
__global__ void plan_runs_fill_kernel(int64_t n, int64_t T, int nwin, uint16_t* __restrict__ start) {
    const int64_t ntiles = (n + T - 1) / T;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += stride) {
        uint16_t* s = start + t * run_sstride(nwin);
        s[nwin] = (uint16_t)(n - t * T < T ? n - t * T : T);
        for (int d = nwin - 1; d >= 0; d--)
            if (s[d] == 0xFFFF) s[d] = s[d + 1];
    }
}

// Generic pass 1 in units U (uint4 for 16-B-multiple pitches, else words);
// wu = pitch in U.  Stores are evict-first: L2 appears to keep evict-normal
// DIRTY lines ahead of clean ones, so normal stores here leave pass 2 an L2
// in which its window does not stay resident (pass 2 measured 2.26 -> 5.5
// ms, DRAM reads 9.7 -> 28.6 GB; profiles/r01_c5_plan.md).
template <typename U>
__global__ void __launch_bounds__(512) plan_partition_kernel(const U* __restrict__ m1, const U* __restrict__ m2,
                                                             const U* __restrict__ m4, const uint16_t* __restrict__ srow,
                                                             const int32_t* __restrict__ gdst, int64_t rows, int T,
                                                             int wu, U* __restrict__ inter) {
    extern __shared__ __align__(16) unsigned char part_smem[];
    U* tile = reinterpret_cast<U*>(part_smem);
    const int64_t ntiles = (rows + T - 1) / T;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t r0 = t * T;
        const int nr = (int)min((int64_t)T, rows - r0);
        const int ne = nr * wu;
        const U* a = m1 + r0 * wu;
        const U* b = m2 ? m2 + r0 * wu : nullptr;
        const U* d = m4 ? m4 + r0 * wu : nullptr;
        for (int e = threadIdx.x; e < ne; e += blockDim.x) {
            U v = __ldcs(a + e);
            if (b) v = xorU(v, __ldcs(b + e));
            if (d) v = xorU(v, __ldcs(d + e));
            tile[e] = v;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < ne; e += blockDim.x) {
            const int k = wu == 1 ? e : e / wu;
            const int c = e - k * wu;
            __stcs(inter + (int64_t)__ldcs(gdst + r0 + k) * wu + c, tile[(int)__ldcs(srow + r0 + k) * wu + c]);
        }
        __syncthreads();
    }
}

// ---- TMA-staged pass 1 for 16-byte rows (the C5 shape) --------------------
// One persistent CTA per SM; stage s holds a tile's rows (m1), srow and gdst,
// filled by cp.async.bulk on mbarrier s, two tiles ahead.  The optional
// terms m2 and m4 (x1's second component; a source-order blind) are read in
// row order, coalesced, into registers one tile ahead, and XORed into the
// staged rows before the scatter; so while tile t is written out, the loads
// of the CTA's next tile are in flight.
constexpr int kTmaTile = 4096;
constexpr int kTmaThreads = 1024;
constexpr int kTmaStageBytes = kTmaTile * (16 + 2 + 4);
constexpr int kTmaSmemBytes = 2 * kTmaStageBytes + 64;

// SLOT_M2: m2 is a blind in SLOT order (tile t, slot k <- source row
// t*T + srow[t*T + k]) and m4 is null: it is XORed into each row as the row
// is scattered, with no shared-memory XOR pass over the staged tile.
// RUNS: destinations from the plan's run table (staged per tile) instead of
// gdst; the stage is then T*18 B plus the tile's table (kTmaRunsStageBytes).
__host__ __device__ constexpr int kTmaRunsStageBytes(int nwin) {
    return kTmaTile * 18 + run_sstride(nwin) * 2 + run_ostride(nwin) * 4;
}

template <bool SLOT_M2, bool RUNS = false>
__global__ void __launch_bounds__(kTmaThreads, 1) plan_partition_tma_kernel(
    const uint4* __restrict__ m1, const uint4* __restrict__ m2, const uint4* __restrict__ m4,
    const uint16_t* __restrict__ srow, const int32_t* __restrict__ gdst, int64_t rows, uint4* __restrict__ inter,
    RunTable rt = RunTable{}) {
    extern __shared__ __align__(128) unsigned char tma_smem[];
    constexpr int T = kTmaTile;
    constexpr int Q = T / kTmaThreads;
    const int SB = RUNS ? kTmaRunsStageBytes(rt.nwin) : kTmaStageBytes;
    const int sst = run_sstride(rt.nwin), ost = run_ostride(rt.nwin);
    uint64_t* bar = reinterpret_cast<uint64_t*>(tma_smem + 2 * SB);
    auto rows_of = [&](int s) { return reinterpret_cast<uint4*>(tma_smem + s * SB); };
    auto srow_of = [&](int s) { return reinterpret_cast<uint16_t*>(tma_smem + s * SB + T * 16); };
    auto gdst_of = [&](int s) { return reinterpret_cast<int32_t*>(tma_smem + s * SB + T * 18); };
    auto start_of = [&](int s) { return reinterpret_cast<uint16_t*>(tma_smem + s * SB + T * 18); };
    auto off_of = [&](int s) { return reinterpret_cast<int32_t*>(tma_smem + s * SB + T * 18 + sst * 2); };
    const int64_t nfull = rows / T;
    const int64_t G = gridDim.x;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int64_t t, int s) {
        mbar_expect_tx(&bar[s], SB);
        bulk_g2s(rows_of(s), m1 + t * T, T * 16, &bar[s]);
        bulk_g2s(srow_of(s), srow + t * T, T * 2, &bar[s]);
        if (RUNS) {
            bulk_g2s(start_of(s), rt.start + t * sst, sst * 2, &bar[s]);
            bulk_g2s(off_of(s), rt.off + t * ost, ost * 4, &bar[s]);
        } else {
            bulk_g2s(gdst_of(s), gdst + t * T, T * 4, &bar[s]);
        }
    };
    // destination of tile t's slot k (stage s)
    auto dest = [&](int s, int64_t t, int k) -> int64_t {
        if (RUNS) return (int64_t)off_of(s)[run_of<false>(start_of(s), rt.nwin, k)] + t * T + k;
        return gdst_of(s)[k];
    };
    if (threadIdx.x == 0) {
        if (blockIdx.x < nfull) issue(blockIdx.x, 0);
        if (blockIdx.x + G < nfull) issue(blockIdx.x + G, 1);
    }
    uint4 ra[Q], rb[Q];
    const uint4 z4 = make_uint4(0, 0, 0, 0);
    auto load = [&](int64_t t) {
#pragma unroll
        for (int i = 0; i < Q; i++) {
            const int64_t e = t * T + threadIdx.x + i * kTmaThreads;
            ra[i] = m2 ? __ldcs(m2 + e) : z4;
            rb[i] = m4 ? __ldcs(m4 + e) : z4;
        }
    };
    if ((int64_t)blockIdx.x < nfull) load(blockIdx.x);
    uint32_t parity = 0;  // bit s: phase of stage s
    int s = 0;
    for (int64_t t = blockIdx.x; t < nfull; t += G) {
        mbar_wait(&bar[s], (parity >> s) & 1);
        parity ^= 1u << s;
        uint4* rs = rows_of(s);
        const uint16_t* sr = srow_of(s);
        if (SLOT_M2) {
            uint4 cur[Q];
#pragma unroll
            for (int i = 0; i < Q; i++) cur[i] = ra[i];
            if (t + G < nfull) load(t + G);   // the next tile's blind streams in during this scatter
#pragma unroll
            for (int i = 0; i < Q; i++) {
                const int k = threadIdx.x + i * kTmaThreads;
                __stcs(inter + dest(s, t, k), xor4(rs[sr[k]], cur[i]));
            }
        } else {
            if (m2 || m4) {
#pragma unroll
                for (int i = 0; i < Q; i++) {
                    const int k = threadIdx.x + i * kTmaThreads;
                    rs[k] = xor4(rs[k], xor4(ra[i], rb[i]));
                }
                __syncthreads();
                if (t + G < nfull) load(t + G);
            }
#pragma unroll
            for (int i = 0; i < Q; i++) {
                const int k = threadIdx.x + i * kTmaThreads;
                __stcs(inter + dest(s, t, k), rs[sr[k]]);
            }
        }
        __syncthreads();  // stage s fully read before it is refilled
        if (threadIdx.x == 0 && t + 2 * G < nfull) issue(t + 2 * G, s);
        s ^= 1;
    }
    // ragged last tile (rows % T): the last CTA, straight from global
    if (blockIdx.x == G - 1 && rows % T) {
        const int64_t b0 = nfull * T;
        const int nr = (int)(rows - b0);
        for (int k = threadIdx.x; k < nr; k += kTmaThreads) {
            const int j = __ldcs(srow + b0 + k);
            uint4 v = __ldcs(m1 + b0 + j);
            if (m2) v = xor4(v, __ldcs(m2 + b0 + (SLOT_M2 ? k : j)));
            if (m4) v = xor4(v, __ldcs(m4 + b0 + j));
            const int64_t dst = RUNS ? (int64_t)__ldg(rt.off + nfull * ost + run_of<true>(rt.start + nfull * sst, rt.nwin, k)) + b0 + k
                                     : (int64_t)__ldcs(gdst + b0 + k);
            __stcs(inter + dst, v);
        }
    }
}


// ---- chained passes: one party's window pass feeding the next party's
// partition pass, tile by tile in shared memory -------------------------------
// In the 3-party shuffle a message is consumed by exactly one gather of the
// receiving party (x1 -> c1 at pi23, y1 -> R3 at k3).  With planned gathers
// the sender's window pass writes the message in order and the receiver's
// partition pass reads it straight back.  Here one persistent CTA per SM
// builds a 4096-row tile of the message from the sender's intermediate
// (random reads inside one 8 MB window), XORs the receiver's source-order
// blind into it in shared memory, and writes the tile out as the receiver's
// window runs.  The message never round-trips HBM (optionally it is also
// stored, for transcripts and tests).
// The window gathers go straight to shared memory with cp.async, three
// tiles deep, so a CTA always has two tiles of random reads in flight while
// it scatters the third (register-staged loads allowed only one: each tile
// then waited out its slowest DRAM miss, 2.7 vs 5.0 TB/s).  q, blind, srow
// and gdst are read in slot / row order, coalesced.
constexpr int kChainStages = 3;
constexpr int kChainSmem2 = kChainStages * kTmaTile * 16;
constexpr int64_t kDualMaxBytes = (int64_t)256 << 20;  // measured: one dual window pass wins up to 2^24 rows

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// SLOT_BLIND: `blind` is in the receiver partition's SLOT order (tile t,
// slot k -> source row t*T + srow[t*T + k], arranged offline), so it is
// XORed into each row as it is scattered: no separate shared-memory XOR pass
// over the staged tile (the pass this kernel was MIO-throttled on).  Else
// `blind` is in source (tile row) order and XORed in place before the scatter.
template <bool SLOT_BLIND>
__global__ void __launch_bounds__(kTmaThreads, 1) plan_chain_kernel(
    const int32_t* __restrict__ q, const uint4* __restrict__ inter_a, const uint4* __restrict__ blind,
    const uint16_t* __restrict__ srow, const int32_t* __restrict__ gdst, int64_t rows, uint4* __restrict__ inter_b,
    uint4* __restrict__ msg) {
    extern __shared__ __align__(128) unsigned char tma_smem[];
    constexpr int T = kTmaTile;
    constexpr int Q = T / kTmaThreads;
    auto buf = [&](int64_t j) { return reinterpret_cast<uint4*>(tma_smem) + (int)(j % kChainStages) * T; };
    const int64_t nfull = rows / T;
    const int64_t G = gridDim.x;
    const int64_t nmine = nfull > blockIdx.x ? (nfull - blockIdx.x + G - 1) / G : 0;
    auto tile = [&](int64_t j) { return blockIdx.x + j * G; };
    int32_t qn[Q];
    auto load_q = [&](int64_t j) {
        if (j < nmine) {
#pragma unroll
            for (int i = 0; i < Q; i++) qn[i] = __ldcs(q + tile(j) * T + threadIdx.x + i * kTmaThreads);
        }
    };
    auto gather = [&](int64_t j) {  // uses qn (tile j), then prefetches q of tile j + 1
        if (j < nmine) {
            uint4* b = buf(j);
#pragma unroll
            for (int i = 0; i < Q; i++) cp_async16(b + threadIdx.x + i * kTmaThreads, inter_a + qn[i]);
        }
        cp_async_commit();  // empty groups keep the wait count uniform
        load_q(j + 1);
    };
    load_q(0);
    gather(0);
    gather(1);
    const uint4 z4 = make_uint4(0, 0, 0, 0);
    for (int64_t j = 0; j < nmine; j++) {
        const int64_t t = tile(j);
        uint4 bl[Q];
        uint16_t sr[Q];
        int32_t gd[Q];
#pragma unroll
        for (int i = 0; i < Q; i++) {
            const int k = threadIdx.x + i * kTmaThreads;
            bl[i] = blind ? __ldcs(blind + t * T + k) : z4;
            sr[i] = __ldcs(srow + t * T + k);
            gd[i] = __ldcs(gdst + t * T + k);
        }
        gather(j + 2);   // buffer (j + 2) % 3 was freed by the barrier closing tile j - 1
        cp_async_wait<2>();  // this thread's gathers of tile j have landed
        uint4* rs = buf(j);
        if ((!SLOT_BLIND && blind) || msg) {
#pragma unroll
            for (int i = 0; i < Q; i++) {
                const int k = threadIdx.x + i * kTmaThreads;
                const uint4 v = rs[k];
                if (msg) __stcs(msg + t * T + k, v);
                if (!SLOT_BLIND) rs[k] = xor4(v, bl[i]);
            }
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < Q; i++) __stcs(inter_b + gd[i], SLOT_BLIND ? xor4(rs[sr[i]], bl[i]) : rs[sr[i]]);
        __syncthreads();
    }
    cp_async_wait<0>();
    // ragged last tile: the last CTA, through buffer 0 (nothing is in flight any more)
    if (blockIdx.x == G - 1 && rows % T) {
        __syncthreads();
        const int64_t b0 = nfull * T;
        const int nr = (int)(rows - b0);
        uint4* rs = buf(0);
        for (int k = threadIdx.x; k < nr; k += kTmaThreads) {
            const uint4 m = __ldcg(inter_a + __ldcs(q + b0 + k));
            if (msg) __stcs(msg + b0 + k, m);
            rs[k] = (!SLOT_BLIND && blind) ? xor4(m, __ldcs(blind + b0 + k)) : m;
        }
        __syncthreads();
        for (int k = threadIdx.x; k < nr; k += kTmaThreads) {
            const uint4 v = rs[__ldcs(srow + b0 + k)];
            __stcs(inter_b + __ldcs(gdst + b0 + k), (SLOT_BLIND && blind) ? xor4(v, __ldcs(blind + b0 + k)) : v);
        }
    }
}

// The chained hand-over without shared memory: the sender's window index,
// composed offline with the receiver partition's slot order
// (qs[t*T + k] = q[t*T + srow[t*T + k]]), lets each slot fetch its message
// row straight from the sender's window and scatter it to the receiver's
// intermediate: ib[gdst[s]] = ia[qs[s]] ^ bl[s] (bl in slot order).  Slots
// of one tile are consecutive, so the reads stay inside one window (L2) and
// consecutive slots of a run write consecutive rows.  A flat streaming pass
// like the window passes: no staging, no barriers, no MIO traffic -- the
// staged kernel above was bound by exactly those (LSU and MIO throttles).
// Chunks of kFlatChunk slots are handed out in order through an atomic
// counter, so the slots in flight stay inside a narrow range of consecutive
// tiles -- one sender window -- however unevenly the blocks progress (a
// grid-stride loop lets slow blocks lag into earlier windows; at 2^26 rows
// that made the window reads miss L2: 77 instead of 40 B/row).  Chunk size
// measured at 256 / 512 / 1024 / 2048 / 4096 slots: 1024 is best (2^24:
// 0.91 / 0.82 / 0.82 / 0.84 / 0.94 ms; 2^28: 15.8 / 15.0 / 14.8 / 15.1 / 17.3).
constexpr int kFlatChunk = 1024;

// the first row of this block's next chunk: handed out in order through the
// counter `next` (all threads get the block's value), or, without a counter,
// round-robin over blocks (grid-stride order)
__device__ __forceinline__ int64_t next_chunk(unsigned long long* next, int64_t* slot, int64_t round) {
    if (!next) return ((int64_t)blockIdx.x + round * gridDim.x) * kFlatChunk;
    if (threadIdx.x == 0) *slot = (int64_t)atomicAdd(next, 1ull);
    __syncthreads();
    const int64_t c = *slot;
    __syncthreads();
    return c * kFlatChunk;
}

__global__ void __launch_bounds__(256) chain_flat_kernel(const int32_t* __restrict__ qs,
                                                         const uint4* __restrict__ ia,
                                                         const uint4* __restrict__ bl,
                                                         const int32_t* __restrict__ gdst, int64_t rows,
                                                         uint4* __restrict__ ib, unsigned long long* next) {
    __shared__ int64_t chunk;
    for (int64_t round = 0;; round++) {
        const int64_t c0 = next_chunk(next, &chunk, round);
        if (c0 >= rows) break;
        const int64_t c1 = min(rows, c0 + kFlatChunk);
#pragma unroll 4
        for (int64_t s = c0 + threadIdx.x; s < c1; s += blockDim.x) {
            uint4 v = __ldcg(ia + __ldcs(qs + s));
            if (bl) v = xor4(v, __ldcs(bl + s));
            __stcs(ib + __ldcs(gdst + s), v);
        }
    }
}

// The flat hand-over in the receiver's I-row order (the product path):
// ib[p] = ia[qi[p]] ^ bl[p] for every I row p of the receiving plan, qi[p] =
// q[src[p]] and bl composed offline in that order -- so no destination
// index is read and every write is sequential (the slot-order pass above
// reads gdst and, at 2^28 rows, scatters 128-B runs).  Chunk c covers rows
// [m*C, (m+1)*C) of region r = c % nreg, m = c / nreg: the chunks in flight
// sit at the same offset of every region, and a region's rows are in source
// order, so their sources -- and the sender window rows they read -- stay
// inside one narrow source range (the L2-resident sender window), as in slot
// order.  Measured per pass: 2^24 142 us (slot order 153), 2^28 1.8-2.2 ms
// (2.0-2.4); whole shuffle -5% at 2^24-2^28 (profiles/r02_c5_chain_ncu.txt).
__global__ void __launch_bounds__(256) chain_inter_kernel(const int32_t* __restrict__ qi,
                                                          const uint4* __restrict__ ia,
                                                          const uint4* __restrict__ bl, int64_t rows, int64_t wr,
                                                          uint4* __restrict__ ib, unsigned long long* next) {
    __shared__ int64_t chunk;
    const int64_t nreg = (rows + wr - 1) / wr, per = (wr + kFlatChunk - 1) / kFlatChunk;
    for (int64_t round = 0;; round++) {
        const int64_t c = next_chunk(next, &chunk, round) / kFlatChunk;
        if (c >= nreg * per) break;
        const int64_t r = c % nreg, m = c / nreg;
        const int64_t p0 = r * wr + m * kFlatChunk;
        const int64_t p1 = min(min(p0 + kFlatChunk, (r + 1) * wr), rows);
#pragma unroll 4
        for (int64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
            uint4 v = __ldcg(ia + __ldcs(qi + p));
            if (bl) v = xor4(v, __ldcs(bl + p));
            __stcs(ib + p, v);
        }
    }
}

// The flag column of a flag-split fetch (csrc/ogm_fetch.cuh) rides along the
// final window passes: composed (ogm_flag_open_composed), it needs the rows
// in output order -- P2's c1 bits, P3's R3 bits and the opened column --
// which these passes walk anyway.  Each warp owns 32 consecutive output
// rows, so a bit column word is one ballot.  All pointers null = a plain
// shuffle.
struct FlagTail {
    const int32_t* kc;        // c1's bits: f12[kc[i]] ^ uwf[i]  (kc = k1 o pi23)
    const int32_t* kr;        // R3's bits: f3[kr[i]] ^ vzf[i] ^ c1  (kr = pi12 o k3)
    const uint32_t* f12;      // P1's f1 ^ f2
    const uint32_t* f3;       // P2's third component
    const uint32_t* uwf;      // composed blinds (output order)
    const uint32_t* vzf;
    const uint32_t* r1f;      // R1, R2 flag columns (for the open)
    const uint32_t* r2f;
    uint32_t* c1f;            // P2's c1 bits (needed between the split passes)
    uint32_t* r3f;            // the new component's flag column
    uint32_t* plain;          // the opened column R1f ^ R2f ^ R3f
};

__device__ __forceinline__ uint32_t tail_bit(const uint32_t* __restrict__ v, int64_t j) {
    return (__ldg(v + (j >> 5)) >> (j & 31)) & 1u;
}

// FLAG: 0 none; 1 c1 bits (the first of the split passes); 2 R3 bits and the
// open (the second split pass, c1 bits from pass 1); 3 both (the dual pass)
template <int FLAG>
__device__ __forceinline__ void flag_tail_word(const FlagTail& ft, int64_t base, int64_t i, bool valid) {
    uint32_t bc = 0, br = 0;
    if (valid) {
        if (FLAG & 1) bc = tail_bit(ft.f12, __ldcs(ft.kc + i));
        if (FLAG & 2) br = tail_bit(ft.f3, __ldcs(ft.kr + i));
    }
    const uint32_t wc = (FLAG & 1) ? __ballot_sync(0xffffffffu, bc) : 0u;
    const uint32_t wr = (FLAG & 2) ? __ballot_sync(0xffffffffu, br) : 0u;
    if ((threadIdx.x & 31) == 0) {
        const int64_t w = base >> 5;
        uint32_t c;
        if (FLAG & 1) {
            c = wc ^ __ldg(ft.uwf + w);
            if (ft.c1f) ft.c1f[w] = c;
        } else {
            c = __ldg(ft.c1f + w);
        }
        if (FLAG & 2) {
            const uint32_t r = wr ^ c ^ __ldg(ft.vzf + w);
            ft.r3f[w] = r;
            if (ft.plain) ft.plain[w] = __ldg(ft.r1f + w) ^ __ldg(ft.r2f + w) ^ r;
        }
    }
}

// the last window passes of two planned gathers with the same output order,
// XORed: R3[i] = Ir[qr[i]] ^ c1[i], c1[i] = Ic[qc[i]] (msg: c1 stored too).
// One row per thread.  Measured: 4 rows per thread LOSE (2^24 0.89 -> 0.93
// ms, 2^28 16.3 -> 22.4 ms): the grid then spans 4x more output rows at once,
// i.e. reads from several windows at a time, and the windows stop staying in
// L2 (the same effect as two windows per pass above 256 MB).  Warps walk 32
// consecutive rows together (the flag tail's ballots).
template <int FLAG>
__global__ void __launch_bounds__(256) win_gather_dual4_kernel(const int32_t* __restrict__ qa,
                                                               const uint4* __restrict__ ia,
                                                               const int32_t* __restrict__ qb,
                                                               const uint4* __restrict__ ib, int64_t rows,
                                                               uint4* __restrict__ out, uint4* __restrict__ msg,
                                                               const uint4* __restrict__ ta,
                                                               const __grid_constant__ FlagTail ft) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < rows; base += stride) {
        const int64_t i = base + (threadIdx.x & 31);
        const bool valid = i < rows;
        if (valid) {
            uint4 va = __ldcg(ia + __ldcs(qa + i));
            if (ta) va = xor4(va, __ldcs(ta + i));
            const uint4 vb = __ldcg(ib + __ldcs(qb + i));
            if (msg) __stcs(msg + i, va);
            __stcs(out + i, xor4(va, vb));
        }
        if (FLAG) flag_tail_word<FLAG>(ft, base, i, valid);
    }
}

// pass 2 for 16-byte rows (the C5 shape): a lean kernel, since with
// window-local sources the instruction count per row matters
template <int FLAG>
__global__ void __launch_bounds__(256) win_gather4_kernel(const int32_t* __restrict__ q, const uint4* __restrict__ m1,
                                                          const uint4* __restrict__ m3, const uint4* __restrict__ r,
                                                          int64_t rows, uint4* __restrict__ out,
                                                          const __grid_constant__ FlagTail ft) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < rows; base += stride) {
        const int64_t i = base + (threadIdx.x & 31);
        const bool valid = i < rows;
        if (valid) {
            uint4 v = __ldcg(m1 + __ldcs(q + i));
            if (m3) v = xor4(v, __ldcs(m3 + i));
            if (r) v = xor4(v, __ldcs(r + i));
            __stcs(out + i, v);
        }
        if (FLAG) flag_tail_word<FLAG>(ft, base, i, valid);
    }
}


// All reservation rounds in ONE CTA (small permutations: no host round
// trips).  Same reserve / commit / reset phases as the multi-kernel loop,
// separated by __syncthreads (which orders global memory inside the block).
constexpr int64_t kPermBlockMax = 1 << 16;

__device__ __forceinline__ void perm_rounds_block_body(const int32_t* __restrict__ H, int32_t* R,
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

__global__ void __launch_bounds__(1024) perm_rounds_block_kernel(const int32_t* __restrict__ H, int32_t* R,
                                                                 int32_t* perm, int32_t* liveA, int32_t* liveB,
                                                                 int32_t n_live) {
    perm_rounds_block_body(H, R, perm, liveA, liveB, n_live);
}

__global__ void __launch_bounds__(1024) perm_rounds3_block_kernel(const __grid_constant__ PermJobs3 jobs, int32_t n_live) {
    const PermJob& j = jobs.j[blockIdx.x];
    perm_rounds_block_body(j.H, j.R, j.perm, j.live0, j.live1, n_live);
}

int shuffle_init() {
    OGM_CUDA_TRY(allow_big_smem(perm_draws_kernel<AesTab>, kAesTableBytes));
    OGM_CUDA_TRY(allow_big_smem(shuffle_gather_kernel<true, AesTab>, kAesTableBytes));
    OGM_CUDA_TRY(prefer_l1(win_gather4_kernel<0>));
    OGM_CUDA_TRY(prefer_l1(win_gather_dual4_kernel<0>));
    OGM_CUDA_TRY(prefer_l1(gather_matrix_kernel));
    OGM_CUDA_TRY(prefer_l1(gather_matrix_rows_kernel));
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
    aes_launch(perm_draws_kernel<AesTab>, perm_draws_kernel<AesTabSmall>, n, kAesThreads, st, ks, label_be(label),
               index, n, H, live[0], perm, R, cnts);
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

// ---------------------------------------------------------------------------
// The online phase of a whole 3-party shuffle (offline material prepared:
// composed permutations, permuted combined blinds) in ONE cooperative launch
// for tables that sit in L2 (<= 64 MB): the four party steps of
// src/shuffle.py:106-143 as three grid-synchronised phases
//   x1 = (a ^ b)[k1] ^ U,  y1 = c[pi12] ^ V     (P1, P2: independent)
//   c1 = x1[pi23] ^ W                           (P2, after x1 arrives)
//   R3 = y1[k3] ^ c1 ^ Z                        (P3, after y1, c1 arrive)
// Every message is still written to memory; only the launch boundaries go.
// 16-byte rows (pitch 4 words).
// ---------------------------------------------------------------------------
struct Shuffle4Args {
    const int32_t *k1, *pi12, *pi23, *k3;
    const uint4 *a, *b, *c, *U, *V, *W, *Z;
    uint4 *x1, *y1, *c1, *r3;
    int64_t rows;
};

__global__ void __launch_bounds__(256) shuffle_online_coop_kernel(const Shuffle4Args p) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t i = t0; i < p.rows; i += stride) {
        const int64_t k = __ldg(p.k1 + i), j = __ldg(p.pi12 + i);
        p.x1[i] = ogm::xor4(ogm::xor4(__ldcg(p.a + k), __ldcg(p.b + k)), __ldcs(p.U + i));
        p.y1[i] = ogm::xor4(__ldcg(p.c + j), __ldcs(p.V + i));
    }
    grid.sync();
    // c1 (P2 -> P3) feeds R3 at the same index: one phase, c1 kept in registers (stored only
    // when the caller wants the message)
    for (int64_t i = t0; i < p.rows; i += stride) {
        const uint4 c = ogm::xor4(__ldcg(p.x1 + __ldg(p.pi23 + i)), __ldcs(p.W + i));
        if (p.c1) p.c1[i] = c;
        p.r3[i] = ogm::xor4(ogm::xor4(__ldcg(p.y1 + __ldg(p.k3 + i)), c), __ldcs(p.Z + i));
    }
}

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

int ogm_perm_invert(int64_t n, const int32_t* perm, int32_t* inv, void* stream) {
    OGM_CHECK_ARG(n >= 0 && n < ((int64_t)1 << 31), OGM_ERR_ARG, "permutation size out of range");
    if (n == 0) return OGM_OK;
    ogm::plan_inv_kernel<<<ogm::grid_for(n), 256, 0, ogm::as_stream(stream)>>>(perm, n, inv);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
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

static void launch_matrix_gather(const ogm::GatherArgs& a, cudaStream_t st) {
    using namespace ogm;
    const bool vec = (a.pitch & 3) == 0 &&
                     ((((uintptr_t)a.M1) | ((uintptr_t)a.M2) | ((uintptr_t)a.M3) | ((uintptr_t)a.out) |
                       ((uintptr_t)a.t1.mat) | ((uintptr_t)a.t2.mat) | ((uintptr_t)a.r.mat)) & 15) == 0;
    const int64_t nch = vec ? (a.pitch >> 2) : ((a.W + 3) >> 2);
    const int64_t cap = (int64_t)sm_count() * 8;
    int64_t g = (vec && nch >= 64) ? a.rows : (a.rows * nch + 255) / 256;
    if (g > cap) g = cap;
    if (vec && nch >= 64)
        gather_matrix_rows_kernel<<<(int)(g < 1 ? 1 : g), 256, 0, st>>>(a, nch);
    else
        gather_matrix_kernel<<<(int)(g < 1 ? 1 : g), 256, 0, st>>>(a, nch, vec ? 1 : 0);
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
        aes_launch(shuffle_gather_kernel<true, AesTab>, shuffle_gather_kernel<true, AesTabSmall>, work, kAesThreads, st,
                   a);
    } else {
        launch_matrix_gather(a, st);
    }
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

int64_t ogm_gather_window_rows(int64_t pitch_words) {
    if (pitch_words <= 0) return 0;
    const int64_t r = ogm::kWindowBytes / (4 * pitch_words);
    return r > 0 ? r : 1;
}

int64_t ogm_gather_tile_rows(int64_t pitch_words) {
    if (pitch_words <= 0) return 0;
    int64_t r = ogm::kPartSmemBytes / (4 * pitch_words);
    if (r > ogm::kPlanSortMax) r = ogm::kPlanSortMax;
    return r > 0 ? r : 1;
}

int64_t ogm_gather_plan_workspace_bytes(int64_t n, int64_t window_rows, int64_t tile_rows) {
    if (n <= 0 || window_rows < 1 || tile_rows < 1) return 256;
    const int64_t nwin = (n + window_rows - 1) / window_rows, ntiles = (n + tile_rows - 1) / tile_rows;
    const int64_t nch = (ntiles + ogm::kPlanScanChunk - 1) / ogm::kPlanScanChunk;
    // inv, P; the (tile, window) run starts and ends/bases; the chunk sums
    return 2 * 4 * n + 2 * 4 * ntiles * nwin + 8 * nch * nwin + 1024;
}

int ogm_gather_plan(int64_t n, const int32_t* idx, int64_t window_rows, int64_t tile_rows, int32_t* q2,
                    int32_t* gdst, uint16_t* srow, void* workspace, int64_t workspace_bytes, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(n >= 0 && n < ((int64_t)1 << 31), OGM_ERR_ARG, "plan size out of range");
    OGM_CHECK_ARG(window_rows >= 1 && tile_rows >= 1 && tile_rows <= kPlanSortMax, OGM_ERR_ARG,
                  "window_rows must be positive and tile_rows in [1, %d]", kPlanSortMax);
    OGM_CHECK_ARG(workspace_bytes >= ogm_gather_plan_workspace_bytes(n, window_rows, tile_rows), OGM_ERR_ARG,
                  "plan workspace too small");
    if (n == 0) return OGM_OK;
    OGM_CHECK_ARG(idx && q2 && gdst && srow && workspace, OGM_ERR_ARG, "idx, the plan outputs and workspace are required");
    const int64_t nwin = (n + window_rows - 1) / window_rows;
    const int64_t ntiles = (n + tile_rows - 1) / tile_rows;
    const int64_t nch = (ntiles + kPlanScanChunk - 1) / kPlanScanChunk;
    cudaStream_t st = as_stream(stream);
    int32_t* inv = (int32_t*)workspace;
    int32_t* P = inv + n;
    int32_t* rstart = P + n;
    int32_t* rend = rstart + ntiles * nwin;
    int64_t* csum = (int64_t*)(((uintptr_t)(rend + ntiles * nwin) + 7) & ~(uintptr_t)7);
    const int g = grid_for(n);
    plan_inv_kernel<<<g, 256, 0, st>>>(idx, n, inv);
    OGM_CUDA_TRY(cudaMemsetAsync(rstart, 0, (size_t)(2 * 4 * ntiles * nwin), st));   // empty runs: count 0
    int Tp = 1;
    while (Tp < tile_rows) Tp <<= 1;
    const int smem = Tp * 8;
    OGM_CUDA_TRY(allow_big_smem(plan_tile_sort_kernel, smem));
    const int gt = (int)std::min<int64_t>(ntiles, (int64_t)sm_count() * (smem <= (48 << 10) ? 4 : 1));
    plan_tile_sort_kernel<<<gt, std::min(1024, std::max(32, Tp / 2)), smem, st>>>(inv, n, tile_rows, Tp,
                                                                                   window_rows, nwin, srow, rstart,
                                                                                   rend);
    const int gc = grid_for(nch * nwin);
    plan_chunk_sums_kernel<<<gc, 256, 0, st>>>(rstart, rend, ntiles, nwin, csum);
    plan_chunk_scan_kernel<<<grid_for(nwin), 256, 0, st>>>(nch, nwin, window_rows, csum);
    plan_chunk_bases_kernel<<<gc, 256, 0, st>>>(rstart, rend, ntiles, nwin, csum);
    plan_slots_kernel<<<g, 256, 0, st>>>(inv, srow, n, tile_rows, window_rows, nwin, rstart, rend, gdst, P);
    plan_q2_kernel<<<g, 256, 0, st>>>(idx, P, n, q2);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

int ogm_gather_plan_runs(int64_t n, int64_t window_rows, int64_t tile_rows, const int32_t* gdst, uint16_t* start,
                         int32_t* off, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(n >= 0 && n < ((int64_t)1 << 31), OGM_ERR_ARG, "plan size out of range");
    OGM_CHECK_ARG(window_rows >= 1 && tile_rows >= 1 && tile_rows <= 32768, OGM_ERR_ARG,
                  "window_rows must be positive and tile_rows in [1, 32768]");
    if (n == 0) return OGM_OK;
    OGM_CHECK_ARG(gdst && start && off, OGM_ERR_ARG, "gdst and the run table are required");
    const int64_t nwin = (n + window_rows - 1) / window_rows;
    OGM_CHECK_ARG(nwin < (1 << 20), OGM_ERR_ARG, "too many windows");
    const int64_t ntiles = (n + tile_rows - 1) / tile_rows;
    cudaStream_t st = as_stream(stream);
    OGM_CUDA_TRY(cudaMemsetAsync(start, 0xFF, (size_t)(ntiles * run_sstride((int)nwin) * 2), st));
    OGM_CUDA_TRY(cudaMemsetAsync(off, 0, (size_t)(ntiles * run_ostride((int)nwin) * 4), st));
    plan_runs_kernel<<<grid_for(n), 256, 0, st>>>(gdst, n, tile_rows, window_rows, (int)nwin, start, off);
    plan_runs_fill_kernel<<<grid_for(ntiles), 256, 0, st>>>(n, tile_rows, (int)nwin, start);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

int ogm_gather_planned(int64_t rows, int64_t words, int64_t pitch, int64_t tile_rows, const int32_t* q2,
                       const int32_t* gdst, const uint16_t* srow, const uint32_t* m1, const uint32_t* m2,
                       const uint32_t* m4, const uint32_t* m3, const uint32_t* r_mat, uint32_t* inter, uint32_t* out,
                       int passes, void* stream) {
    using namespace ogm;
    if (pitch <= 0) pitch = words;
    OGM_CHECK_ARG(passes >= 1 && passes <= 3, OGM_ERR_ARG, "passes must be 1, 2 or 3 (bit 0 pass 1, bit 1 pass 2)");
    OGM_CHECK_ARG(rows >= 0 && words >= 1 && pitch >= words, OGM_ERR_ARG, "bad planned-gather shape");
    OGM_CHECK_ARG(tile_rows >= 1 && tile_rows <= 65536 && tile_rows * pitch * 4 <= (int64_t)kMaxDynSmem,
                  OGM_ERR_ARG, "tile of %lld rows x %lld words exceeds shared memory", (long long)tile_rows,
                  (long long)pitch);
    OGM_CHECK_ARG(q2 && gdst && srow && m1 && inter && out, OGM_ERR_ARG,
                  "q2, gdst, srow, m1, inter and out are required");
    if (rows == 0) return OGM_OK;
    OGM_ENSURE_INIT();
    cudaStream_t st = as_stream(stream);
    const bool vec = (pitch & 3) == 0 && ((((uintptr_t)m1) | ((uintptr_t)m2) | ((uintptr_t)m3) | ((uintptr_t)r_mat) |
                                           ((uintptr_t)m4) | ((uintptr_t)inter) | ((uintptr_t)out)) & 15) == 0;
    const size_t smem = (size_t)(tile_rows * pitch * 4);
    const int64_t ntiles = (rows + tile_rows - 1) / tile_rows;
    int per_sm = 1;
    int64_t g;
    if (!(passes & 1)) {
    } else if (vec && pitch == 4 && tile_rows == kTmaTile) {
        OGM_CUDA_TRY(allow_big_smem(plan_partition_tma_kernel<false>, kTmaSmemBytes));
        g = std::min<int64_t>(std::max<int64_t>(ntiles, 1), (int64_t)sm_count());
        plan_partition_tma_kernel<false><<<(int)g, kTmaThreads, kTmaSmemBytes, st>>>(
            (const uint4*)m1, (const uint4*)m2, (const uint4*)m4, srow, gdst, rows, (uint4*)inter);
    } else if (vec) {
        OGM_CUDA_TRY(allow_big_smem(plan_partition_kernel<uint4>, (int)smem));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, plan_partition_kernel<uint4>, 512, smem);
        g = std::min<int64_t>(ntiles, (int64_t)sm_count() * std::max(per_sm, 1));
        plan_partition_kernel<uint4><<<(int)g, 512, smem, st>>>((const uint4*)m1, (const uint4*)m2, (const uint4*)m4,
                                                                srow, gdst, rows,
                                                                (int)tile_rows, (int)(pitch / 4), (uint4*)inter);
    } else {
        OGM_CUDA_TRY(allow_big_smem(plan_partition_kernel<uint32_t>, (int)smem));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, plan_partition_kernel<uint32_t>, 512, smem);
        g = std::min<int64_t>(ntiles, (int64_t)sm_count() * std::max(per_sm, 1));
        plan_partition_kernel<uint32_t><<<(int)g, 512, smem, st>>>(m1, m2, m4, srow, gdst, rows, (int)tile_rows,
                                                                   (int)pitch, inter);
    }
    if (passes == 3 && rows * pitch * 4 >= kScrubMinBytes) {
        int64_t sb = 0;
        if (void* sc = scrub_buffer(&sb)) OGM_CUDA_TRY(cudaMemsetAsync(sc, 0, (size_t)sb, st));
    }
    if (!(passes & 2)) {
    } else if (pitch == 4 && vec) {
        int64_t g2 = std::min<int64_t>((rows + 255) / 256, (int64_t)sm_count() * 8);
        win_gather4_kernel<0><<<(int)g2, 256, 0, st>>>(q2, (const uint4*)inter, (const uint4*)m3, (const uint4*)r_mat,
                                                    rows, (uint4*)out, FlagTail{});
    } else {
        GatherArgs a{};
        a.rows = rows;
        a.W = words;
        a.width = 32 * words;
        a.pitch = pitch;
        a.P1 = q2;
        a.M1 = inter;
        a.M3 = m3;
        if (r_mat) {
            a.r.on = 2;
            a.r.mat = r_mat;
        }
        a.out = out;
        launch_matrix_gather(a, st);
    }
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

// ---------------------------------------------------------------------------
// Trio fast path: one whole 3-party shuffle (src/shuffle.py:80-144) for the
// three co-resident parties in ONE call -- offline material and online steps
// -- replacing ~25 host dispatches per shuffle (trio.Trio.shuffle).  Same
// launches, same order, same results as the Python composition:
//   pi12, pi23, pi31 = SHPI permutations of table id `tid`
//   k1 = pi12 o pi31, k3 = pi31 o pi23                    (perm_compose)
//   U = T12[k1] ^ T31[pi31], V = T12[pi12], W = T23[pi23] ^ R2,
//   Z = T31[k3] ^ T23[pi23] ^ R1     (AES on the fly for narrow rows, from
//                                     ogm_prf_rows tables for >= 64 words)
//   x1 = pack(c1 ^ c2)[k1] ^ U, y1 = pack(c3)[pi12] ^ V       (P1, P2)
//   c1 = x1[pi23] ^ W                                          (P2)
//   R3 = y1[k3] ^ c1 ^ Z                                       (P3)
// out = (R1, R2, R3), the new components.
// ---------------------------------------------------------------------------
static int64_t al256(int64_t b) { return (b + 255) & ~(int64_t)255; }

namespace ogm {
// the three SHPI permutations of one small shuffle: one draws launch, one
// rounds launch (a CTA per permutation); ws holds 3 perm workspaces
static int seeded_permutations3_small(const uint8_t* const keys[3], const uint8_t* label, uint64_t index,
                                      int64_t n, int32_t* const perms[3], uint8_t* ws, cudaStream_t st) {
    PermJobs3 J{};
    for (int q = 0; q < 3; q++) {
        int32_t* H = (int32_t*)(ws + q * perm_ws_bytes(n) + 256);
        J.j[q] = PermJob{make_sched(keys[q]), H, H + n, H + 2 * n, H + 3 * n, perms[q]};
    }
    const int64_t g = (n + kAesSmallThreads - 1) / kAesSmallThreads;
    perm_draws3_kernel<AesTabSmall><<<dim3((unsigned)(g > 0 ? g : 1), 3), kAesSmallThreads, kAesSmallBytes, st>>>(
        J, label_be(label), index, n);
    if (n >= 2) perm_rounds3_block_kernel<<<3, 1024, 0, st>>>(J, (int32_t)(n - 1));
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}
}  // namespace ogm

int64_t ogm_trio_shuffle_workspace_bytes(int64_t rows, int64_t pitch) {
    if (rows <= 0) return 256;
    return 5 * al256(rows * 4) + 3 * al256(ogm_perm_workspace_bytes(rows)) + 7 * al256(rows * pitch * 4);
}

int ogm_trio_shuffle(const uint8_t* s12, const uint8_t* s23, const uint8_t* s31, uint64_t tid, int64_t rows,
                     int64_t width_bits, int64_t pitch, int nfields, const uint32_t* const* fields,
                     const int64_t* fpitch, const int64_t* fwidth, const uint32_t* const* flags,
                     uint32_t* const* out, void* workspace, int64_t workspace_bytes, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(s12 && s23 && s31 && out && fields, OGM_ERR_ARG, "seeds, fields and outputs are required");
    OGM_CHECK_ARG(rows >= 0 && nfields >= 1 && width_bits >= 1 && pitch >= (width_bits + 31) / 32 && pitch % 4 == 0,
                  OGM_ERR_ARG, "bad trio shuffle shape");
    OGM_CHECK_ARG(workspace_bytes >= ogm_trio_shuffle_workspace_bytes(rows, pitch), OGM_ERR_ARG,
                  "trio shuffle workspace too small");
    if (rows == 0) return OGM_OK;
    static const uint8_t kPi[4] = {'S', 'H', 'P', 'I'}, kTb[4] = {'S', 'H', 'T', 'B'}, kRd[4] = {'S', 'H', 'R', 'D'};
    uint8_t* w = (uint8_t*)workspace;
    auto take = [&](int64_t bytes) { uint8_t* p = w; w += al256(bytes); return p; };
    int32_t* pi12 = (int32_t*)take(rows * 4);
    int32_t* pi23 = (int32_t*)take(rows * 4);
    int32_t* pi31 = (int32_t*)take(rows * 4);
    int32_t* k1 = (int32_t*)take(rows * 4);
    int32_t* k3 = (int32_t*)take(rows * 4);
    void* pws = take(3 * al256(ogm_perm_workspace_bytes(rows)));
    const int64_t tb = rows * pitch * 4;
    uint32_t *u = (uint32_t*)take(tb), *v = (uint32_t*)take(tb), *wm = (uint32_t*)take(tb), *z = (uint32_t*)take(tb);
    uint32_t *x1 = (uint32_t*)take(tb), *y1 = (uint32_t*)take(tb), *c1 = (uint32_t*)take(tb);
    const int64_t W = (width_bits + 31) / 32;
    int rc;
#define OGM_TRY(x) \
    if ((rc = (x)) != OGM_OK) return rc
    OGM_ENSURE_INIT();
    const bool small = rows <= kPermBlockMax && rows <= kAesSmallMaxWork && (width_bits + 31) / 32 < 64;
    if (small) {
        // small tables (the trio executor's shuffles): 3 permutations per launch, all six
        // blinding/output tables in one launch
        const uint8_t* keys[3] = {s12, s23, s31};
        int32_t* perms[3] = {pi12, pi23, pi31};
        static_assert(sizeof(void*) == 8, "64-bit");
        OGM_TRY(seeded_permutations3_small(keys, kPi, tid, rows, perms, (uint8_t*)pws, as_stream(stream)));
    } else {
        OGM_TRY(ogm_seeded_permutation(s12, kPi, tid, rows, pi12, pws, stream));
        OGM_TRY(ogm_seeded_permutation(s23, kPi, tid, rows, pi23, pws, stream));
        OGM_TRY(ogm_seeded_permutation(s31, kPi, tid, rows, pi31, pws, stream));
    }
    if (small) {
        perm_compose2_kernel<<<dim3((unsigned)((rows + 255) / 256), 2), 256, 0, as_stream(stream)>>>(
            pi31, pi12, k1, pi23, pi31, k3, rows);
        OGM_LAUNCH_CHECK();
    } else {
        OGM_TRY(ogm_perm_compose(rows, pi31, pi12, k1, stream));
        OGM_TRY(ogm_perm_compose(rows, pi23, pi31, k3, stream));
    }
    uint32_t *r1 = out[0], *r2 = out[1], *r3 = out[2];
    const int64_t P = pitch;
    if (small) {
        // U = T12[k1] ^ T31[pi31], V = T12[pi12], W = T23[pi23] ^ R2, Z = T31[k3] ^ T23[pi23] ^ R1, R1, R2:
        // the same six gathers as below, blockIdx.y-indexed in one launch
        GatherArgsN m{};
        auto base = [&](GatherArgs& a, uint32_t* o) {
            a.out = o;
            a.rows = rows;
            a.W = W;
            a.width = width_bits;
            a.row0 = 0;
            a.pitch = P;
        };
        auto term = [&](GatherTerm& g, const uint8_t* key, const uint8_t* label) { set_term(g, key, label, tid, nullptr); };
        GatherArgs* g = m.g;
        base(g[0], u); g[0].P2 = pi31; g[0].P1 = pi12; term(g[0].t1, s12, kTb); term(g[0].t2, s31, kTb);
        base(g[1], v); g[1].P1 = pi12; term(g[1].t1, s12, kTb);
        base(g[2], wm); g[2].P1 = pi23; term(g[2].t1, s23, kTb); term(g[2].r, s12, kRd);
        base(g[3], z); g[3].P2 = pi23; g[3].P1 = pi31; term(g[3].t1, s31, kTb); term(g[3].t2, s23, kTb);
        term(g[3].r, s31, kRd);
        base(g[4], r1); term(g[4].r, s31, kRd);
        base(g[5], r2); term(g[5].r, s12, kRd);
        const int64_t work = rows * ((P + 3) / 4);
        const int64_t gx = (work + kAesSmallThreads - 1) / kAesSmallThreads;
        shuffle_gather_multi_kernel<AesTabSmall><<<dim3((unsigned)(gx > 0 ? gx : 1), kMultiGather), kAesSmallThreads,
                                                   kAesSmallBytes, as_stream(stream)>>>(m);
        OGM_LAUNCH_CHECK();
    } else {
    OGM_TRY(ogm_prf_rows(s31, kRd, tid, rows, width_bits, pitch, r1, stream));
    OGM_TRY(ogm_prf_rows(s12, kRd, tid, rows, width_bits, pitch, r2, stream));
    }
    if (small) {
    } else if (W >= 64) {
        // wide rows: each blinding table once at the AES rate, then streaming combines
        uint32_t *t12 = x1, *t31 = y1, *t23 = c1;  // scratch until the online steps
        OGM_TRY(ogm_prf_rows(s12, kTb, tid, rows, width_bits, pitch, t12, stream));
        OGM_TRY(ogm_prf_rows(s31, kTb, tid, rows, width_bits, pitch, t31, stream));
        OGM_TRY(ogm_prf_rows(s23, kTb, tid, rows, width_bits, pitch, t23, stream));
        OGM_TRY(ogm_shuffle_gather(rows, W, width_bits, pi31, pi12, nullptr, nullptr, nullptr, nullptr, nullptr, 0,
                                   t12, nullptr, nullptr, 0, t31, nullptr, nullptr, 0, nullptr, 0, P, u, stream));
        OGM_TRY(ogm_shuffle_gather(rows, W, width_bits, nullptr, pi12, nullptr, nullptr, nullptr, nullptr, nullptr, 0,
                                   t12, nullptr, nullptr, 0, nullptr, nullptr, nullptr, 0, nullptr, 0, P, v, stream));
        OGM_TRY(ogm_shuffle_gather(rows, W, width_bits, nullptr, pi23, nullptr, nullptr, nullptr, nullptr, nullptr, 0,
                                   t23, nullptr, nullptr, 0, nullptr, nullptr, nullptr, 0, r2, 0, P, wm, stream));
        OGM_TRY(ogm_shuffle_gather(rows, W, width_bits, pi23, pi31, nullptr, nullptr, nullptr, nullptr, nullptr, 0,
                                   t31, nullptr, nullptr, 0, t23, nullptr, nullptr, 0, r1, 0, P, z, stream));
    } else {
        OGM_TRY(ogm_shuffle_gather(rows, W, width_bits, pi31, pi12, nullptr, nullptr, nullptr, s12, kTb, tid, nullptr,
                                   s31, kTb, tid, nullptr, nullptr, nullptr, 0, nullptr, 0, P, u, stream));
        OGM_TRY(ogm_shuffle_gather(rows, W, width_bits, nullptr, pi12, nullptr, nullptr, nullptr, s12, kTb, tid,
                                   nullptr, nullptr, nullptr, 0, nullptr, nullptr, nullptr, 0, nullptr, 0, P, v,
                                   stream));
        OGM_TRY(ogm_shuffle_gather(rows, W, width_bits, nullptr, pi23, nullptr, nullptr, nullptr, s23, kTb, tid,
                                   nullptr, nullptr, nullptr, 0, nullptr, s12, kRd, tid, nullptr, 0, P, wm, stream));
        OGM_TRY(ogm_shuffle_gather(rows, W, width_bits, pi23, pi31, nullptr, nullptr, nullptr, s31, kTb, tid, nullptr,
                                   s23, kTb, tid, nullptr, s31, kRd, tid, nullptr, 0, P, z, stream));
    }
    // online: P1 packs c1 ^ c2 at k1, P2 packs c3 at pi12 (ogm_pack_gather, set-major field lists)
    const uint32_t* set01[2 * 64];
    OGM_CHECK_ARG(nfields <= 64, OGM_ERR_ARG, "at most 64 fields");
    for (int f = 0; f < nfields; f++) {
        set01[f] = fields[f];
        set01[nfields + f] = fields[nfields + f];
    }
    const uint32_t* fl01[2] = {flags ? flags[0] : nullptr, flags ? flags[1] : nullptr};
    const uint32_t* fl2[1] = {flags ? flags[2] : nullptr};
    OGM_TRY(ogm_pack_gather(rows, k1, 2, flags ? fl01 : nullptr, nfields, set01, fpitch, fwidth, u, x1, P, stream));
    OGM_TRY(ogm_pack_gather(rows, pi12, 1, flags ? fl2 : nullptr, nfields, fields + 2 * nfields, fpitch + 2 * nfields,
                            fwidth, v, y1, P, stream));
    OGM_TRY(ogm_shuffle_gather(rows, W, width_bits, nullptr, pi23, x1, nullptr, nullptr, nullptr, nullptr, 0, nullptr,
                               nullptr, nullptr, 0, nullptr, nullptr, nullptr, 0, wm, 0, P, c1, stream));
    OGM_TRY(ogm_shuffle_gather(rows, W, width_bits, nullptr, k3, y1, nullptr, c1, nullptr, nullptr, 0, nullptr, nullptr,
                               nullptr, 0, nullptr, nullptr, nullptr, 0, z, 0, P, r3, stream));
#undef OGM_TRY
    return OGM_OK;
}

// The online phase of one 3-party shuffle of 16-byte rows for the three
// co-resident parties over planned gathers, with each message handed from
// sender to receiver in shared memory (plan_chain_kernel).  Plans in
// step order x1 (k1), y1 (pi12), c1 (pi23), R3 (k3); every blind is in the
// source order of its step (ShuffleOffline with plans):
//   P1: I1 = part1(a ^ b ^ U')            P2: Iy = part2(c ^ V')
//   P1 -> P2: x1 = win1(I1); Ic = part3(x1 ^ W')
//   P2 -> P3: y1 = win2(Iy); Ir = part4(y1 ^ Z')
//   P2 -> P3, P3: c1 = win3(Ic); R3 = win4(Ir) ^ c1
// x1, y1, c1 are optional copies of the messages; inter[0..2] are three
// table-sized scratch buffers.
}  // extern "C"
namespace ogm {
int shuffle_online_planned_impl(int64_t rows, const int32_t* const* q2, const int32_t* const* gdst,
                                const uint16_t* const* srow, const uint32_t* a, const uint32_t* b, const uint32_t* c,
                                const uint32_t* u_src, const uint32_t* v_src, int v_order, const uint32_t* w_src,
                                int w_order, const uint32_t* z_src, int z_order, uint32_t* const* inter, uint32_t* x1,
                                uint32_t* y1, uint32_t* c1, uint32_t* r3, const FlagTail* ft,
                                const int32_t* const* qs, const RunTable* runs, const int64_t* wrows,
                                void* stream);
}
extern "C" {

int ogm_shuffle_online_planned_w_output_order(int64_t rows) {
    return rows * 16 > ogm::kDualMaxBytes ? 1 : 0;
}

int ogm_shuffle_online_planned(int64_t rows, const int32_t* const* q2, const int32_t* const* gdst,
                               const uint16_t* const* srow, const uint32_t* a, const uint32_t* b, const uint32_t* c,
                               const uint32_t* u_src, const uint32_t* v_src, const uint32_t* w_src,
                               const uint32_t* z_src, uint32_t* const* inter, uint32_t* x1, uint32_t* y1, uint32_t* c1,
                               uint32_t* r3, void* stream) {
    return ogm_shuffle_online_planned_ex(rows, q2, gdst, srow, a, b, c, u_src, v_src, 0, w_src, 0, z_src, 0, inter,
                                         x1, y1, c1, r3, stream);
}

int ogm_shuffle_online_planned_ex(int64_t rows, const int32_t* const* q2, const int32_t* const* gdst,
                                  const uint16_t* const* srow, const uint32_t* a, const uint32_t* b,
                                  const uint32_t* c, const uint32_t* u_src, const uint32_t* v_src, int v_order,
                                  const uint32_t* w_src, int w_order, const uint32_t* z_src, int z_order,
                                  uint32_t* const* inter, uint32_t* x1, uint32_t* y1, uint32_t* c1, uint32_t* r3,
                                  void* stream) {
    return ogm::shuffle_online_planned_impl(rows, q2, gdst, srow, a, b, c, u_src, v_src, v_order, w_src, w_order,
                                            z_src, z_order, inter, x1, y1, c1, r3, nullptr, nullptr, nullptr, nullptr, stream);
}
}  // extern "C"

namespace ogm {
// the chained online shuffle; ft (optional) adds the flag-split fetch's flag
// tail to the final window passes (ogm_fetch128_online)
int shuffle_online_planned_impl(int64_t rows, const int32_t* const* q2, const int32_t* const* gdst,
                                const uint16_t* const* srow, const uint32_t* a, const uint32_t* b, const uint32_t* c,
                                const uint32_t* u_src, const uint32_t* v_src, int v_order, const uint32_t* w_src,
                                int w_order, const uint32_t* z_src, int z_order, uint32_t* const* inter, uint32_t* x1,
                                uint32_t* y1, uint32_t* c1, uint32_t* r3, const FlagTail* ft,
                                const int32_t* const* qs, const RunTable* runs, const int64_t* wrows,
                                void* stream) {
    OGM_CHECK_ARG(rows >= 0 && rows < ((int64_t)1 << 31), OGM_ERR_ARG, "rows out of range");
    OGM_CHECK_ARG(q2 && gdst && srow && inter, OGM_ERR_ARG, "plans and scratch are required");
    const void* need[] = {a, b, c, u_src, v_src, w_src, z_src, r3, inter[0], inter[1], inter[2]};
    for (const void* p : need)
        OGM_CHECK_ARG(p && (((uintptr_t)p) & 15) == 0, OGM_ERR_ARG, "16-byte aligned tables are required");
    const void* opt[] = {x1, y1, c1};
    for (const void* p : opt) OGM_CHECK_ARG((((uintptr_t)p) & 15) == 0, OGM_ERR_ARG, "16-byte aligned tables are required");
    for (int k = 0; k < 4; k++) OGM_CHECK_ARG(q2[k] && gdst[k] && srow[k], OGM_ERR_ARG, "plan %d is incomplete", k);
    if (rows == 0) return OGM_OK;
    OGM_ENSURE_INIT();
    cudaStream_t st = as_stream(stream);
    OGM_CHECK_ARG((v_order == 0 || v_order == 2) && w_order >= 0 && w_order <= 3 && z_order >= 0 && z_order <= 3 &&
                      z_order != 1,
                  OGM_ERR_ARG, "blind orders: v 0 (source) / 2 (slot), w 0 / 1 (output) / 2 / 3 (I order), z 0 / 2 / 3");
    OGM_CHECK_ARG((w_order != 3 && z_order != 3) || (qs && qs[0] && qs[1] && wrows && wrows[2] > 0 && wrows[3] > 0),
                  OGM_ERR_ARG, "I-order blinds need the I-order indices and the receiving plans' window rows");
    OGM_CUDA_TRY(allow_big_smem(plan_partition_tma_kernel<false>, kTmaSmemBytes));
    OGM_CUDA_TRY(allow_big_smem(plan_partition_tma_kernel<true>, kTmaSmemBytes));
    if (runs)
        for (int k = 0; k < 4; k++)
            OGM_CHECK_ARG(runs[k].start && runs[k].off && runs[k].nwin >= 1 &&
                              2 * kTmaRunsStageBytes(runs[k].nwin) + 64 <= kMaxDynSmem,
                          OGM_ERR_ARG, "run table %d is incomplete or too large", k);
    const int runs_smem0 = runs ? 2 * kTmaRunsStageBytes(runs[0].nwin) + 64 : 0;
    const int runs_smem1 = runs ? 2 * kTmaRunsStageBytes(runs[1].nwin) + 64 : 0;
    if (runs) {
        OGM_CUDA_TRY(allow_big_smem(plan_partition_tma_kernel<false, true>, std::max(runs_smem0, runs_smem1)));
        OGM_CUDA_TRY(allow_big_smem(plan_partition_tma_kernel<true, true>, std::max(runs_smem0, runs_smem1)));
    }
    OGM_CUDA_TRY(allow_big_smem(plan_chain_kernel<false>, kChainSmem2));
    OGM_CUDA_TRY(allow_big_smem(plan_chain_kernel<true>, kChainSmem2));
    const int64_t ntiles = (rows + kTmaTile - 1) / kTmaTile;
    const int g = (int)std::min<int64_t>(ntiles, (int64_t)sm_count());
    const bool scrub = rows * 16 >= kScrubMinBytes;
    auto scrub_l2 = [&]() -> int {
        int64_t sb = 0;
        if (scrub)
            if (void* sc = scrub_buffer(&sb)) OGM_CUDA_TRY(cudaMemsetAsync(sc, 0, (size_t)sb, st));
        return OGM_OK;
    };
    using U4 = const uint4*;
    uint4 *i0 = (uint4*)inter[0], *i1 = (uint4*)inter[1], *i2 = (uint4*)inter[2];
    constexpr int TT = kTmaThreads;
    if (runs) {
        plan_partition_tma_kernel<false, true><<<g, TT, runs_smem0, st>>>((U4)a, (U4)b, (U4)u_src, srow[0], nullptr,
                                                                          rows, i0, runs[0]);
        if (v_order == 2)
            plan_partition_tma_kernel<true, true><<<g, TT, runs_smem1, st>>>((U4)c, (U4)v_src, nullptr, srow[1],
                                                                             nullptr, rows, i1, runs[1]);
        else
            plan_partition_tma_kernel<false, true><<<g, TT, runs_smem1, st>>>((U4)c, (U4)v_src, nullptr, srow[1],
                                                                              nullptr, rows, i1, runs[1]);
    } else {
        plan_partition_tma_kernel<false><<<g, TT, kTmaSmemBytes, st>>>((U4)a, (U4)b, (U4)u_src, srow[0], gdst[0],
                                                                       rows, i0);
        if (v_order == 2)
            plan_partition_tma_kernel<true><<<g, TT, kTmaSmemBytes, st>>>((U4)c, (U4)v_src, nullptr, srow[1], gdst[1],
                                                                          rows, i1);
        else
            plan_partition_tma_kernel<false><<<g, TT, kTmaSmemBytes, st>>>((U4)c, (U4)v_src, nullptr, srow[1],
                                                                           gdst[1], rows, i1);
    }
    const int64_t gf = std::min<int64_t>((rows + kFlatChunk - 1) / kFlatChunk, (int64_t)sm_count() * 8);
    if (scrub_l2() != OGM_OK) return OGM_ERR_CUDA;
    // above the dual-pass size P2's blind W stays in c1's OUTPUT order: the x1 -> c1 chain kernel
    // then needs no XOR pass (it is MIO-bound) and W streams in c1's own window pass (2-3% at
    // 2^26-2^28; with the dual pass an extra stream costs more than it saves)
    const bool w_out = w_order == 1;
    auto chain = [&](bool slot, const int32_t* q, const uint4* ia, const uint4* bl, const uint16_t* sr,
                     const int32_t* gd, uint4* ib, uint4* msg) {
        if (slot)
            plan_chain_kernel<true><<<g, TT, kChainSmem2, st>>>(q, ia, bl, sr, gd, rows, ib, msg);
        else
            plan_chain_kernel<false><<<g, TT, kChainSmem2, st>>>(q, ia, bl, sr, gd, rows, ib, msg);
    };
    unsigned long long* ctr = flat_counters(st);   // the two chain passes' chunk counters
    if (!ctr) {
        set_error("could not allocate the chunk counters");
        return OGM_ERR_CUDA;
    }
    OGM_CUDA_TRY(cudaMemsetAsync(ctr, 0, 2 * sizeof(unsigned long long), st));
    // the flat hand-over needs the composed indices, slot-order (or no) blinds and no message copies
    const bool inter_order = z_order == 3;   // the I-order hand-over (w_order 3, or 1 with W streamed later)
    if (inter_order && !x1)
        chain_inter_kernel<<<(int)gf, 256, 0, st>>>(qs[0], i0, w_out ? nullptr : (U4)w_src, rows, wrows[2], i2, ctr);
    else if (qs && qs[0] && !x1 && (w_order == 2 || w_out))
        chain_flat_kernel<<<(int)gf, 256, 0, st>>>(qs[0], i0, w_out ? nullptr : (U4)w_src, gdst[2], rows, i2, ctr);
    else
        chain(w_order == 2, q2[0], i0, w_out ? nullptr : (U4)w_src, srow[2], gdst[2], i2, (uint4*)x1);
    if (scrub_l2() != OGM_OK) return OGM_ERR_CUDA;
    if (inter_order && !y1)
        chain_inter_kernel<<<(int)gf, 256, 0, st>>>(qs[1], i1, (U4)z_src, rows, wrows[3], i0, ctr + 1);
    else if (qs && qs[1] && !y1 && z_order == 2)
        chain_flat_kernel<<<(int)gf, 256, 0, st>>>(qs[1], i1, (U4)z_src, gdst[3], rows, i0, ctr + 1);
    else
        chain(z_order == 2, q2[1], i1, (U4)z_src, srow[3], gdst[3], i0, (uint4*)y1);
    if (scrub_l2() != OGM_OK) return OGM_ERR_CUDA;
    // window passes keep one row per thread over a grid-stride loop: handing them ordered chunks
    // (as the flat chain passes) measured 2-4% slower at 2^24-2^28
    const int64_t g2 = std::min<int64_t>((rows + 255) / 256, (int64_t)sm_count() * 8);
    const FlagTail none{};
    if (rows * 16 <= kDualMaxBytes) {
        if (ft)
            win_gather_dual4_kernel<3><<<(int)g2, 256, 0, st>>>(q2[2], i2, q2[3], i0, rows, (uint4*)r3, (uint4*)c1,
                                                                w_out ? (U4)w_src : nullptr, *ft);
        else
            win_gather_dual4_kernel<0><<<(int)g2, 256, 0, st>>>(q2[2], i2, q2[3], i0, rows, (uint4*)r3, (uint4*)c1,
                                                                w_out ? (U4)w_src : nullptr, none);
    } else {
        // two random windows at once thrash L2 far above its size (2^26 rows: 2.06 ms and 11 GB read
        // instead of 2.7; smaller windows do not rescue it, scripts/exp_chain_win.py): c1's window
        // pass, then R3's with c1 streamed
        uint4* c1m = c1 ? (uint4*)c1 : i1;
        if (ft)
            win_gather4_kernel<1><<<(int)g2, 256, 0, st>>>(q2[2], i2, w_out ? (U4)w_src : nullptr, nullptr, rows, c1m,
                                                           *ft);
        else
            win_gather4_kernel<0><<<(int)g2, 256, 0, st>>>(q2[2], i2, w_out ? (U4)w_src : nullptr, nullptr, rows, c1m,
                                                           none);
        if (scrub_l2() != OGM_OK) return OGM_ERR_CUDA;
        if (ft)
            win_gather4_kernel<2><<<(int)g2, 256, 0, st>>>(q2[3], i0, c1m, nullptr, rows, (uint4*)r3, *ft);
        else
            win_gather4_kernel<0><<<(int)g2, 256, 0, st>>>(q2[3], i0, c1m, nullptr, rows, (uint4*)r3, none);
    }
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}
}  // namespace ogm

extern "C" {

int ogm_shuffle_online_planned_slots(int64_t rows, const int32_t* const* q2, const int32_t* const* gdst,
                                     const uint16_t* const* srow, const int32_t* const* qs,
                                     const uint16_t* const* run_start, const int32_t* const* run_off,
                                     const int64_t* run_nwin, const int64_t* wrows, const uint32_t* a,
                                     const uint32_t* b, const uint32_t* c, const uint32_t* u_src,
                                     const uint32_t* v_src, const uint32_t* w_blind, int w_order,
                                     const uint32_t* z_slot, int z_order, uint32_t* const* inter, uint32_t* r3,
                                     void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(qs && qs[0] && qs[1], OGM_ERR_ARG, "the two composed slot indices are required");
    OGM_CHECK_ARG(w_order >= 1 && w_order <= 3 && (z_order == 2 || z_order == 3), OGM_ERR_ARG,
                  "W in c1's output (1), slot (2) or I (3) order; Z in slot (2) or I (3) order");
    RunTable rt[4];
    const bool runs = run_tables(run_start, run_off, run_nwin, rt);
    return shuffle_online_planned_impl(rows, q2, gdst, srow, a, b, c, u_src, v_src, 0, w_blind, w_order, z_slot,
                                       z_order, inter, nullptr, nullptr, nullptr, r3, nullptr, qs,
                                       runs ? rt : nullptr, wrows, stream);
}

int ogm_shuffle_online_fused(int64_t rows, const int32_t* k1, const int32_t* pi12, const int32_t* pi23,
                             const int32_t* k3, const uint32_t* a, const uint32_t* b, const uint32_t* c,
                             const uint32_t* U, const uint32_t* V, const uint32_t* W, const uint32_t* Z, uint32_t* x1,
                             uint32_t* y1, uint32_t* c1, uint32_t* r3, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(rows >= 0 && rows < ((int64_t)1 << 31), OGM_ERR_ARG, "rows out of range");
    const void* ptrs[] = {a, b, c, U, V, W, Z, x1, y1, r3};
    for (const void* q : ptrs)
        OGM_CHECK_ARG(q && (((uintptr_t)q) & 15) == 0, OGM_ERR_ARG, "16-byte aligned tables are required");
    OGM_CHECK_ARG((((uintptr_t)c1) & 15) == 0, OGM_ERR_ARG, "16-byte aligned tables are required");
    OGM_CHECK_ARG(k1 && pi12 && pi23 && k3, OGM_ERR_ARG, "permutations are required");
    if (rows == 0) return OGM_OK;
    OGM_ENSURE_INIT();
    Shuffle4Args p{k1, pi12, pi23, k3, (const uint4*)a, (const uint4*)b, (const uint4*)c, (const uint4*)U,
                   (const uint4*)V, (const uint4*)W, (const uint4*)Z, (uint4*)x1, (uint4*)y1, (uint4*)c1,
                   (uint4*)r3, rows};
    int per_sm = 0;
    OGM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, shuffle_online_coop_kernel, 256, 0));
    int64_t g = (int64_t)sm_count() * std::max(per_sm, 1);
    const int64_t need = (rows + 255) / 256;
    if (g > need) g = need;
    void* args[] = {&p};
    OGM_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)shuffle_online_coop_kernel, dim3((unsigned)g), dim3(256),
                                             args, 0, as_stream(stream)));
    return OGM_OK;
}

}  // extern "C"
