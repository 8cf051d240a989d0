// ogm_fetch.cuh -- the fetch of flagged rows after a shuffle (src/engine.py:
// 220-270, sec_fetch_multi) for the C5 shape, and the hand-written public
// compaction behind every open-and-keep (src/engine.py:252,327 np.nonzero).
//
// Flag-split layout.  sec_fetch_multi packs each row as [flag | fields] with
// the flag at bit 0 (src/engine.py:227-233), so a 128-bit payload row is 129
// bits = 5 words, its payload shifted by one bit.  Every step of the shuffle
// (src/shuffle.py:106-143) is a row permutation plus XORs of equally laid out
// rows, and both commute with any fixed re-layout of the bits inside a row.
// So the rows are kept SPLIT -- the 128-bit payload as one aligned 16-byte
// row and the flag as a bit column -- and the data-independent blinds, drawn
// in the reference's 5-word layout, are split the same way offline
// (split_flag_rows_kernel).  The payload then shuffles through the 16-byte
// chained planned gathers of ogm_shuffle.cuh, the flag column through two
// small bit-gather kernels here, and the kept rows' payloads are exactly the
// bits 1..128 the reference slices out.
#pragma once

#include "ogm_common.cuh"

namespace ogm {

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t bit_at(const uint32_t* __restrict__ v, int64_t j) {
    return (__ldg(v + (j >> 5)) >> (j & 31)) & 1u;
}

// in: rows of `pitch` words, 129 logical bits; out: payload bits 1..128 as
// one uint4 per row, flag bit 0 packed 32 rows per word (clean tail).
__global__ void __launch_bounds__(256) split_flag_rows_kernel(const uint32_t* __restrict__ in, int64_t pitch,
                                                              int64_t rows, uint4* __restrict__ payload,
                                                              uint32_t* __restrict__ flags) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < rows; base += stride) {
        const int64_t i = base + lane_id();
        uint32_t f = 0;
        if (i < rows) {
            const uint32_t* r = in + i * pitch;
            const uint32_t w0 = __ldcs(r), w1 = __ldcs(r + 1), w2 = __ldcs(r + 2), w3 = __ldcs(r + 3),
                           w4 = __ldcs(r + 4);
            payload[i] = make_uint4(__funnelshift_r(w0, w1, 1), __funnelshift_r(w1, w2, 1), __funnelshift_r(w2, w3, 1),
                                    __funnelshift_r(w3, w4, 1));
            f = w0 & 1u;
        }
        const uint32_t b = __ballot_sync(0xffffffffu, f);
        if (lane_id() == 0) flags[base >> 5] = b;
    }
}

// Flag column of the 3-party shuffle, phase 1 (P1's x1 and P2's y1 bits):
//   x1f[i] = f12[k1[i]] ^ Uf[i],   y1f[i] = f3[pi12[i]] ^ Vf[i]
// (f12 = f1 ^ f2, P1's two components XORed in one streaming pass first).
// One warp per 32 output rows = one output word.  The bit columns are small
// (rows / 8 bytes) and stay in L2; what bounds these kernels is the L1
// rate for uncoalesced loads (~1 sector per clock per SM: every random bit
// read is its own sector), so each row costs exactly one random read per
// gather step (profiles/r02_c5_fetch_ncu.md).
__global__ void __launch_bounds__(256) flag_xor2_kernel(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                                                        int64_t nw, uint32_t* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += stride) out[w] = a[w] ^ b[w];
}

__global__ void __launch_bounds__(256) flag_shuffle1_kernel(int64_t rows, const int32_t* __restrict__ k1,
                                                            const int32_t* __restrict__ pi12,
                                                            const uint32_t* __restrict__ f12,
                                                            const uint32_t* __restrict__ f3,
                                                            const uint32_t* __restrict__ uf,
                                                            const uint32_t* __restrict__ vf, uint32_t* __restrict__ x1f,
                                                            uint32_t* __restrict__ y1f) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < rows; base += stride) {
        const int64_t i = base + lane_id();
        uint32_t bx = 0, by = 0;
        if (i < rows) {
            bx = bit_at(f12, __ldcs(k1 + i));
            by = bit_at(f3, __ldcs(pi12 + i));
        }
        const uint32_t wx = __ballot_sync(0xffffffffu, bx), wy = __ballot_sync(0xffffffffu, by);
        if (lane_id() == 0) {
            const int64_t w = base >> 5;
            x1f[w] = wx ^ __ldg(uf + w);
            y1f[w] = wy ^ __ldg(vf + w);
        }
    }
}

// Phase 2 (P2's c1 and P3's R3 bits), plus the opened flag column:
//   c1f[i] = x1f[pi23[i]] ^ Wf[i],   r3f[i] = y1f[k3[i]] ^ c1f[i] ^ Zf[i]
//   plain  = R1f ^ R2f ^ r3f          (src/rss.py:184-206: every party ends
//                                      up with share_a ^ share_b ^ missing)
__global__ void __launch_bounds__(256) flag_shuffle2_kernel(
    int64_t rows, const int32_t* __restrict__ pi23, const int32_t* __restrict__ k3, const uint32_t* __restrict__ x1f,
    const uint32_t* __restrict__ y1f, const uint32_t* __restrict__ wf, const uint32_t* __restrict__ zf,
    const uint32_t* __restrict__ r1f, const uint32_t* __restrict__ r2f, uint32_t* __restrict__ c1f,
    uint32_t* __restrict__ r3f, uint32_t* __restrict__ plain) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < rows; base += stride) {
        const int64_t i = base + lane_id();
        uint32_t bc = 0, br = 0;
        if (i < rows) {
            bc = bit_at(x1f, __ldcs(pi23 + i));
            br = bit_at(y1f, __ldcs(k3 + i));
        }
        const uint32_t wc = __ballot_sync(0xffffffffu, bc), wr = __ballot_sync(0xffffffffu, br);
        if (lane_id() == 0) {
            const int64_t w = base >> 5;
            const uint32_t c = wc ^ __ldg(wf + w);
            const uint32_t r = wr ^ c ^ __ldg(zf + w);
            if (c1f) c1f[w] = c;
            r3f[w] = r;
            if (plain) plain[w] = __ldg(r1f + w) ^ __ldg(r2f + w) ^ r;
        }
    }
}

// ---- the whole fetch shuffle in one cooperative launch (<= 2^21 rows) -------
// ogm_shuffle_online_fused's two phases with the composed flag column of
// ogm_flag_open_composed folded in: phase 1 also XORs P1's two flag
// components, phase 2 -- which walks the rows in output order anyway -- also
// gathers the two composed flag bits per row and writes the new component's
// flag column and the opened column (one ballot per warp).  Two launches fewer
// than the separate shuffle + flag kernels.
struct Fetch4Flags {
    const int32_t *kc, *kr;
    const uint32_t *f1, *f2, *f3, *uwf, *vzf, *r1f, *r2f;
    uint32_t *f12, *r3f, *plain;
};

__global__ void __launch_bounds__(256) fetch128_coop_kernel(const Shuffle4Args p, const Fetch4Flags q) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nw = (p.rows + 31) >> 5;
    for (int64_t w = t0; w < nw; w += stride) q.f12[w] = __ldg(q.f1 + w) ^ __ldg(q.f2 + w);
    for (int64_t i = t0; i < p.rows; i += stride) {
        const int64_t k = __ldg(p.k1 + i), j = __ldg(p.pi12 + i);
        p.x1[i] = xor4(xor4(__ldcg(p.a + k), __ldcg(p.b + k)), __ldcs(p.U + i));
        p.y1[i] = xor4(__ldcg(p.c + j), __ldcs(p.V + i));
    }
    grid.sync();
    const int lane = threadIdx.x & 31;
    for (int64_t base = t0 - lane; base < p.rows; base += stride) {   // warp-uniform: the ballots need every lane
        const int64_t i = base + lane;
        uint32_t bc = 0, br = 0;
        if (i < p.rows) {
            const uint4 c = xor4(__ldcg(p.x1 + __ldg(p.pi23 + i)), __ldcs(p.W + i));
            if (p.c1) p.c1[i] = c;
            p.r3[i] = xor4(xor4(__ldcg(p.y1 + __ldg(p.k3 + i)), c), __ldcs(p.Z + i));
            const int32_t jc = __ldcs(q.kc + i), jr = __ldcs(q.kr + i);
            bc = (__ldcg(q.f12 + (jc >> 5)) >> (jc & 31)) & 1u;   // written above: no read-only path
            br = (__ldg(q.f3 + (jr >> 5)) >> (jr & 31)) & 1u;
        }
        const uint32_t wc = __ballot_sync(0xffffffffu, bc), wr = __ballot_sync(0xffffffffu, br);
        if (lane == 0) {
            const int64_t w = base >> 5;
            const uint32_t cw = wc ^ __ldg(q.uwf + w);
            const uint32_t r = wr ^ cw ^ __ldg(q.vzf + w);
            q.r3f[w] = r;
            q.plain[w] = __ldg(q.r1f + w) ^ __ldg(q.r2f + w) ^ r;
        }
    }
}

// ---- public compaction: keep the rows whose opened bit is set, in order ----
// Three launches, no library: per-chunk popcounts (one warp per chunk of
// 32..256 mask words, sized for >= 4096 chunks so every SM has warps),
// one CTA scanning the chunk counts, then one warp per chunk emitting: it
// loads 32 mask words at once, scans their popcounts in registers, and for
// each word the set lanes write their row index and/or copy their 16-byte
// rows of every matrix to consecutive output slots (coalesced both ways).
constexpr int kKeepMaxMats = 8;

// mask words per chunk: 32..256, a power of two, >= 4096 chunks when the mask allows
inline int64_t keep_chunk_words(int64_t rows) {
    const int64_t nw = (rows + 31) / 32;
    int64_t cw = 256;
    while (cw > 32 && nw / cw < 4096) cw >>= 1;
    return cw;
}
inline int64_t keep_chunks(int64_t rows) {
    const int64_t cw = keep_chunk_words(rows);
    return ((rows + 31) / 32 + cw - 1) / cw;
}

struct KeepMats {
    const uint4* in[kKeepMaxMats];
    uint4* out[kKeepMaxMats];
    int n;
    int64_t pitch;   // in uint4
    int64_t opitch;  // in uint4
};

__device__ __forceinline__ uint32_t mask_word(const uint32_t* __restrict__ bits, int64_t w, int64_t rows) {
    uint32_t v = __ldg(bits + w);
    const int64_t lo = w * 32;
    if (lo + 32 > rows) v &= (rows - lo) >= 32 ? 0xffffffffu : ((1u << (rows - lo)) - 1u);
    return v;
}

__global__ void __launch_bounds__(256) keep_count_kernel(const uint32_t* __restrict__ bits, int64_t rows,
                                                         int64_t nchunks, int64_t chunk_words,
                                                         int32_t* __restrict__ counts) {
    const int64_t nw = (rows + 31) / 32;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; c < nchunks; c += warps) {
        int s = 0;
        const int64_t end = min(nw, (c + 1) * chunk_words);
        for (int64_t w = c * chunk_words + lane_id(); w < end; w += 32) s += __popc(mask_word(bits, w, rows));
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane_id() == 0) counts[c] = s;
    }
}

// exclusive scan of n chunk counts -> offsets[n]; total -> *total (one CTA of 1024)
__global__ void __launch_bounds__(1024) keep_scan_kernel(const int32_t* __restrict__ counts, int64_t n,
                                                         int64_t* __restrict__ offsets, int64_t* __restrict__ total) {
    __shared__ int64_t warp_sum[32];
    const int64_t per = (n + blockDim.x - 1) / blockDim.x;
    const int64_t lo = min(n, (int64_t)threadIdx.x * per), hi = min(n, lo + per);
    int64_t s = 0;
    for (int64_t i = lo; i < hi; i++) s += counts[i];
    int64_t incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if ((int)lane_id() >= o) incl += v;
    }
    if (lane_id() == 31) warp_sum[threadIdx.x / 32] = incl;
    __syncthreads();
    if (threadIdx.x < 32) {
        int64_t v = threadIdx.x < blockDim.x / 32 ? warp_sum[threadIdx.x] : 0;
        int64_t wi = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t u = __shfl_up_sync(0xffffffffu, wi, o);
            if ((int)threadIdx.x >= o) wi += u;
        }
        warp_sum[threadIdx.x] = wi - v;  // exclusive prefix of the warps
        if (threadIdx.x == 31) *total = wi;
    }
    __syncthreads();
    int64_t run = warp_sum[threadIdx.x / 32] + incl - s;
    for (int64_t i = lo; i < hi; i++) {
        offsets[i] = run;
        run += counts[i];
    }
}

// Emit: each warp walks its chunk 32 mask words at a time.  Kept rows are
// queued in a per-warp shared-memory list (position, source row) in order;
// whenever the list could overflow it is flushed with ALL lanes copying one
// queued row each, so a sparse mask (1% kept) still has 32 independent row
// copies in flight per warp instead of one at a time.
constexpr int kKeepQueue = 64;

__global__ void __launch_bounds__(256) keep_emit_kernel(const uint32_t* __restrict__ bits, int64_t rows,
                                                        int64_t nchunks, int64_t chunk_words,
                                                        const int64_t* __restrict__ offsets,
                                                        const __grid_constant__ KeepMats m,
                                                        int32_t* __restrict__ out_idx) {
    __shared__ int64_t q_pos[8][kKeepQueue];
    __shared__ int32_t q_row[8][kKeepQueue];
    const int64_t nw = (rows + 31) / 32;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    const uint32_t lane = lane_id();
    const int wi = threadIdx.x / 32;
    const uint32_t below = (1u << lane) - 1u;
    int queued = 0;
    // one kept row of every matrix: all loads issued before any store (the matrices may not
    // alias, but the compiler cannot know it)
    auto copy_row = [&](int64_t pos, int64_t row) {
        uint4 v[kKeepMaxMats];
#pragma unroll
        for (int j = 0; j < kKeepMaxMats; j++)
            if (j < m.n) v[j] = __ldcs(m.in[j] + row * m.pitch);
#pragma unroll
        for (int j = 0; j < kKeepMaxMats; j++)
            if (j < m.n) __stcs(m.out[j] + pos * m.opitch, v[j]);
    };
    auto flush = [&]() {
        __syncwarp();
        for (int e = (int)lane; e < queued; e += 32) copy_row(q_pos[wi][e], q_row[wi][e]);
        __syncwarp();
        queued = 0;
    };
    for (int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; c < nchunks; c += warps) {
        int64_t base = __ldg(offsets + c);
        const int64_t end = min(nw, (c + 1) * chunk_words);
        for (int64_t wb = c * chunk_words; wb < end; wb += 32) {
            const uint32_t mine = (wb + lane < end) ? mask_word(bits, wb + lane, rows) : 0u;
            const int cnt = __popc(mine);
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if ((int)lane >= o) incl += v;
            }
            const int excl = incl - cnt;
            for (int k = 0; k < 32; k++) {
                const uint32_t word = __shfl_sync(0xffffffffu, mine, k);
                if (!word) continue;
                const int off = __shfl_sync(0xffffffffu, excl, k);
                if (word == 0xffffffffu) {   // 32 kept rows in a row: straight to their consecutive slots
                    const int64_t pos = base + off + lane, row = (wb + k) * 32 + lane;
                    if (out_idx) out_idx[pos] = (int32_t)row;
                    if (m.n) copy_row(pos, row);
                    continue;
                }
                const int n = __popc(word);
                if (m.n && queued + n > kKeepQueue) flush();
                if ((word >> lane) & 1u) {
                    const int r = __popc(word & below);
                    const int64_t pos = base + off + r;
                    const int64_t row = (wb + k) * 32 + lane;
                    if (out_idx) out_idx[pos] = (int32_t)row;
                    if (m.n) {
                        q_pos[wi][queued + r] = pos;
                        q_row[wi][queued + r] = (int32_t)row;
                    }
                }
                queued += m.n ? n : 0;
            }
            base += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
    if (m.n) flush();
}

}  // namespace ogm

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int ogm_split_flag_rows(int64_t rows, const uint32_t* in, int64_t pitch, uint32_t* payload, uint32_t* flags,
                        void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(rows >= 0 && pitch >= 5, OGM_ERR_ARG, "split needs rows of at least 5 words (129 bits)");
    OGM_CHECK_ARG(rows == 0 || (in && payload && flags), OGM_ERR_ARG, "in, payload and flags are required");
    OGM_CHECK_ARG((((uintptr_t)payload) & 15) == 0, OGM_ERR_ARG, "16-byte aligned payload rows are required");
    if (rows == 0) return OGM_OK;
    split_flag_rows_kernel<<<grid_for(rows), 256, 0, as_stream(stream)>>>(in, pitch, rows, (uint4*)payload, flags);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

int ogm_flag_shuffle_trio(int64_t rows, const int32_t* k1, const int32_t* pi12, const int32_t* pi23,
                          const int32_t* k3, const uint32_t* f1, const uint32_t* f2, const uint32_t* f3,
                          const uint32_t* uf, const uint32_t* vf, const uint32_t* wf, const uint32_t* zf,
                          const uint32_t* r1f, const uint32_t* r2f, uint32_t* x1f, uint32_t* y1f, uint32_t* c1f,
                          uint32_t* r3f, uint32_t* plain, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(rows >= 0 && rows < ((int64_t)1 << 31), OGM_ERR_ARG, "rows out of range");
    if (rows == 0) return OGM_OK;
    const void* need[] = {k1, pi12, pi23, k3, f1, f2, f3, uf, vf, wf, zf, x1f, y1f, r3f};
    for (const void* p : need) OGM_CHECK_ARG(p, OGM_ERR_ARG, "permutations, flag columns, blinds and x1f/y1f/r3f "
                                                           "scratch are required");
    OGM_CHECK_ARG(!plain || (r1f && r2f), OGM_ERR_ARG, "the opened column needs R1f and R2f");
    cudaStream_t st = as_stream(stream);
    const int g = grid_for(rows);
    const int64_t nw = (rows + 31) / 32;
    // P1's f1 ^ f2 is staged in r3f's words: phase 1 reads it, only phase 2 writes r3f
    uint32_t* f12 = r3f;
    flag_xor2_kernel<<<grid_for(nw), 256, 0, st>>>(f1, f2, nw, f12);
    flag_shuffle1_kernel<<<g, 256, 0, st>>>(rows, k1, pi12, f12, f3, uf, vf, x1f, y1f);
    flag_shuffle2_kernel<<<g, 256, 0, st>>>(rows, pi23, k3, x1f, y1f, wf, zf, r1f, r2f, c1f, r3f, plain);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

// The flag column of the co-resident trio with each party's step composed
// with the next one's, as the payload's flat hand-over composes them: the
// message bits x1f / y1f exist only in flight (each read once, where the
// receiver's step needs it), so the column costs two random bit reads per
// row instead of four:
//   c1f[i] = f12[kc[i]] ^ uwf[i],  kc = k1 o pi23, uwf[i] = Uf[pi23[i]] ^ Wf[i]
//   r3f[i] = f3[kr[i]] ^ vzf[i] ^ c1f[i],  kr = pi12 o k3, vzf[i] = Vf[k3[i]] ^ Zf[i]
// (offline compositions; phase 2's kernel computes exactly this given them).
int ogm_flag_open_composed(int64_t rows, const int32_t* kc, const int32_t* kr, const uint32_t* f1,
                           const uint32_t* f2, const uint32_t* f3, const uint32_t* uwf, const uint32_t* vzf,
                           const uint32_t* r1f, const uint32_t* r2f, uint32_t* f12, uint32_t* c1f, uint32_t* r3f,
                           uint32_t* plain, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(rows >= 0 && rows < ((int64_t)1 << 31), OGM_ERR_ARG, "rows out of range");
    if (rows == 0) return OGM_OK;
    const void* need[] = {kc, kr, f1, f2, f3, uwf, vzf, f12, r3f};
    for (const void* p : need)
        OGM_CHECK_ARG(p, OGM_ERR_ARG, "composed indices, flag columns, blinds and f12/r3f scratch are required");
    OGM_CHECK_ARG(!plain || (r1f && r2f), OGM_ERR_ARG, "the opened column needs R1f and R2f");
    cudaStream_t st = as_stream(stream);
    const int64_t nw = (rows + 31) / 32;
    flag_xor2_kernel<<<grid_for(nw), 256, 0, st>>>(f1, f2, nw, f12);
    flag_shuffle2_kernel<<<grid_for(rows), 256, 0, st>>>(rows, kc, kr, f12, f3, uwf, vzf, r1f, r2f, c1f, r3f, plain);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

// The whole online fetch shuffle of flag-split rows (>= 2^22 rows) in one
// call: f12 = f1 ^ f2, then the chained planned payload shuffle whose final
// window passes also compute the flag column -- composed as in
// ogm_flag_open_composed, so each pass makes one random bit read per row --
// and the opened column (FlagTail; they walk the rows in output order
// anyway).  Arguments as ogm_shuffle_online_planned_slots (qs: the composed
// indices, may be null for the staged hand-over; run_*: the plans' run
// tables, or null) and ogm_flag_open_composed; c1f is scratch when the
// passes are split (> 256 MB).
int ogm_fetch128_online_planned(int64_t rows, const int32_t* const* q2, const int32_t* const* gdst,
                                const uint16_t* const* srow, const int32_t* const* qs,
                                const uint16_t* const* run_start, const int32_t* const* run_off,
                                const int64_t* run_nwin, const int64_t* wrows, const uint32_t* a, const uint32_t* b,
                                const uint32_t* c, const uint32_t* u_src, const uint32_t* v_src,
                                const uint32_t* w_blind, int w_order, const uint32_t* z_slot, int z_order,
                                uint32_t* const* inter, uint32_t* r3, const int32_t* kc, const int32_t* kr,
                                const uint32_t* f1, const uint32_t* f2, const uint32_t* f3, const uint32_t* uwf,
                                const uint32_t* vzf, const uint32_t* r1f, const uint32_t* r2f, uint32_t* f12,
                                uint32_t* c1f, uint32_t* r3f, uint32_t* plain, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(rows >= 0 && rows < ((int64_t)1 << 31), OGM_ERR_ARG, "rows out of range");
    if (rows == 0) return OGM_OK;
    const void* need[] = {kc, kr, f1, f2, f3, uwf, vzf, r1f, r2f, f12, c1f, r3f, plain};
    for (const void* p : need)
        OGM_CHECK_ARG(p, OGM_ERR_ARG, "composed indices, flag columns, blinds and scratch are required");
    cudaStream_t st = as_stream(stream);
    const int64_t nw = (rows + 31) / 32;
    flag_xor2_kernel<<<grid_for(nw), 256, 0, st>>>(f1, f2, nw, f12);
    OGM_LAUNCH_CHECK();
    const FlagTail ft{kc, kr, f12, f3, uwf, vzf, r1f, r2f, c1f, r3f, plain};
    RunTable rt[4];
    const bool runs = run_tables(run_start, run_off, run_nwin, rt);
    return shuffle_online_planned_impl(rows, q2, gdst, srow, a, b, c, u_src, v_src, 0, w_blind, w_order, z_slot,
                                       z_order, inter, nullptr, nullptr, nullptr, r3, &ft, qs, runs ? rt : nullptr,
                                       wrows, stream);
}

// One cooperative launch: the shuffle of ogm_shuffle_online_fused (x1 / y1
// scratch tables, R3 out) and the composed flag column of
// ogm_flag_open_composed (f12 scratch; r3f and the opened column out).
int ogm_fetch128_online_fused(int64_t rows, const int32_t* k1, const int32_t* pi12, const int32_t* pi23,
                              const int32_t* k3, const uint32_t* a, const uint32_t* b, const uint32_t* c,
                              const uint32_t* U, const uint32_t* V, const uint32_t* W, const uint32_t* Z,
                              uint32_t* x1, uint32_t* y1, uint32_t* r3, const int32_t* kc, const int32_t* kr,
                              const uint32_t* f1, const uint32_t* f2, const uint32_t* f3, const uint32_t* uwf,
                              const uint32_t* vzf, const uint32_t* r1f, const uint32_t* r2f, uint32_t* f12,
                              uint32_t* r3f, uint32_t* plain, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(rows >= 0 && rows < ((int64_t)1 << 31), OGM_ERR_ARG, "rows out of range");
    const void* ptrs[] = {a, b, c, U, V, W, Z, x1, y1, r3};
    for (const void* q : ptrs)
        OGM_CHECK_ARG(q && (((uintptr_t)q) & 15) == 0, OGM_ERR_ARG, "16-byte aligned tables are required");
    const void* need[] = {k1, pi12, pi23, k3, kc, kr, f1, f2, f3, uwf, vzf, r1f, r2f, f12, r3f, plain};
    for (const void* q : need)
        OGM_CHECK_ARG(q, OGM_ERR_ARG, "permutations, composed indices, flag columns and scratch are required");
    if (rows == 0) return OGM_OK;
    OGM_ENSURE_INIT();
    Shuffle4Args p{k1, pi12, pi23, k3, (const uint4*)a, (const uint4*)b, (const uint4*)c, (const uint4*)U,
                   (const uint4*)V, (const uint4*)W, (const uint4*)Z, (uint4*)x1, (uint4*)y1, nullptr,
                   (uint4*)r3, rows};
    Fetch4Flags q{kc, kr, f1, f2, f3, uwf, vzf, r1f, r2f, f12, r3f, plain};
    int per_sm = 0;
    OGM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fetch128_coop_kernel, 256, 0));
    int64_t g = (int64_t)sm_count() * std::max(per_sm, 1);
    const int64_t need_g = (rows + 255) / 256;
    if (g > need_g) g = need_g;
    void* args[] = {&p, &q};
    OGM_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)fetch128_coop_kernel, dim3((unsigned)g), dim3(256), args, 0,
                                             as_stream(stream)));
    return OGM_OK;
}

int64_t ogm_keep_rows_workspace_bytes(int64_t rows) {
    const int64_t nc = ((rows > 0 ? rows : 1) + 1023) / 1024;  // chunks of the smallest size (32 words)
    return ((nc * 4 + 255) & ~(int64_t)255) + nc * 8 + 256;
}

int ogm_keep_rows(int64_t rows, const uint32_t* bits, int nmat, const uint32_t* const* mats, int64_t pitch,
                  uint32_t* const* outs, int64_t opitch, int32_t* out_idx, int64_t* count, void* workspace,
                  int64_t workspace_bytes, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(rows >= 0 && rows < ((int64_t)1 << 31), OGM_ERR_ARG, "rows out of range");
    OGM_CHECK_ARG(nmat >= 0 && nmat <= kKeepMaxMats, OGM_ERR_ARG, "at most %d matrices", kKeepMaxMats);
    OGM_CHECK_ARG(count, OGM_ERR_ARG, "count (device int64) is required");
    OGM_CHECK_ARG(workspace_bytes >= ogm_keep_rows_workspace_bytes(rows), OGM_ERR_ARG, "keep workspace too small");
    KeepMats m{};
    m.n = nmat;
    if (nmat) {
        OGM_CHECK_ARG(pitch > 0 && pitch % 4 == 0 && opitch > 0 && opitch % 4 == 0, OGM_ERR_ARG,
                      "row copies need 16-byte row pitches");
        m.pitch = pitch / 4;
        m.opitch = opitch / 4;
        for (int j = 0; j < nmat; j++) {
            OGM_CHECK_ARG(mats[j] && outs[j] && ((((uintptr_t)mats[j]) | ((uintptr_t)outs[j])) & 15) == 0,
                          OGM_ERR_ARG, "matrix %d: 16-byte aligned rows are required", j);
            m.in[j] = (const uint4*)mats[j];
            m.out[j] = (uint4*)outs[j];
        }
    }
    cudaStream_t st = as_stream(stream);
    if (rows == 0) {
        OGM_CUDA_TRY(cudaMemsetAsync(count, 0, 8, st));
        return OGM_OK;
    }
    OGM_CHECK_ARG(bits, OGM_ERR_ARG, "mask bits are required");
    const int64_t nc = keep_chunks(rows), cw = keep_chunk_words(rows);
    int32_t* counts = (int32_t*)workspace;
    int64_t* offsets = (int64_t*)((uint8_t*)workspace + ((nc * 4 + 255) & ~(int64_t)255));
    const int g = (int)std::min<int64_t>((nc + 7) / 8, (int64_t)sm_count() * 8);
    keep_count_kernel<<<g, 256, 0, st>>>(bits, rows, nc, cw, counts);
    keep_scan_kernel<<<1, 1024, 0, st>>>(counts, nc, offsets, count);
    keep_emit_kernel<<<g, 256, 0, st>>>(bits, rows, nc, cw, offsets, m, out_idx);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

}  // extern "C"
