// ogm_fss.cuh -- PRG/PRF and FSS kernels (src/prf.py, src/fss.py) for sm_100a.
//
// All kernels here are integer-ALU / shared-memory-lookup bound (no tensor
// cores, no floating point).  Grids are sized to one 128 KiB-table CTA per SM
// (148 on B200) and loop over work, so the table fill is paid once per SM.
#pragma once

#include "ogm_aes.cuh"
#include "ogm_common.cuh"
#include "ogm_host.cuh"

namespace ogm {

constexpr int kFssThreads = kAesThreads;

#define OGM_AES_PROLOGUE_T(TABT)                        \
    extern __shared__ __align__(128) uint8_t smem_raw[]; \
    TABT::fill(smem_raw);                               \
    __syncthreads();                                    \
    const TABT T(smem_raw)
#define OGM_AES_PROLOGUE() OGM_AES_PROLOGUE_T(AesTab)

// ---------------------------------------------------------------------------
// src/prf.py:41-57 prg_expand: one thread per seed, 2 full AES + ctrl AES.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kFssThreads) prg_expand_kernel(
    const uint4* __restrict__ seeds, int64_t n, uint4* __restrict__ left, uint4* __restrict__ right,
    uint8_t* __restrict__ tl, uint8_t* __restrict__ tr, uint8_t* __restrict__ val) {
    OGM_AES_PROLOGUE();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        uint4 s = seeds[i];
        uint32_t c = prg_ctrl_bits(T, s);
        left[i] = prg_child(T, s, PrgKey<0>());
        right[i] = prg_child(T, s, PrgKey<1>());
        tl[i] = c & 1;
        tr[i] = (c >> 1) & 1;
        val[i] = (c >> 2) & 1;
    }
}

// ---------------------------------------------------------------------------
// src/fss.py:116-157 _tree_gen, one thread per key pair (6 AES per level:
// both children + control for both parties' seeds).
// ---------------------------------------------------------------------------
template <bool DCF, class TAB = AesTab>
__global__ void __launch_bounds__(kFssThreads) fss_gen_kernel(
    int bits, int64_t K, const uint32_t* __restrict__ alphas, const uint4* __restrict__ roots0,
    const uint4* __restrict__ roots1, uint4* __restrict__ scw_out, uint32_t* __restrict__ ctrl_out,
    uint8_t* __restrict__ final_out, uint8_t* __restrict__ flags1_out) {
    OGM_AES_PROLOGUE_T(TAB);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < K; k += stride) {
        uint4 s0 = roots0[k], s1 = roots1[k];
        uint32_t t0 = 0, t1 = 1;
        uint32_t a = alphas[k] << (32 - bits);
        uint32_t tlw = 0, trw = 0, vw = 0;
        for (int lvl = 0; lvl < bits; lvl++) {
            const uint32_t ab = a >> 31;
            a <<= 1;
            const uint32_t c0 = prg_ctrl_bits(T, s0), c1 = prg_ctrl_bits(T, s1);
            const uint4 L0 = prg_child(T, s0, PrgKey<0>()), R0 = prg_child(T, s0, PrgKey<1>());
            const uint4 L1 = prg_child(T, s1, PrgKey<0>()), R1 = prg_child(T, s1, PrgKey<1>());
            const uint32_t cx = c0 ^ c1;
            const uint32_t v_cw = ((cx >> 2) & 1) ^ (DCF ? ab : 0u);
            const uint4 s_cw = ab ? xor4(L0, L1) : xor4(R0, R1);          // lose-side XOR
            const uint32_t tau_l = (cx & 1) ^ ab ^ 1u;
            const uint32_t tau_r = ((cx >> 1) & 1) ^ ab;
            scw_out[(int64_t)lvl * K + k] = s_cw;
            tlw |= tau_l << lvl;
            trw |= tau_r << lvl;
            vw |= v_cw << lvl;
            const uint32_t tau_keep = ab ? tau_r : tau_l;
            const uint4 keep0 = ab ? R0 : L0, keep1 = ab ? R1 : L1;
            const uint32_t kt0 = (c0 >> ab) & 1, kt1 = (c1 >> ab) & 1;
            s0 = xor4(keep0, and4(s_cw, 0u - t0));
            s1 = xor4(keep1, and4(s_cw, 0u - t1));
            t0 = kt0 ^ (t0 & tau_keep);
            t1 = kt1 ^ (t1 & tau_keep);
        }
        ctrl_out[k] = tlw;
        ctrl_out[K + k] = trw;
        ctrl_out[2 * K + k] = vw;
        const uint8_t fin = DCF ? 0 : (uint8_t)((((s0.x ^ s1.x) & 1u)) ^ 1u);
        if (flags1_out) {   // the eval kernels' flag bytes (bit 0 root_t, bit 1 final_cw) of both parties
            final_out[k] = (uint8_t)(fin << 1);
            flags1_out[k] = (uint8_t)((fin << 1) | 1u);
        } else {
            final_out[k] = fin;
        }
    }
}

// ---------------------------------------------------------------------------
// src/fss.py:257-281 _walk_eval: one thread per (key, point), 2 AES per level
// (the taken child under a per-lane left/right key, plus the truncated
// control AES).  A DCF never needs the last level's child seed.  Warps cover
// 32 consecutive keys so the result word is one ballot.
// ---------------------------------------------------------------------------
template <bool DCF>
__global__ void __launch_bounds__(kFssThreads) fss_eval_kernel(
    int bits, int64_t K, const uint4* __restrict__ root, const uint4* __restrict__ scw,
    const uint32_t* __restrict__ ctrl, const uint8_t* __restrict__ flags,
    const uint32_t* __restrict__ points, uint32_t* __restrict__ out) {
    OGM_AES_PROLOGUE();
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t nchunks = (K + 31) >> 5;
    for (int64_t chunk = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); chunk < nchunks;
         chunk += warps) {
        const int64_t k = (chunk << 5) + lane;
        uint32_t bit = 0;
        if (k < K) {
            uint4 s = root[k];
            const uint32_t f = flags[k];
            uint32_t t = f & 1u;
            uint32_t x = points[k] << (32 - bits);
            const uint32_t tlw = ctrl[k], trw = ctrl[K + k], vw = ctrl[2 * K + k];
            uint32_t acc = 0;
            const uint4* cwp = scw + k;
            for (int lvl = 0; lvl < bits; lvl++, cwp += K) {
                const uint32_t xb = x >> 31;
                x <<= 1;
                const bool need_child = !DCF || lvl + 1 < bits;
                uint4 cw = make_uint4(0, 0, 0, 0);
                if (need_child) cw = __ldg(cwp);
                const uint32_t c = prg_ctrl_bits(T, s);
                if (DCF) acc ^= (xb ^ 1u) & ((c >> 2) ^ (t & (vw >> lvl))) & 1u;
                if (need_child) {
                    const uint4 child = prg_child(T, s, PrgChildKey{0u - xb});
                    const uint32_t tm = 0u - t;
                    s = xor4(child, and4(cw, tm));
                    t = ((c >> xb) & 1u) ^ (t & ((xb ? trw : tlw) >> lvl) & 1u);
                }
            }
            bit = DCF ? acc : ((s.x & 1u) ^ (t & (f >> 1) & 1u));
            bit ^= (f >> 2) & 1u;
        }
        const uint32_t word = __ballot_sync(0xffffffffu, bit);
        if (lane == 0) out[chunk] = word;
    }
}

// ---------------------------------------------------------------------------
// src/fss.py:302-344 _full_domain_tree.  Thread (key, word, sub) owns a
// subtree of L = 2^kk leaves: it walks from the root to the subtree root (2
// AES per level) and expands the subtree depth-first (3 AES per internal node,
// 1 for a DCF's last internal level).  G = 32/L lanes OR their bits into one
// output word.  Leaves >= n are zero, add_const is folded in (src/fss.py:336).
// ---------------------------------------------------------------------------
struct FdeNode {
    uint4 s;
    uint32_t t, acc, idx, rd;
};

template <bool DCF, class TAB = AesTab>
__global__ void __launch_bounds__(kFssThreads) fss_fde_kernel(
    int bits, int nkeys, const uint4* __restrict__ root, const uint4* __restrict__ scw,
    const uint32_t* __restrict__ ctrl, const uint8_t* __restrict__ flags, int64_t n, int kk,
    uint32_t* __restrict__ out, int64_t pitch) {
    OGM_AES_PROLOGUE_T(TAB);
    const int lane = threadIdx.x & 31;
    const int L = 1 << kk;
    const int G = 32 / L;
    const int64_t words = (n + 31) >> 5;
    const int64_t slots = (int64_t)nkeys * words * G;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t nwt = (slots + 31) >> 5;
    const int d = bits - kk;
    for (int64_t wt = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); wt < nwt; wt += warps) {
        const int64_t slot = (wt << 5) + lane;
        uint32_t mybits = 0;
        int key = 0, sub = 0;
        int64_t word = 0;
        const bool active = slot < slots;
        if (active) {
            sub = (int)(slot % G);
            word = (slot / G) % words;
            key = (int)(slot / G / words);
        }
        const uint64_t base = (uint64_t)word * 32 + (uint64_t)sub * L;
        if (active && base < (uint64_t)n) {
            const uint32_t f = flags[key];
            const uint32_t tlw = ctrl[key], trw = ctrl[nkeys + key], vw = ctrl[2 * nkeys + key];
            uint4 s = root[key];
            uint32_t t = f & 1u, acc = 0;
            const uint64_t sidx = base >> kk;  // subtree index at depth d
            // walk to the subtree root (same step as the pointwise walk)
            for (int lvl = 0; lvl < d; lvl++) {
                const uint32_t xb = (uint32_t)(sidx >> (d - 1 - lvl)) & 1u;
                const uint4 cw = __ldg(scw + (int64_t)lvl * nkeys + key);
                const uint32_t c = prg_ctrl_bits(T, s);
                if (DCF) acc ^= (xb ^ 1u) & ((c >> 2) ^ (t & (vw >> lvl))) & 1u;
                const uint4 child = prg_child(T, s, PrgChildKey{0u - xb});
                s = xor4(child, and4(cw, 0u - t));
                t = ((c >> xb) & 1u) ^ (t & ((xb ? trw : tlw) >> lvl) & 1u);
            }
            // depth-first expansion; leaves come out in natural order
            FdeNode stack[6];
            int sp = 0;
            FdeNode cur{s, t, acc, 0u, 0u};
            while (true) {
                if ((int)cur.rd == kk) {
                    const uint32_t b = DCF ? cur.acc : ((cur.s.x & 1u) ^ (cur.t & (f >> 1)));
                    mybits |= (b & 1u) << cur.idx;
                    if (sp == 0) break;
                    cur = stack[--sp];
                    continue;
                }
                const int lvl = d + (int)cur.rd;
                const uint32_t c = prg_ctrl_bits(T, cur.s);
                FdeNode lc, rc;
                lc.t = (c & 1u) ^ (cur.t & (tlw >> lvl) & 1u);
                rc.t = ((c >> 1) & 1u) ^ (cur.t & (trw >> lvl) & 1u);
                lc.acc = cur.acc ^ (((c >> 2) ^ (cur.t & (vw >> lvl))) & 1u);
                rc.acc = cur.acc;
                if (!DCF || (int)cur.rd + 1 < kk) {
                    const uint4 cw = and4(__ldg(scw + (int64_t)lvl * nkeys + key), 0u - cur.t);
                    lc.s = xor4(prg_child(T, cur.s, PrgKey<0>()), cw);
                    rc.s = xor4(prg_child(T, cur.s, PrgKey<1>()), cw);
                } else {
                    lc.s = rc.s = make_uint4(0, 0, 0, 0);
                }
                lc.idx = cur.idx * 2;
                rc.idx = cur.idx * 2 + 1;
                lc.rd = rc.rd = cur.rd + 1;
                stack[sp++] = rc;
                cur = lc;
            }
            const uint32_t lmask = (L == 32) ? 0xffffffffu : ((1u << L) - 1u);
            if ((f >> 2) & 1u) mybits ^= lmask;
            const uint64_t valid = (uint64_t)n - base;  // > 0
            if (valid < (uint64_t)L) mybits &= (1u << valid) - 1u;
        }
        // OR the G lanes of one word together (groups are G-aligned)
        uint32_t w = (L == 32) ? mybits : (mybits << (sub * L));
        for (int off = G >> 1; off > 0; off >>= 1) w |= __shfl_xor_sync(0xffffffffu, w, off);
        if (active && sub == 0) out[(int64_t)key * pitch + word] = w;
    }
}

// ---------------------------------------------------------------------------
// src/prf.py:70-92 prf_stream as words: one thread per 16-byte CTR block.
// src/rss.py:143-148 zero shares: two keys, XOR, tail mask, optional fold.
// ---------------------------------------------------------------------------
template <bool ZERO, class TAB = AesTab>
__global__ void __launch_bounds__(kFssThreads) prf_words_kernel(
    const __grid_constant__ AesKeySched k1, const __grid_constant__ AesKeySched k2, uint32_t label_be, uint64_t index, uint64_t first_word,
    int64_t nwords, int64_t nbits, const uint32_t* __restrict__ xor_into, uint32_t* __restrict__ out) {
    OGM_AES_PROLOGUE_T(TAB);
    const uint64_t b0 = first_word >> 2;
    const uint64_t b1 = (first_word + (uint64_t)nwords + 3) >> 2;
    const int64_t nblk = (int64_t)(b1 - b0);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nblk; i += stride) {
        const uint64_t blk = b0 + (uint64_t)i;
        const uint4 ctr = ctr_block(label_be, index, blk);
        uint4 ks = aes128_enc(T, ctr, ParamKey{k1.rk});
        if (ZERO) ks = xor4(ks, aes128_enc(T, ctr, ParamKey{k2.rk}));
        const uint32_t kw[4] = {ks.x, ks.y, ks.z, ks.w};
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int64_t o = (int64_t)(blk * 4 + j) - (int64_t)first_word;
            if (o < 0 || o >= nwords) continue;
            uint32_t v = kw[j];
            if (ZERO) {
                // BitVector(additive ^ share, n) semantics: tail masked after the fold
                if (xor_into) v ^= xor_into[o];
                if ((nbits & 31) && (int64_t)(blk * 4 + j) == ((nbits + 31) >> 5) - 1) v &= (1u << (nbits & 31)) - 1u;
            }
            out[o] = v;
        }
    }
}

// ---------------------------------------------------------------------------
// src/shuffle.py:69-73 blinding table as pitched rows: row r = PRF stream
// words [r*W, r*W + W) of (key, label, index), tail masked to the logical
// width, stored at `pitch` >= W words with zero padding.  One thread per
// 16-byte CTR block whatever W's alignment, so the AES rate is the bound
// (generating such rows inside a 4-word-chunked gather costs up to two AES
// blocks per chunk when W is not a multiple of 4).
// ---------------------------------------------------------------------------
template <class TAB = AesTab>
__global__ void __launch_bounds__(kFssThreads) prf_rows_kernel(const __grid_constant__ AesKeySched k, uint32_t label_be, uint64_t index,
                                                               int64_t rows, int64_t W, uint32_t tail,
                                                               int64_t pitch, uint32_t* __restrict__ out) {
    OGM_AES_PROLOGUE_T(TAB);
    const int64_t nblk = (rows * W + 3) >> 2;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t blk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; blk < nblk; blk += stride) {
        const uint4 ks = aes128_enc(T, ctr_block(label_be, index, (uint64_t)blk), ParamKey{k.rk});
        const uint32_t kw[4] = {ks.x, ks.y, ks.z, ks.w};
        int64_t r = (blk * 4) / W;
        int64_t col = blk * 4 - r * W;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            if (r < rows) {
                uint32_t* row = out + r * pitch;
                if (col == W - 1) {
                    row[col] = kw[j] & tail;
                    for (int64_t p = W; p < pitch; p++) row[p] = 0;
                } else {
                    row[col] = kw[j];
                }
            }
            if (++col == W) {
                col = 0;
                r++;
            }
        }
    }
}

int fss_init() {
    OGM_CUDA_TRY(allow_big_smem(prg_expand_kernel, kAesTableBytes));
    OGM_CUDA_TRY(allow_big_smem(fss_gen_kernel<false, AesTab>, kAesTableBytes));
    OGM_CUDA_TRY(allow_big_smem(fss_gen_kernel<true, AesTab>, kAesTableBytes));
    OGM_CUDA_TRY(allow_big_smem(fss_eval_kernel<false>, kAesTableBytes));
    OGM_CUDA_TRY(allow_big_smem(fss_eval_kernel<true>, kAesTableBytes));
    OGM_CUDA_TRY(allow_big_smem(fss_fde_kernel<false, AesTab>, kAesTableBytes));
    OGM_CUDA_TRY(allow_big_smem(fss_fde_kernel<true, AesTab>, kAesTableBytes));
    OGM_CUDA_TRY(allow_big_smem(prf_words_kernel<false, AesTab>, kAesTableBytes));
    OGM_CUDA_TRY(allow_big_smem(prf_words_kernel<true, AesTab>, kAesTableBytes));
    OGM_CUDA_TRY(allow_big_smem(prf_rows_kernel<AesTab>, kAesTableBytes));
    return OGM_OK;
}

}  // namespace ogm
