// ogm_engine.cuh -- secEval / combine / fetch / access kernels for sm_100a
// (src/engine.py, src/rss.py).  These are HBM-bound streaming kernels over
// row-major (rows, pitch) uint32 share matrices; no tensor cores, no FP.
//
// Party mapping: with the three logical servers co-resident on one GPU, each
// share component x_j is stored once; party q holds (x_q, x_{q+1})
// (src/graphs.py:382-399).  Kernels take component pointers plus per-party
// component indices, so a "trio" launch reads every component once for all
// three parties while a per-party launch (the drop-in path, one CUDA stream
// per party thread) reads only its own two.
#pragma once


#include "ogm_aes.cuh"
#include "ogm_common.cuh"
#include "ogm_host.cuh"

namespace ogm {

constexpr int kMaxComp = 3;
constexpr int kMaxParty = 3;
constexpr int kMaxPass = 2;

// ---------------------------------------------------------------------------
// src/engine.py:76-80 + :162 (interval passes :147-164): per candidate row c,
// additive bit = parity((A[c] & IA) ^ (B[c] & IB)) for every (pass, party).
// G lanes cooperate on a row (G chosen on the host from the row length), a
// warp owns 32 consecutive rows so every output word is assembled from
// ballots.  Indicator vectors are re-read through L1 (__ldg), share rows are
// streamed once from HBM with 128-bit loads when aligned.
// ---------------------------------------------------------------------------
struct ParityArgs {
    const uint32_t* comp[kMaxComp];
    const uint32_t* ind[kMaxPass * kMaxParty * 2];
    uint32_t* out[kMaxPass * kMaxParty];
    int a_idx[kMaxParty], b_idx[kMaxParty];
    int ncomp, nparty, npass, G;
    int acc;  // XOR the parities into out (caller-initialised) instead of overwriting it
    int64_t rows, words, pitch;
};

template <bool VEC4, int NPARTY, int NPASS>
__global__ void __launch_bounds__(256) masked_parity_kernel(const ParityArgs p) {
    constexpr int NJ = NPARTY * NPASS;
    constexpr int NCOMP = NPARTY == 1 ? 2 : 3;  // per party: (A, B); trio: x1, x2, x3
    const int lane = threadIdx.x & 31;
    const int G = p.G;
    const int rows_per_pass = 32 / G;
    const int sub = lane % G;
    const int64_t tiles = (p.rows + 31) >> 5;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t nvec = VEC4 ? (p.words >> 2) : 0;
    const int64_t tail0 = nvec << 2;
    for (int64_t tile = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); tile < tiles;
         tile += warps) {
        uint32_t outw[NJ];
#pragma unroll
        for (int j = 0; j < NJ; j++) outw[j] = 0;
        for (int ps = 0; ps < G; ps++) {
            const int64_t row = (tile << 5) + ps * rows_per_pass + lane / G;
            uint32_t acc[NJ];
#pragma unroll
            for (int j = 0; j < NJ; j++) acc[j] = 0;
            if (row < p.rows) {
                const uint32_t* rp[NCOMP];
#pragma unroll
                for (int c = 0; c < NCOMP; c++) rp[c] = p.comp[c] + row * p.pitch;
                if (VEC4) {
                    for (int64_t u = sub; u < nvec; u += G) {
                        uint4 cv[NCOMP];
#pragma unroll
                        for (int c = 0; c < NCOMP; c++) cv[c] = __ldcs(reinterpret_cast<const uint4*>(rp[c]) + u);
#pragma unroll
                        for (int ps2 = 0; ps2 < NPASS; ps2++) {
#pragma unroll
                            for (int q = 0; q < NPARTY; q++) {
                                const int j = ps2 * NPARTY + q;
                                const uint4 ia = __ldg(reinterpret_cast<const uint4*>(p.ind[2 * j]) + u);
                                const uint4 ib = __ldg(reinterpret_cast<const uint4*>(p.ind[2 * j + 1]) + u);
                                const uint4 A = cv[q], B = cv[(q + 1) % NCOMP];
                                acc[j] ^= ((A.x & ia.x) ^ (B.x & ib.x)) ^ ((A.y & ia.y) ^ (B.y & ib.y)) ^
                                          ((A.z & ia.z) ^ (B.z & ib.z)) ^ ((A.w & ia.w) ^ (B.w & ib.w));
                            }
                        }
                    }
                }
                for (int64_t w = tail0 + sub; w < p.words; w += G) {
                    uint32_t cv[NCOMP];
#pragma unroll
                    for (int c = 0; c < NCOMP; c++) cv[c] = __ldcs(rp[c] + w);
#pragma unroll
                    for (int ps2 = 0; ps2 < NPASS; ps2++) {
#pragma unroll
                        for (int q = 0; q < NPARTY; q++) {
                            const int j = ps2 * NPARTY + q;
                            acc[j] ^= (cv[q] & __ldg(p.ind[2 * j] + w)) ^
                                      (cv[(q + 1) % NCOMP] & __ldg(p.ind[2 * j + 1] + w));
                        }
                    }
                }
            }
            // XOR-reduce each row's G lanes (aligned groups), then ballot.
#pragma unroll
            for (int j = 0; j < NJ; j++) {
                uint32_t a = acc[j];
                for (int off = G >> 1; off > 0; off >>= 1) a ^= __shfl_xor_sync(0xffffffffu, a, off);
                const bool leader = sub == 0 && row < p.rows;
                const uint32_t b = __ballot_sync(0xffffffffu, leader && (__popc(a) & 1));
                if (G == 1) {
                    outw[j] = b;
                } else {
                    uint32_t packed = 0;
                    for (int g = 0; g < rows_per_pass; g++) packed |= ((b >> (g * G)) & 1u) << g;
                    outw[j] |= packed << (ps * rows_per_pass);
                }
            }
        }
        if (lane == 0) {
#pragma unroll
            for (int j = 0; j < NJ; j++) p.out[j][tile] = p.acc ? p.out[j][tile] ^ outw[j] : outw[j];
        }
    }
}


// ---------------------------------------------------------------------------
// Masked parity, register-resident indicators (the bandwidth path).
//
// The indicator vectors are identical for every candidate row, so a CTA owns
// a chunk of columns and keeps its slice of all 2*NPARTY*NPASS indicators in
// registers (one uint4 per vector per lane); warps then stream rows through
// it.  For each row a lane folds its 4 words into a 32-bit partial per
// (pass, party).  Trio: each lane shifts popc(partial) & 1 into a per-(pass,
// party) word, one bit per row, and after 32 rows one butterfly XOR over the
// lanes gives the warp's 128-column partial parities of the tile (an output
// word); per party the row's parity is popc(ballot(popc(partial) & 1)) & 1.
// The word is XORed into the (pre-zeroed) result -- parity is XOR-linear, so column
// chunks and warps combine with atomicXor.  Shares are read exactly once,
// with 128-bit loads, and the indicator traffic is paid once per CTA.
// ---------------------------------------------------------------------------
template <int NPARTY, int NPASS>
__global__ void __launch_bounds__(256, 2) masked_parity_v2_kernel(const ParityArgs p, int CW, int64_t tiles_per_block) {
    constexpr int NJ = NPARTY * NPASS;
    constexpr int NCOMP = NPARTY == 1 ? 2 : 3;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int RG = (int)(blockDim.x >> 5) / CW;  // row groups per CTA (CW need not be a power of 2)
    const int rg = warp / CW, wc = warp % CW;
    const int64_t col0 = ((int64_t)blockIdx.x * CW + wc) * 128 + lane * 4;  // first word of this lane
    uint4 ia[NJ], ib[NJ];
#pragma unroll
    for (int j = 0; j < NJ; j++) {
        uint32_t a4[4], b4[4];
#pragma unroll
        for (int e = 0; e < 4; e++) {
            const bool in = col0 + e < p.words;
            a4[e] = in ? __ldg(p.ind[2 * j] + col0 + e) : 0u;
            b4[e] = in ? __ldg(p.ind[2 * j + 1] + col0 + e) : 0u;
        }
        ia[j] = make_uint4(a4[0], a4[1], a4[2], a4[3]);
        ib[j] = make_uint4(b4[0], b4[1], b4[2], b4[3]);
    }
    const bool lane_live = col0 < p.words;
    const int64_t ntiles = (p.rows + 31) >> 5;
    const int64_t t0 = (int64_t)blockIdx.y * tiles_per_block;
    const int64_t t1 = min(ntiles, t0 + tiles_per_block);
    for (int64_t tile = t0 + rg; tile < t1; tile += RG) {
        uint32_t word[NJ];
#pragma unroll
        for (int j = 0; j < NJ; j++) word[j] = 0;
        const int64_t rbase = tile << 5;
        const int nrow = (int)min((int64_t)32, p.rows - rbase);
        // rows in batches of RB: issue all RB x NCOMP 128-bit loads before the
        // first ballot so each lane keeps RB*NCOMP*16 B in flight.
        // (RB divides 32: the row bits of a tile are shifted in per batch; two CTAs per SM.
        // Measured for the trio's single pass at w = 5691: RB 2 / 4 / 8 = 2.13 / 2.03 / 2.01 ms)
        constexpr int RB = (NPARTY == 1 || NPASS == 1) ? 8 : 4;
        static_assert(32 % RB == 0, "a batch of rows must divide the 32-row tile");
        for (int i0 = 0; i0 < nrow; i0 += RB) {
            uint4 cv[RB][NCOMP];
#pragma unroll
            for (int r = 0; r < RB; r++) {
                const int64_t row = rbase + i0 + r;
                const bool ok = lane_live && (i0 + r) < nrow;
#pragma unroll
                for (int c = 0; c < NCOMP; c++)
                    cv[r][c] = ok ? __ldcs(reinterpret_cast<const uint4*>(p.comp[c] + row * p.pitch + col0))
                                  : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int r = 0; r < RB; r++) {
#pragma unroll
                for (int ps = 0; ps < NPASS; ps++) {
#pragma unroll
                    for (int q = 0; q < NPARTY; q++) {
                        const int j = ps * NPARTY + q;
                        const uint4 A = cv[r][q], B = cv[r][(q + 1) % NCOMP];
                        const uint32_t part = ((A.x & ia[j].x) ^ (B.x & ib[j].x)) ^ ((A.y & ia[j].y) ^ (B.y & ib[j].y)) ^
                                              ((A.z & ia[j].z) ^ (B.z & ib[j].z)) ^ ((A.w & ia[j].w) ^ (B.w & ib[j].w));
                        if constexpr (NPARTY == 1) {  // measured faster per party (C3 uniform 3.9 vs 5.5 ms)
                            const uint32_t bal = __ballot_sync(0xffffffffu, __popc(part) & 1);
                            word[j] |= (uint32_t)(__popc(bal) & 1) << (i0 + r);
                        } else {
                            word[j] = (word[j] << 1) | (__popc(part) & 1u);  // lane-local, row i0 + r
                        }
                    }
                }
            }
        }
        // rows were shifted in first-to-last over a whole number of RB batches:
        // bit-reverse, drop the padding, then XOR over the lanes (one butterfly per j)
        const int npad = (nrow + RB - 1) / RB * RB;
        uint32_t v = 0;
#pragma unroll
        for (int j = 0; j < NJ; j++) {
            uint32_t w = word[j];
            if constexpr (NPARTY != 1) {
                w = __brev(w) >> (32 - npad);
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) w ^= __shfl_xor_sync(0xffffffffu, w, off);
            }
            if (j == lane) v = w;
        }
        if (lane < NJ && v) atomicXor(p.out[lane] + tile, v);
    }
}

// ---------------------------------------------------------------------------
// Masked parity for rows of at most 1024 words (the Zipf attributes of
// C3/C4, w = 313): indicators in registers as in v2, but the share rows are
// staged in shared memory by bulk copies (TMA), S stages deep, so the bytes
// in flight no longer ride on the registers of two CTAs per SM (v2 at C4:
// 128 registers, 18.75% occupancy, 5.26 TB/s).  One persistent CTA per SM;
// a stage is RT consecutive rows of every component -- contiguous at the row
// pitch, so one bulk copy per component.  Warp (rg, wc) owns the 128-word
// column chunk wc and rows rg, rg + RGW, ... of each stage; RT divides 32,
// so a stage's rows fall in one output word.
// ---------------------------------------------------------------------------
constexpr int kParTmaSmemMax = 200 * 1024;
constexpr int kParTmaMaxWords = 1024;

template <int NPARTY, int NPASS>
__global__ void __launch_bounds__(512, 1) masked_parity_tma_kernel(const ParityArgs p, int CW, int RT, int S) {
    constexpr int NJ = NPARTY * NPASS;
    constexpr int NCOMP = NPARTY == 1 ? 2 : 3;
    extern __shared__ __align__(128) unsigned char par_smem[];
    const int64_t P = p.pitch;
    const int64_t comp_bytes = (int64_t)RT * P * 4;  // one component's rows in a stage
    uint64_t* bar = reinterpret_cast<uint64_t*>(par_smem + S * NCOMP * comp_bytes);
    auto stage = [&](int s, int c) {
        return reinterpret_cast<const uint32_t*>(par_smem + (s * NCOMP + c) * comp_bytes);
    };
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int RGW = (int)(blockDim.x >> 5) / CW;
    const int rg = warp / CW, wc = warp % CW;
    const int64_t col0 = (int64_t)wc * 128 + lane * 4;
    uint4 ia[NJ], ib[NJ];
#pragma unroll
    for (int j = 0; j < NJ; j++) {
        uint32_t a4[4], b4[4];
#pragma unroll
        for (int e = 0; e < 4; e++) {
            const bool in = col0 + e < p.words;
            a4[e] = in ? __ldg(p.ind[2 * j] + col0 + e) : 0u;
            b4[e] = in ? __ldg(p.ind[2 * j + 1] + col0 + e) : 0u;
        }
        ia[j] = make_uint4(a4[0], a4[1], a4[2], a4[3]);
        ib[j] = make_uint4(b4[0], b4[1], b4[2], b4[3]);
    }
    const bool lane_live = col0 < P;
    const int64_t ntile = (p.rows + RT - 1) / RT;
    const int64_t G = gridDim.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; s++) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int64_t t, int s) {
        const int64_t r0 = t * RT;
        const uint32_t bytes = (uint32_t)(min((int64_t)RT, p.rows - r0) * P * 4);
        mbar_expect_tx(&bar[s], NCOMP * bytes);
#pragma unroll
        for (int c = 0; c < NCOMP; c++)
            bulk_g2s((void*)stage(s, c), p.comp[c] + r0 * P, bytes, &bar[s]);
    };
    if (threadIdx.x == 0)
        for (int s = 0; s < S; s++)
            if (blockIdx.x + s * G < ntile) issue(blockIdx.x + s * G, s);
    uint32_t phase = 0;  // bit s: phase of stage s
    int s = 0;
    for (int64_t t = blockIdx.x; t < ntile; t += G) {
        mbar_wait(&bar[s], (phase >> s) & 1);
        phase ^= 1u << s;
        const int64_t r0 = t * RT;
        const int nr = (int)min((int64_t)RT, p.rows - r0);
        const int sh = (int)(r0 & 31);
        // lane-local parity bits, one per (row, j), shifted in (no ballot per row);
        // then ONE butterfly XOR over the lanes of all j's bits packed in a word
        uint32_t acc[NJ];
#pragma unroll
        for (int j = 0; j < NJ; j++) acc[j] = 0;
        int nrw = 0;
        for (int r = rg; r < nr; r += RGW, nrw++) {
            uint4 cv[NCOMP];
#pragma unroll
            for (int c = 0; c < NCOMP; c++)
                cv[c] = lane_live ? *reinterpret_cast<const uint4*>(stage(s, c) + r * P + col0)
                                  : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int ps = 0; ps < NPASS; ps++) {
#pragma unroll
                for (int q = 0; q < NPARTY; q++) {
                    const int j = ps * NPARTY + q;
                    const uint4 A = cv[q], B = cv[(q + 1) % NCOMP];
                    const uint32_t part = ((A.x & ia[j].x) ^ (B.x & ib[j].x)) ^ ((A.y & ia[j].y) ^ (B.y & ib[j].y)) ^
                                          ((A.z & ia[j].z) ^ (B.z & ib[j].z)) ^ ((A.w & ia[j].w) ^ (B.w & ib[j].w));
                    acc[j] = (acc[j] << 1) | (__popc(part) & 1u);
                }
            }
        }
        if (nrw > 0) {  // warp-uniform; NJ * nrw <= 32 (host picks RT accordingly)
            uint32_t packed = 0;
#pragma unroll
            for (int j = 0; j < NJ; j++) packed |= acc[j] << (j * nrw);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) packed ^= __shfl_xor_sync(0xffffffffu, packed, off);
            if (lane < NJ) {
                const uint32_t a = packed >> (lane * nrw);
                uint32_t v = 0;
                for (int i = 0; i < nrw; i++) v |= ((a >> (nrw - 1 - i)) & 1u) << (sh + rg + i * RGW);
                if (v) atomicXor(p.out[lane] + (r0 >> 5), v);
            }
        }
        __syncthreads();  // stage s fully read before it is refilled
        if (threadIdx.x == 0 && t + S * G < ntile) issue(t + S * G, s);
        s = s + 1 == S ? 0 : s + 1;
    }
}

// ---------------------------------------------------------------------------
// src/rss.py:143-148 for all three parties at once: alpha_q = F(k_q) ^
// F(k_{q-1}) (party q holds its own key and its predecessor's,
// src/net.py:229-232), optionally XORed into per-party buffers.  3 AES per
// 16-byte block instead of 6.
// ---------------------------------------------------------------------------
struct Zs3Args {
    AesKeySched k[3];
    const uint32_t* xin[2][3];  // per pass (two zero-share counters per launch at most)
    uint32_t* out[2][3];
    uint64_t counter[2];
    int npass;
    int fold;   // 1: one output, zero share of counter[0] XOR that of counter[1] (npass = 1)
};

template <class TAB = AesTab>
__global__ void __launch_bounds__(kAesThreads) zero_share3_kernel(const __grid_constant__ Zs3Args a, uint32_t label_be,
                                                                   int64_t nwords, int64_t nbits, int64_t w0,
                                                                   int64_t nloc, int64_t row_words,
                                                                   uint32_t row_tail) {
    // words [w0, w0 + nloc) of the nwords-word stream (w0 % 4 == 0: whole
    // CTR blocks) for each of npass counters, written to out[pass][q][0 .. nloc)
    extern __shared__ __align__(128) uint8_t smem_raw[];
    TAB::fill(smem_raw);
    __syncthreads();
    const TAB T(smem_raw);
    const int64_t nblk = (nloc + 3) >> 2;
    const int64_t b0 = w0 >> 2;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nblk * a.npass; t += stride) {
        const int ps = t >= nblk ? 1 : 0;
        const int64_t b = t - ps * nblk;
        const uint4 ctr = ctr_block(label_be, a.counter[ps], (uint64_t)(b0 + b));
        uint4 f[3];
#pragma unroll
        for (int q = 0; q < 3; q++) f[q] = aes128_enc(T, ctr, ParamKey{a.k[q].rk});
        if (a.fold) {   // the two streams' shares XOR: F(c0) ^ F(c1) per key, then the partner XOR
            const uint4 ctr2 = ctr_block(label_be, a.counter[1], (uint64_t)(b0 + b));
#pragma unroll
            for (int q = 0; q < 3; q++) f[q] = xor4(f[q], aes128_enc(T, ctr2, ParamKey{a.k[q].rk}));
        }
#pragma unroll
        for (int q = 0; q < 3; q++) {
            const uint4 z = xor4(f[q], f[(q + 2) % 3]);
            const uint32_t zw[4] = {z.x, z.y, z.z, z.w};
            const uint32_t* xin = a.xin[ps][q];
            uint32_t* out = a.out[ps][q];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int64_t o = b * 4 + j;
                if (o >= nloc) break;
                uint32_t v = zw[j];
                if (xin) v ^= xin[o];
                if (w0 + o == nwords - 1 && (nbits & 31)) v &= (1u << (nbits & 31)) - 1u;
                // matrix re-share (src/engine.py:86-89): every row's tail masked after the XOR
                if (row_words && (w0 + o) % row_words == row_words - 1) v &= row_tail;
                out[o] = v;
            }
        }
    }
}

// The same stream for small launches (the latency-bound zero shares of C1 and
// of a rank's secEval slice): a CTA of three warps, warp q encrypting 32
// counter blocks under party q's key only (one AES per thread instead of
// three, and a warp-uniform key), partners exchanged through shared memory.
template <class TAB>
__global__ void __launch_bounds__(96) zero_share3x_kernel(const __grid_constant__ Zs3Args a, uint32_t label_be,
                                                          int64_t nwords, int64_t nbits, int64_t w0, int64_t nloc,
                                                          int64_t row_words, uint32_t row_tail) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    TAB::fill(smem_raw);
    uint4* xch = reinterpret_cast<uint4*>(smem_raw + TAB::kBytes);  // [3][32]
    __syncthreads();
    const TAB T(smem_raw);
    const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nblk = (nloc + 3) >> 2;
    const int64_t items = nblk * a.npass;
    const int64_t b0 = w0 >> 2;
    for (int64_t g = blockIdx.x; g * 32 < items; g += gridDim.x) {
        const int64_t t = g * 32 + lane;
        const bool valid = t < items;
        const int ps = t >= nblk ? 1 : 0;
        const int64_t b = t - ps * nblk;
        uint4 f = make_uint4(0, 0, 0, 0);
        if (valid) {
            f = aes128_enc(T, ctr_block(label_be, a.counter[ps], (uint64_t)(b0 + b)), ParamKey{a.k[q].rk});
            if (a.fold) f = xor4(f, aes128_enc(T, ctr_block(label_be, a.counter[1], (uint64_t)(b0 + b)), ParamKey{a.k[q].rk}));
        }
        xch[q * 32 + lane] = f;
        __syncthreads();
        if (valid) {
            const uint4 z = xor4(f, xch[((q + 2) % 3) * 32 + lane]);
            const uint32_t zw[4] = {z.x, z.y, z.z, z.w};
            const uint32_t* xin = a.xin[ps][q];
            uint32_t* out = a.out[ps][q];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int64_t o = b * 4 + j;
                if (o >= nloc) break;
                uint32_t v = zw[j];
                if (xin) v ^= xin[o];
                if (w0 + o == nwords - 1 && (nbits & 31)) v &= (1u << (nbits & 31)) - 1u;
                if (row_words && (w0 + o) % row_words == row_words - 1) v &= row_tail;
                out[o] = v;
            }
        }
        __syncthreads();  // xch is rewritten by the next group
    }
}

// ---------------------------------------------------------------------------
// src/rss.py:115-126 and_terms (per party), src/engine.py:174-189 XOR folds.
// ---------------------------------------------------------------------------
struct AndArgs {
    const uint32_t* aa[kMaxParty];
    const uint32_t* ab[kMaxParty];
    const uint32_t* ba[kMaxParty];
    const uint32_t* bb[kMaxParty];
    uint32_t* out[kMaxParty];
    int nparty;
};

__global__ void and_terms_kernel(const AndArgs a, int64_t nwords) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += stride) {
#pragma unroll
        for (int q = 0; q < kMaxParty; q++) {
            if (q >= a.nparty) break;
            const uint32_t x = a.aa[q][i], y = a.ab[q][i], u = a.ba[q][i], v = a.bb[q][i];
            a.out[q][i] = (x & u) ^ (x & v) ^ (y & u);
        }
    }
}

__global__ void xor3_kernel(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                            const uint32_t* __restrict__ c, uint32_t* __restrict__ out, int64_t nwords) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool vec = ((((uintptr_t)a) | ((uintptr_t)b) | ((uintptr_t)c) | ((uintptr_t)out)) & 15) == 0;
    int64_t done = 0;
    if (vec) {  // 128-bit streaming body
        const int64_t n4 = nwords >> 2;
        const uint4 *a4 = (const uint4*)a, *b4 = (const uint4*)b, *c4 = (const uint4*)c;
        uint4* o4 = (uint4*)out;
        for (int64_t i = t0; i < n4; i += stride) {
            uint4 v = xor4(__ldcs(a4 + i), __ldcs(b4 + i));
            if (c) v = xor4(v, __ldcs(c4 + i));
            __stcs(o4 + i, v);
        }
        done = n4 << 2;
    }
    for (int64_t i = done + t0; i < nwords; i += stride) out[i] = a[i] ^ b[i] ^ (c ? c[i] : 0u);
}

// ---------------------------------------------------------------------------
// src/engine.py:95-102 _select_one_additive: out_q = XOR_c [fa_q(c) (A_q[c] ^
// B_q[c]) ^ fb_q(c) A_q[c]] (flag bits are the party's two flag shares).
// Column-parallel partial folds, combined with atomicXor (out pre-zeroed).
// ---------------------------------------------------------------------------
struct FoldArgs {
    const uint32_t* A[kMaxParty];
    const uint32_t* B[kMaxParty];
    const uint32_t* fa[kMaxParty];
    const uint32_t* fb[kMaxParty];
    uint32_t* out[kMaxParty];
    int nparty;
    int64_t rows, words, pitch;
};

__global__ void select_fold_kernel(const FoldArgs a) {
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t w = t % a.words;
    const int64_t rstride = T / a.words;
    const int64_t r0 = t / a.words;
    if (r0 >= rstride) return;  // trailing threads of an incomplete column set
    uint32_t acc[kMaxParty] = {0, 0, 0};
    for (int64_t r = r0; r < a.rows; r += rstride) {
#pragma unroll
        for (int q = 0; q < kMaxParty; q++) {
            if (q >= a.nparty) break;
            const uint32_t fa = (__ldg(a.fa[q] + (r >> 5)) >> (r & 31)) & 1u;
            const uint32_t fb = (__ldg(a.fb[q] + (r >> 5)) >> (r & 31)) & 1u;
            const uint32_t x = a.A[q][r * a.pitch + w], y = a.B[q][r * a.pitch + w];
            acc[q] ^= ((x ^ y) & (0u - fa)) ^ (x & (0u - fb));
        }
    }
#pragma unroll
    for (int q = 0; q < kMaxParty; q++) {
        if (q >= a.nparty) break;
        if (acc[q]) atomicXor(a.out[q] + w, acc[q]);
    }
}

// The fold as a bandwidth kernel for aligned 16-byte-pitched tensors -- the
// sec_access posting fold (src/engine.py:309-311) and the Case I fold stream
// whole tensors.  NP = 3 is the trio case (B_q = A_{q+1}, fb_q = fa_{q+1}: the
// three co-resident parties, each component stored once and loaded once per
// row; the generic kernel loads it twice), NP = 1 one party's (A, B).  Each
// thread owns one 16-byte column chunk and a strided set of RB-row blocks
// (RB rows of 128-bit loads in flight), the row's selection bits are
// warp-broadcast loads, and partial folds combine with atomicXor.
template <int NP, int RB>
__global__ void __launch_bounds__(256) select_fold_vec4_kernel(const FoldArgs a, int64_t nch, int64_t rgroups) {
    constexpr int NC = NP == 1 ? 2 : 3;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t c = t % nch;
    const int64_t g = t / nch;
    if (g >= rgroups) return;
    const int64_t p4 = a.pitch >> 2;
    const uint4* X[NC];
    const uint32_t* F[NC];
#pragma unroll
    for (int k = 0; k < NC; k++) {
        X[k] = reinterpret_cast<const uint4*>(NP == 1 && k == 1 ? a.B[0] : a.A[k]) + c;
        F[k] = NP == 1 && k == 1 ? a.fb[0] : a.fa[k];
    }
    uint4 acc[NP];
#pragma unroll
    for (int q = 0; q < NP; q++) acc[q] = make_uint4(0, 0, 0, 0);
    for (int64_t r0 = g * RB; r0 < a.rows; r0 += rgroups * RB) {
        uint4 v[RB][NC];
        uint32_t f[RB][NC];
#pragma unroll
        for (int k = 0; k < RB; k++) {
            const int64_t r = r0 + k;
            const bool ok = r < a.rows;
            const int64_t o = ok ? r * p4 : 0;
#pragma unroll
            for (int m = 0; m < NC; m++) {
                v[k][m] = ok ? __ldcs(X[m] + o) : make_uint4(0, 0, 0, 0);
                f[k][m] = ok ? (__ldg(F[m] + (r >> 5)) >> (r & 31)) & 1u : 0u;
            }
        }
#pragma unroll
        for (int k = 0; k < RB; k++) {
#pragma unroll
            for (int q = 0; q < NP; q++) {
                const uint32_t ma = 0u - f[k][q], mb = 0u - f[k][(q + 1) % NC];
                const uint4 x = v[k][q], y = v[k][(q + 1) % NC];
                acc[q].x ^= ((x.x ^ y.x) & ma) ^ (x.x & mb);
                acc[q].y ^= ((x.y ^ y.y) & ma) ^ (x.y & mb);
                acc[q].z ^= ((x.z ^ y.z) & ma) ^ (x.z & mb);
                acc[q].w ^= ((x.w ^ y.w) & ma) ^ (x.w & mb);
            }
        }
    }
#pragma unroll
    for (int q = 0; q < NP; q++) {
        const int64_t w = c * 4;
        const uint32_t vals[4] = {acc[q].x, acc[q].y, acc[q].z, acc[q].w};
#pragma unroll
        for (int j = 0; j < 4; j++)
            if (w + j < a.words && vals[j]) atomicXor(a.out[q] + w + j, vals[j]);
    }
}

// ---------------------------------------------------------------------------
// Bit-granular row packing (src/engine.py:227-233, 317-318), fused with the
// first gather of the shuffle that consumes the rows (src/shuffle.py:106-118):
//
//   out[i] = XOR_s ( flag_s[src] || field_s0[src] || field_s1[src] ... ) ^ R[i]
//   src = idx ? idx[i] : i
//
// Each field keeps its logical width; rows are packed LE with a clean tail
// and zero padding up to the output pitch.  With s over two share
// components the kernel emits a^b directly, and with idx = the party's
// composed permutation it is the party's first shuffle step -- the packed
// rows never round-trip through HBM.
// ---------------------------------------------------------------------------
constexpr int kMaxFields = 8;
constexpr int kMaxSets = 3;

struct PackArgs {
    const int32_t* idx;
    const uint32_t* flag[kMaxSets];  // bit vectors (bit 0 of each row), all null if the rows carry no flag
    const uint32_t* f[kMaxSets][kMaxFields];
    int64_t fpitch[kMaxSets][kMaxFields];
    int64_t fwidth[kMaxFields];
    int64_t foff[kMaxFields];
    int nsets, nfields;
    int vec_fields;  // every field row is 16-B aligned with a 16-B pitch
    const uint32_t* r;  // XORed rows (pitch opitch) or null
    uint32_t* out;
    int64_t opitch, owidth, rows;
};

__device__ __forceinline__ uint32_t field_bits32(const uint32_t* row, int64_t width, int64_t s) {
    // 32 bits of a width-bit field starting at (possibly negative) position s
    uint32_t lo = 0, hi = 0;
    const int64_t wi = s >= 0 ? (s >> 5) : -1;
    const int sh = (int)(s & 31);
    const int64_t nw = (width + 31) >> 5;
    if (wi >= 0 && wi < nw) lo = row[wi];
    if (wi + 1 >= 0 && wi + 1 < nw) hi = row[wi + 1];
    return sh ? __funnelshift_r(lo, hi, sh) : lo;
}

// output word k of source row src (any position: flag, field boundaries, tail)
__device__ __forceinline__ uint32_t pack_word(const PackArgs& a, int64_t src, int64_t k, int64_t ow) {
    if (k >= ow) return 0;
    uint32_t v = 0;
    const int64_t lo = k * 32;
    for (int s = 0; s < a.nsets; s++) {
        if (lo == 0 && a.flag[s]) v ^= (__ldg(a.flag[s] + (src >> 5)) >> (src & 31)) & 1u;
        for (int f = 0; f < a.nfields; f++) {
            const int64_t o = a.foff[f], wdt = a.fwidth[f];
            if (o >= lo + 32 || o + wdt <= lo) continue;
            const uint32_t bits = field_bits32(a.f[s][f] + src * a.fpitch[s][f], wdt, lo - o);
            // keep only positions inside [o, o+wdt) of this word
            const int64_t b0 = o > lo ? o - lo : 0;
            const int64_t b1 = (o + wdt < lo + 32) ? o + wdt - lo : 32;
            const uint32_t m = (b1 - b0 >= 32) ? 0xffffffffu : (((1u << (b1 - b0)) - 1u) << b0);
            v ^= bits & m;
        }
    }
    return v;
}

template <int D>
__device__ __forceinline__ void take4(const uint32_t w[8], int sh, uint32_t o[4]) {
#pragma unroll
    for (int j = 0; j < 4; j++) o[j] ^= __funnelshift_r(w[D + j], w[D + j + 1], sh);
}

// output words [4c, 4c+4) of source row src
__device__ __forceinline__ void pack_chunk(const PackArgs& a, int64_t src, int64_t c, int64_t ow, uint32_t o[4]) {
    const int64_t b = c * 128;
    int f = -1;
    for (int g = 0; g < a.nfields; g++)
        if (a.foff[g] <= b && b + 128 <= a.foff[g] + a.fwidth[g]) f = g;
    o[0] = o[1] = o[2] = o[3] = 0;
    if (f < 0) {  // flag word, field boundary or tail: word by word
#pragma unroll
        for (int j = 0; j < 4; j++) o[j] = pack_word(a, src, 4 * c + j, ow);
        return;
    }
    // interior of one field: 4 output words = a funnel shift of 5 field words
    const int64_t s0 = b - a.foff[f];
    const int64_t q = s0 >> 5;
    const int sh = (int)(s0 & 31);
    const int d = (int)(q & 3);  // uniform across a warp inside one field
    const int64_t nw = (a.fwidth[f] + 31) >> 5;
    for (int s = 0; s < a.nsets; s++) {
        const uint32_t* row = a.f[s][f] + src * a.fpitch[s][f];
        uint32_t w[8];
        if (a.vec_fields) {
            const uint4 x = __ldg(reinterpret_cast<const uint4*>(row + (q - d)));
            w[0] = x.x; w[1] = x.y; w[2] = x.z; w[3] = x.w;
            if (d || sh) {
                const uint4 y = __ldg(reinterpret_cast<const uint4*>(row + (q - d) + 4));
                w[4] = y.x; w[5] = y.y; w[6] = y.z; w[7] = y.w;
            } else {
                w[4] = w[5] = w[6] = w[7] = 0;
            }
            switch (d) {
                case 0: take4<0>(w, sh, o); break;
                case 1: take4<1>(w, sh, o); break;
                case 2: take4<2>(w, sh, o); break;
                default: take4<3>(w, sh, o); break;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 4; j++) w[j] = __ldg(row + q + j);
            w[4] = (sh && q + 4 < nw) ? __ldg(row + q + 4) : 0;
            take4<0>(w, sh, o);
        }
    }
}

// the field whose interior holds output bits [128c, 128c+128), or -1
__device__ __forceinline__ int interior_field(const PackArgs& a, int64_t c) {
    const int64_t b = c * 128;
    int f = -1;
    for (int g = 0; g < a.nfields; g++)
        if (a.foff[g] <= b && b + 128 <= a.foff[g] + a.fwidth[g]) f = g;
    return f;
}

// wide rows, NS share sets with 16-B aligned field rows: a CTA walks rows;
// each thread issues every load of two 128-bit output groups (field words
// of all sets + the XORed row) before it computes either, so twice the
// bytes are in flight per warp (four measured slower: registers halve the
// occupancy).  Field words are read through L1 (a lane's second group is its
// neighbour's first: evict-first loads re-read it from L2/DRAM, 8.6 vs 7.9 ms
// at C3).  NS = 0: unaligned fields, generic loads.
// TAB: the per-chunk field, shift and source offset -- the same for every row
// -- computed once per CTA into a shared-memory table (8 B per 128-bit
// output chunk, rows up to kPackTabChunks chunks) instead of per chunk and
// row (the field search and 64-bit offset math made the kernel issue-bound:
// ~250 warp instructions per chunk at C3).
constexpr int kPackTabChunks = 6144;   // 48 KB of table: rows up to 98 KB

template <int NS, bool TAB = false>
__global__ void __launch_bounds__(256) pack_gather_rows_kernel(const PackArgs a) {
    const int64_t ow = (a.owidth + 31) >> 5;
    const int64_t ng = a.opitch >> 2;
    const int bd = blockDim.x;
    extern __shared__ uint2 pk_tab[];   // TAB: x = (field + 1) | du << 8 | sh << 16, y = source group offset
    if (TAB) {
        for (int64_t c = threadIdx.x; c < ng; c += bd) {
            const int f = interior_field(a, c);
            uint2 e = make_uint2(0u, 0u);
            if (f >= 0) {
                const int64_t s0 = c * 128 - a.foff[f];
                const int64_t q = s0 >> 5;
                const int du = (int)(q & 3);
                e = make_uint2((uint32_t)(f + 1) | ((uint32_t)du << 8) | ((uint32_t)(s0 & 31) << 16),
                               (uint32_t)(q - du));
            }
            pk_tab[c] = e;
        }
        __syncthreads();
    }
    for (int64_t i = blockIdx.x; i < a.rows; i += gridDim.x) {
        const int64_t src = a.idx ? (int64_t)__ldg(a.idx + i) : i;
        uint4* orow = reinterpret_cast<uint4*>(a.out + i * a.opitch);
        const uint4* rrow = a.r ? reinterpret_cast<const uint4*>(a.r + i * a.opitch) : nullptr;
        if constexpr (NS == 0) {
            for (int64_t c = threadIdx.x; c < ng; c += bd) {
                uint32_t o[4];
                pack_chunk(a, src, c, ow, o);
                uint4 v = make_uint4(o[0], o[1], o[2], o[3]);
                if (rrow) v = xor4(v, __ldcs(rrow + c));
                orow[c] = v;
            }
        } else {
            for (int64_t c0 = threadIdx.x; c0 < ng; c0 += 2 * bd) {
                int64_t cc[2] = {c0, c0 + bd};
                int fu[2], shu[2], du[2];
                uint4 rv[2], A[2][NS], B[2][NS];
#pragma unroll
                for (int u = 0; u < 2; u++) {
                    const bool valid = cc[u] < ng;
                    rv[u] = (rrow && valid) ? __ldcs(rrow + cc[u]) : make_uint4(0, 0, 0, 0);
                    int f;
                    int64_t base = 0;
                    shu[u] = du[u] = 0;
                    if (TAB) {
                        const uint2 e = valid ? pk_tab[cc[u]] : make_uint2(0u, 0u);
                        f = (int)(e.x & 0xffu) - 1;
                        du[u] = (int)((e.x >> 8) & 3u);
                        shu[u] = (int)((e.x >> 16) & 31u);
                        base = (int64_t)e.y;
                    } else {
                        f = valid ? interior_field(a, cc[u]) : -1;
                        if (f >= 0) {
                            const int64_t s0 = cc[u] * 128 - a.foff[f];
                            const int64_t q = s0 >> 5;
                            shu[u] = (int)(s0 & 31);
                            du[u] = (int)(q & 3);
                            base = q - du[u];
                        }
                    }
                    fu[u] = valid ? f : -2;
#pragma unroll
                    for (int s = 0; s < NS; s++) {
                        A[u][s] = B[u][s] = make_uint4(0, 0, 0, 0);
                        if (f >= 0) {
                            const uint4* row = reinterpret_cast<const uint4*>(a.f[s][f] + src * a.fpitch[s][f] + base);
                            A[u][s] = __ldg(row);
                            if (du[u] || shu[u]) B[u][s] = __ldg(row + 1);
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < 2; u++) {
                    if (fu[u] == -2) continue;
                    uint32_t o[4] = {0, 0, 0, 0};
                    if (fu[u] < 0) {
#pragma unroll
                        for (int j = 0; j < 4; j++) o[j] = pack_word(a, src, 4 * cc[u] + j, ow);
                    } else {
#pragma unroll
                        for (int s = 0; s < NS; s++) {
                            const uint32_t w[8] = {A[u][s].x, A[u][s].y, A[u][s].z, A[u][s].w,
                                                   B[u][s].x, B[u][s].y, B[u][s].z, B[u][s].w};
                            switch (du[u]) {
                                case 0: take4<0>(w, shu[u], o); break;
                                case 1: take4<1>(w, shu[u], o); break;
                                case 2: take4<2>(w, shu[u], o); break;
                                default: take4<3>(w, shu[u], o); break;
                            }
                        }
                    }
                    orow[cc[u]] = xor4(make_uint4(o[0], o[1], o[2], o[3]), rv[u]);
                }
            }
        }
    }
}

// narrow or unaligned rows: thread per (row, output word)
__global__ void pack_gather_kernel(const PackArgs a) {
    const int64_t total = a.rows * a.opitch;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t ow = (a.owidth + 31) >> 5;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
        const int64_t i = t / a.opitch, k = t - i * a.opitch;
        const int64_t src = a.idx ? (int64_t)__ldg(a.idx + i) : i;
        uint32_t v = pack_word(a, src, k, ow);
        if (a.r) v ^= a.r[t];
        a.out[t] = v;
    }
}

// out[k] = bits [off, off+width) of row idx[k] (idx null -> identity).
__global__ void extract_field_kernel(const uint32_t* __restrict__ src, int64_t spitch,
                                     const int32_t* __restrict__ idx, int64_t n, int64_t off, int64_t width,
                                     uint32_t* __restrict__ out, int64_t opitch) {
    const int64_t ow = (width + 31) >> 5;
    const int64_t total = n * opitch;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t sw = (off + width + 31) >> 5;  // words of the source row that are read
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
        const int64_t k = t / opitch, j = t % opitch;
        uint32_t v = 0;
        if (j < ow) {
            const int64_t r = idx ? idx[k] : k;
            v = field_bits32(src + r * spitch, sw * 32, off + j * 32);
            if (j == ow - 1 && (width & 31)) v &= (1u << (width & 31)) - 1u;
        }
        out[k * opitch + j] = v;
    }
}

// Several narrow extractions from the same kept rows in one launch
// (blockIdx.y = job): the trio open-keep's 3 components x fields.
constexpr int kMaxExtract = 24;
struct ExtractJob {
    const uint32_t* src;
    uint32_t* out;
    int64_t off, width, opitch;
};
struct ExtractJobs {
    ExtractJob j[kMaxExtract];
    const int32_t* idx;
    int64_t spitch, n;
};

__global__ void extract_field_multi_kernel(const __grid_constant__ ExtractJobs J) {
    const ExtractJob& e = J.j[blockIdx.y];
    const int64_t ow = (e.width + 31) >> 5;
    const int64_t total = J.n * e.opitch;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t sw = (e.off + e.width + 31) >> 5;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
        const int64_t k = t / e.opitch, j = t % e.opitch;
        uint32_t v = 0;
        if (j < ow) {
            const int64_t r = J.idx ? J.idx[k] : k;
            v = field_bits32(e.src + r * J.spitch, sw * 32, e.off + j * 32);
            if (j == ow - 1 && (e.width & 31)) v &= (1u << (e.width & 31)) - 1u;
        }
        e.out[k * e.opitch + j] = v;
    }
}

// clean row tails after a matrix re-share (src/engine.py:88-89)
__global__ void mask_row_tails_kernel(uint32_t* __restrict__ mat, int64_t rows, int64_t pitch, int64_t w,
                                      uint32_t mask) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += stride)
        mat[r * pitch + w - 1] &= mask;
}

__global__ void extract_field_rows_kernel(const uint32_t* __restrict__ src, int64_t spitch,
                                          const int32_t* __restrict__ idx, int64_t n, int64_t off, int64_t width,
                                          uint32_t* __restrict__ out, int64_t opitch) {
    const int64_t ow = (width + 31) >> 5;
    const int64_t sw = (off + width + 31) >> 5;
    for (int64_t k = blockIdx.x; k < n; k += gridDim.x) {
        const int64_t r = idx ? idx[k] : k;
        for (int64_t j = threadIdx.x; j < opitch; j += blockDim.x) {
            uint32_t v = 0;
            if (j < ow) {
                v = field_bits32(src + r * spitch, sw * 32, off + j * 32);
                if (j == ow - 1 && (width & 31)) v &= (1u << (width & 31)) - 1u;
            }
            out[k * opitch + j] = v;
        }
    }
}

// bit r of out = mat[r][0] & 1 (the flag column, src/engine.py:241-245).
__global__ void column_bit_kernel(const uint32_t* __restrict__ mat, int64_t pitch, int64_t rows,
                                  uint32_t* __restrict__ out) {
    const int64_t nw = (rows + 31) >> 5;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += stride) {
        uint32_t v = 0;
        const int64_t r0 = w << 5;
        const int n = (int)min((int64_t)32, rows - r0);
        for (int i = 0; i < n; i++) v |= (mat[(r0 + i) * pitch] & 1u) << i;
        out[w] = v;
    }
}

// The opened flag column of a trio table: bit i of word w = XOR over the
// three components of bit 0 of row 32w+i (src/rss.py:184-206 on the column).
__global__ void column_open3_kernel(const uint32_t* __restrict__ m0, const uint32_t* __restrict__ m1,
                                    const uint32_t* __restrict__ m2, int64_t pitch, int64_t rows,
                                    uint32_t* __restrict__ out) {
    const int64_t nw = (rows + 31) >> 5;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += stride) {
        uint32_t v = 0;
        const int64_t r0 = w << 5;
        const int n = (int)min((int64_t)32, rows - r0);
        for (int i = 0; i < n; i++) {
            const int64_t o = (r0 + i) * pitch;
            v |= ((m0[o] ^ m1[o] ^ m2[o]) & 1u) << i;
        }
        out[w] = v;
    }
}

// ---------------------------------------------------------------------------
// src/engine.py:105-120 _select_many_additive: GF(2) product of K one-hot
// selector rows (K, X) with (X, W) share rows.  Selectors are transposed to
// one 32-bit mask per x per chunk of 32 selectors; a thread owns one word
// column and a range of x, folding into 32 accumulators.
// ---------------------------------------------------------------------------
__global__ void transpose_sel_kernel(const uint32_t* __restrict__ sel, int64_t spitch, int64_t K,
                                     int64_t k0, int64_t X, uint32_t* __restrict__ tmask) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int kn = (int)min((int64_t)32, K - k0);
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < X; x += stride) {
        uint32_t m = 0;
        for (int k = 0; k < kn; k++) m |= ((sel[(k0 + k) * spitch + (x >> 5)] >> (x & 31)) & 1u) << k;
        tmask[x] = m;
    }
}

__global__ void select_many_kernel(const uint32_t* __restrict__ ta, const uint32_t* __restrict__ tb,
                                   const uint32_t* __restrict__ A, const uint32_t* __restrict__ B,
                                   int64_t X, int64_t words, int64_t pitch, int kn,
                                   uint32_t* __restrict__ out, int64_t opitch) {
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t w = t % words;
    const int64_t xs = T / words;
    const int64_t x0 = t / words;
    if (x0 >= xs) return;
    uint32_t acc[32];
#pragma unroll
    for (int k = 0; k < 32; k++) acc[k] = 0;
    for (int64_t x = x0; x < X; x += xs) {
        const uint32_t ma = __ldg(ta + x), mb = __ldg(tb + x);
        if (!(ma | mb)) continue;
        const uint32_t a = A[x * pitch + w], b = B[x * pitch + w];
        const uint32_t ab = a ^ b;
#pragma unroll
        for (int k = 0; k < 32; k++) acc[k] ^= (ab & (0u - ((ma >> k) & 1u))) ^ (a & (0u - ((mb >> k) & 1u)));
    }
#pragma unroll
    for (int k = 0; k < 32; k++)
        if (k < kn && acc[k]) atomicXor(out + k * opitch + w, acc[k]);
}

// OGMS record payloads (src/storage.py:43-65) -> device matrices.  A warp per
// record; payloads sit at arbitrary byte offsets (15-byte headers), so each
// word is a funnel shift of two aligned words of the file image.
__global__ void unpack_records_kernel(const uint32_t* __restrict__ blob_words, int64_t blob_bytes, int64_t nrec,
                                      const int64_t* __restrict__ src_off, const int64_t* __restrict__ dst_off,
                                      const int32_t* __restrict__ nwords, uint32_t* __restrict__ arena) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t nblob = (blob_bytes + 3) >> 2;
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < nrec; r += warps) {
        const int64_t src = src_off[r];
        const int64_t base = src >> 2;
        const int sh = (int)(src & 3) * 8;
        const int n = nwords[r];
        uint32_t* dst = arena + dst_off[r];
        for (int j = lane; j < n; j += 32) {
            const uint32_t lo = blob_words[base + j];
            const uint32_t hi = (base + j + 1 < nblob) ? blob_words[base + j + 1] : 0u;
            dst[j] = sh ? __funnelshift_r(lo, hi, sh) : lo;
        }
    }
}

int engine_init() {
    OGM_CUDA_TRY(allow_big_smem(zero_share3_kernel<AesTab>, kAesTableBytes));
    return OGM_OK;
}

static int grid_for(int64_t work, int threads = 256) {
    int64_t g = (work + threads - 1) / threads;
    int64_t cap = (int64_t)sm_count() * 16;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

}  // namespace ogm

// ===========================================================================
// C ABI
// ===========================================================================
namespace ogm {
static int masked_parity_impl(int64_t rows, int64_t words, int64_t pitch, int ncomp, const uint32_t* const* comps,
                              int nparty, const int32_t* a_idx, const int32_t* b_idx, int npass,
                              const uint32_t* const* ind, uint32_t* const* out, bool acc, void* stream) {
    OGM_CHECK_ARG(rows >= 0 && words >= 0 && pitch >= words, OGM_ERR_ARG, "bad matrix shape");
    OGM_CHECK_ARG((nparty == 1 && ncomp == 2) || (nparty == 3 && ncomp == 3), OGM_ERR_ARG,
                  "need nparty=1 with 2 components (A, B) or nparty=3 with 3 components");
    OGM_CHECK_ARG(npass == 1 || npass == 2, OGM_ERR_ARG, "npass must be 1 or 2");
    if (rows == 0) return OGM_OK;
    ParityArgs p{};
    bool aligned = (pitch % 4) == 0;
    for (int c = 0; c < ncomp; c++) {
        p.comp[c] = comps[c];
        aligned = aligned && (((uintptr_t)comps[c]) & 15) == 0;
    }
    for (int q = 0; q < nparty; q++) {
        // party q reads (x_q, x_{q+1}) (src/graphs.py:382-399): fixed mapping
        OGM_CHECK_ARG(a_idx[q] == q && b_idx[q] == (q + 1) % ncomp, OGM_ERR_ARG,
                      "party %d must read components (%d, %d)", q, q, (q + 1) % ncomp);
        p.a_idx[q] = a_idx[q];
        p.b_idx[q] = b_idx[q];
    }
    for (int j = 0; j < npass * nparty; j++) {
        p.ind[2 * j] = ind[2 * j];
        p.ind[2 * j + 1] = ind[2 * j + 1];
        aligned = aligned && ((((uintptr_t)ind[2 * j]) | ((uintptr_t)ind[2 * j + 1])) & 15) == 0;
        p.out[j] = out[j];
    }
    p.ncomp = ncomp;
    p.nparty = nparty;
    p.npass = npass;
    p.acc = acc ? 1 : 0;
    p.rows = rows;
    p.words = words;
    p.pitch = pitch;
    cudaStream_t st = as_stream(stream);
    if (aligned && words >= 64 && pitch <= kParTmaMaxWords) {
        // short rows: bulk-copy staged rows (masked_parity_tma_kernel)
        const int CW = (int)((words + 127) / 128);
        int RGW = 1;
        while (RGW * 2 * CW <= 16) RGW <<= 1;
        // a warp's rows per stage times the (pass, party) count must fit one packed word
        const int rows_per_warp = 32 / (npass * nparty);
        int RT = 32;
        // stages as large as three fit (smaller stages measured far slower at C4: RT 16 / 8 / 4 =
        // 1.24 / 1.70 / 2.51 ms -- the per-stage barrier and butterfly amortise over fewer rows)
        while (RT > 1 && ((int64_t)ncomp * RT * pitch * 4 > kParTmaSmemMax / 3 || RT > RGW * rows_per_warp)) RT >>= 1;
        if (RGW > RT) RGW = RT;
        const int64_t stage_bytes = (int64_t)ncomp * RT * pitch * 4;
        const int S = (int)std::min<int64_t>(6, kParTmaSmemMax / stage_bytes);
        const int64_t ntile = (rows + RT - 1) / RT;
        const int G = (int)std::min<int64_t>(ntile, (int64_t)sm_count());
        const size_t smem = (size_t)(S * stage_bytes + 8 * S);
        if (!acc)
            for (int j = 0; j < npass * nparty; j++)
                OGM_CUDA_TRY(cudaMemsetAsync(out[j], 0, 4 * ((rows + 31) / 32), st));
#define OGM_PARITY_TMA(NP, NS)                                                                   \
    do {                                                                                         \
        OGM_CUDA_TRY(allow_big_smem(masked_parity_tma_kernel<NP, NS>, (int)smem));               \
        masked_parity_tma_kernel<NP, NS><<<G, 32 * CW * RGW, smem, st>>>(p, CW, RT, S);          \
    } while (0)
        if (nparty == 1 && npass == 1) OGM_PARITY_TMA(1, 1);
        else if (nparty == 1) OGM_PARITY_TMA(1, 2);
        else if (npass == 1) OGM_PARITY_TMA(3, 1);
        else OGM_PARITY_TMA(3, 2);
#undef OGM_PARITY_TMA
        OGM_LAUNCH_CHECK();
        return OGM_OK;
    }
    if (aligned && words >= 64) {
        // register-resident indicators; CW warps (x128 columns) per row group
        // as many 128-word warp columns as the row needs (<= 8): at w = 313 (the
        // Zipf attributes of C3/C4) 3 warps keep 82% of lanes live where a
        // power-of-two 4 kept 61%
        const int CW = (int)std::min<int64_t>(8, (words + 127) / 128);
        const int64_t col_chunks = (words + CW * 128 - 1) / (CW * 128);
        const int64_t ntiles = (rows + 31) / 32;
        const int64_t want_blocks = (int64_t)sm_count() * 6;
        int64_t row_blocks = want_blocks / col_chunks;
        if (row_blocks < 1) row_blocks = 1;
        if (row_blocks > 65535) row_blocks = 65535;
        const int RG = std::max(1, 8 / CW);
        int64_t tpb = (ntiles + row_blocks - 1) / row_blocks;
        tpb = (tpb + RG - 1) / RG * RG;
        row_blocks = (ntiles + tpb - 1) / tpb;
        if (!acc)
            for (int j = 0; j < npass * nparty; j++)
                OGM_CUDA_TRY(cudaMemsetAsync(out[j], 0, 4 * ntiles, st));
        dim3 grid((unsigned)col_chunks, (unsigned)row_blocks);
#define OGM_PARITY2(NP, NS) masked_parity_v2_kernel<NP, NS><<<grid, 32 * RG * CW, 0, st>>>(p, CW, tpb)
        if (nparty == 1 && npass == 1) OGM_PARITY2(1, 1);
        else if (nparty == 1) OGM_PARITY2(1, 2);
        else if (npass == 1) OGM_PARITY2(3, 1);
        else OGM_PARITY2(3, 2);
#undef OGM_PARITY2
        OGM_LAUNCH_CHECK();
        return OGM_OK;
    }
    const int64_t units = aligned ? (words + 3) / 4 : words;
    int G = 1;
    while (G < 32 && G * 4 < units) G <<= 1;  // >= ~4 loads per lane per row
    p.G = G;
    const int64_t tiles = (rows + 31) / 32;
    int64_t grid = (tiles + 7) / 8;
    int64_t cap = (int64_t)sm_count() * 8;
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
#define OGM_PARITY_LAUNCH(V, NP, NS) masked_parity_kernel<V, NP, NS><<<(int)grid, 256, 0, st>>>(p)
    if (aligned) {
        if (nparty == 1 && npass == 1) OGM_PARITY_LAUNCH(true, 1, 1);
        else if (nparty == 1) OGM_PARITY_LAUNCH(true, 1, 2);
        else if (npass == 1) OGM_PARITY_LAUNCH(true, 3, 1);
        else OGM_PARITY_LAUNCH(true, 3, 2);
    } else {
        if (nparty == 1 && npass == 1) OGM_PARITY_LAUNCH(false, 1, 1);
        else if (nparty == 1) OGM_PARITY_LAUNCH(false, 1, 2);
        else if (npass == 1) OGM_PARITY_LAUNCH(false, 3, 1);
        else OGM_PARITY_LAUNCH(false, 3, 2);
    }
#undef OGM_PARITY_LAUNCH
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}
}  // namespace ogm

extern "C" {

int ogm_masked_parity(int64_t rows, int64_t words, int64_t pitch, int ncomp, const uint32_t* const* comps,
                      int nparty, const int32_t* a_idx, const int32_t* b_idx, int npass,
                      const uint32_t* const* ind, uint32_t* const* out, void* stream) {
    return ogm::masked_parity_impl(rows, words, pitch, ncomp, comps, nparty, a_idx, b_idx, npass, ind, out, false,
                                   stream);
}

int ogm_masked_parity_acc(int64_t rows, int64_t words, int64_t pitch, int ncomp, const uint32_t* const* comps,
                          int nparty, const int32_t* a_idx, const int32_t* b_idx, int npass,
                          const uint32_t* const* ind, uint32_t* const* out, void* stream) {
    return ogm::masked_parity_impl(rows, words, pitch, ncomp, comps, nparty, a_idx, b_idx, npass, ind, out, true,
                                   stream);
}

static int zero_share_trio_impl(const uint8_t* k1, const uint8_t* k2, const uint8_t* k3, uint64_t counter,
                                int64_t nbits, int64_t w0, int64_t nloc, const uint32_t* const* xor_into,
                                uint32_t* const* out, void* stream, int64_t row_words = 0,
                                uint32_t row_tail = 0xffffffffu, int npass = 1, uint64_t counter2 = 0,
                                const uint32_t* const* xor_into2 = nullptr, uint32_t* const* out2 = nullptr,
                                int fold = 0) {
    using namespace ogm;
    OGM_CHECK_ARG(k1 && k2 && k3 && out && (npass == 1 || out2), OGM_ERR_ARG,
                  "zero-share keys and outputs are required");
    OGM_CHECK_ARG(nbits >= 0, OGM_ERR_ARG, "negative bit count");
    const int64_t nwords = (nbits + 31) / 32;
    OGM_CHECK_ARG(w0 >= 0 && (w0 & 3) == 0 && nloc >= 0 && w0 + nloc <= nwords, OGM_ERR_ARG,
                  "slice [%lld, +%lld) must start on a CTR block inside %lld words", (long long)w0,
                  (long long)nloc, (long long)nwords);
    if (nloc == 0) return OGM_OK;
    OGM_ENSURE_INIT();
    static const uint8_t kZshr[4] = {'Z', 'S', 'H', 'R'};
    Zs3Args a{};
    a.k[0] = make_sched(k1);
    a.k[1] = make_sched(k2);
    a.k[2] = make_sched(k3);
    a.npass = npass;
    a.fold = fold;
    a.counter[0] = counter;
    a.counter[1] = counter2;
    for (int q = 0; q < 3; q++) {
        a.xin[0][q] = xor_into ? xor_into[q] : nullptr;
        a.out[0][q] = out[q];
        if (npass == 2) {
            a.xin[1][q] = xor_into2 ? xor_into2[q] : nullptr;
            a.out[1][q] = out2[q];
        }
    }
    const int64_t items = npass * ((nloc + 3) / 4);
    if (items <= kAesSmallMaxWork) {
        const int64_t g = (items + 31) / 32;
        zero_share3x_kernel<AesTabSmall><<<(int)g, 96, kAesSmallBytes + 3 * 32 * 16, as_stream(stream)>>>(
            a, label_be(kZshr), nwords, nbits, w0, nloc, row_words, row_tail);
    } else {
        aes_launch(zero_share3_kernel<AesTab>, zero_share3_kernel<AesTabSmall>, items, kAesThreads,
                   as_stream(stream), a, label_be(kZshr), nwords, nbits, w0, nloc, row_words, row_tail);
    }
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

int ogm_zero_share_trio(const uint8_t* k1, const uint8_t* k2, const uint8_t* k3, uint64_t counter,
                        int64_t nbits, const uint32_t* const* xor_into, uint32_t* const* out, void* stream) {
    return zero_share_trio_impl(k1, k2, k3, counter, nbits, 0, (nbits + 31) / 32, xor_into, out, stream);
}

int ogm_zero_share_trio_rows(const uint8_t* k1, const uint8_t* k2, const uint8_t* k3, uint64_t counter, int64_t rows,
                             int64_t words, int64_t width, const uint32_t* const* xor_into, uint32_t* const* out,
                             void* stream) {
    OGM_CHECK_ARG(rows >= 0 && words >= 0 && width >= 0 && (width + 31) / 32 <= words, OGM_ERR_ARG,
                  "bad re-share matrix shape");
    const uint32_t tail = (width & 31) ? ((1u << (width & 31)) - 1u) : 0xffffffffu;
    return zero_share_trio_impl(k1, k2, k3, counter, rows * words * 32, 0, rows * words, xor_into, out, stream,
                                words, tail);
}

int ogm_zero_share_trio_slice2(const uint8_t* k1, const uint8_t* k2, const uint8_t* k3, uint64_t counter1,
                               uint64_t counter2, int64_t nbits, int64_t w0, int64_t nwords,
                               const uint32_t* const* xor_into1, uint32_t* const* out1,
                               const uint32_t* const* xor_into2, uint32_t* const* out2, void* stream) {
    return zero_share_trio_impl(k1, k2, k3, counter1, nbits, w0, nwords, xor_into1, out1, stream, 0, 0xffffffffu, 2,
                                counter2, xor_into2, out2);
}

int ogm_zero_share_trio_fold2(const uint8_t* k1, const uint8_t* k2, const uint8_t* k3, uint64_t counter1,
                              uint64_t counter2, int64_t nbits, int64_t w0, int64_t nwords,
                              const uint32_t* const* xor_into, uint32_t* const* out, void* stream) {
    return zero_share_trio_impl(k1, k2, k3, counter1, nbits, w0, nwords, xor_into, out, stream, 0, 0xffffffffu, 1,
                                counter2, nullptr, nullptr, 1);
}

int ogm_zero_share_trio_slice(const uint8_t* k1, const uint8_t* k2, const uint8_t* k3, uint64_t counter,
                              int64_t nbits, int64_t w0, int64_t nwords, const uint32_t* const* xor_into,
                              uint32_t* const* out, void* stream) {
    return zero_share_trio_impl(k1, k2, k3, counter, nbits, w0, nwords, xor_into, out, stream);
}

int ogm_and_terms(int64_t nwords, int nparty, const uint32_t* const* a_a, const uint32_t* const* a_b,
                  const uint32_t* const* b_a, const uint32_t* const* b_b, uint32_t* const* out, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(nparty >= 1 && nparty <= kMaxParty, OGM_ERR_ARG, "nparty must be 1..3");
    OGM_CHECK_ARG(nwords >= 0, OGM_ERR_ARG, "negative length");
    if (nwords == 0) return OGM_OK;
    AndArgs a{};
    for (int q = 0; q < nparty; q++) {
        a.aa[q] = a_a[q];
        a.ab[q] = a_b[q];
        a.ba[q] = b_a[q];
        a.bb[q] = b_b[q];
        a.out[q] = out[q];
    }
    a.nparty = nparty;
    and_terms_kernel<<<grid_for(nwords), 256, 0, as_stream(stream)>>>(a, nwords);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

int ogm_xor_words(int64_t nwords, const uint32_t* a, const uint32_t* b, const uint32_t* c, uint32_t* out,
                  void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(nwords >= 0, OGM_ERR_ARG, "negative length");
    if (nwords == 0) return OGM_OK;
    xor3_kernel<<<grid_for(nwords), 256, 0, as_stream(stream)>>>(a, b, c, out, nwords);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

int ogm_select_fold(int64_t rows, int64_t words, int64_t pitch, int nparty, const uint32_t* const* A,
                    const uint32_t* const* B, const uint32_t* const* fa, const uint32_t* const* fb,
                    uint32_t* const* out, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(nparty >= 1 && nparty <= kMaxParty, OGM_ERR_ARG, "nparty must be 1..3");
    OGM_CHECK_ARG(rows >= 0 && words >= 0 && pitch >= words, OGM_ERR_ARG, "bad matrix shape");
    cudaStream_t st = as_stream(stream);
    FoldArgs a{};
    for (int q = 0; q < nparty; q++) {
        a.A[q] = A[q];
        a.B[q] = B[q];
        a.fa[q] = fa[q];
        a.fb[q] = fb[q];
        a.out[q] = out[q];
        if (words) OGM_CUDA_TRY(cudaMemsetAsync(out[q], 0, 4 * words, st));
    }
    if (rows == 0 || words == 0) return OGM_OK;
    a.nparty = nparty;
    a.rows = rows;
    a.words = words;
    a.pitch = pitch;
    bool vec = (pitch & 3) == 0 && (nparty == 1 || nparty == 3);
    for (int q = 0; q < nparty && vec; q++) {
        vec = (((uintptr_t)A[q]) & 15) == 0 && (((uintptr_t)B[q]) & 15) == 0;
        if (nparty == 3) vec = vec && B[q] == A[(q + 1) % 3] && fb[q] == fa[(q + 1) % 3];
    }
    if (vec) {
        // ~32K threads' worth of (chunk, row-group) work per SM: many short row
        // strides beat few long ones (access fold at 20K x 40K words: 2048/SM
        // 5.3 TB/s, 16384/SM 6.59, 32768/SM 6.64, 65536/SM 6.53)
        constexpr int RB = 4;
        const int64_t nch = (words + 3) / 4;
        int64_t rgroups = ((int64_t)sm_count() * 32768 + nch - 1) / nch;
        const int64_t rblocks = (rows + RB - 1) / RB;
        // but every row group ends in one atomicXor per output word: for narrow rows
        // (Case I fold, 1024-word rows) that many groups made the fold atomic-bound
        // (200K rows: 2.7 TB/s), so a group walks at least 16 row blocks
        // (never below one resident wave's worth of threads: small folds stay latency-bound)
        const int64_t fill = ((int64_t)sm_count() * 2048 + nch - 1) / nch;
        const int64_t cap16 = std::max(rblocks / 16, fill);
        if (rgroups > cap16) rgroups = cap16;
        if (rgroups > rblocks) rgroups = rblocks;
        if (rgroups < 1) rgroups = 1;
        const int blocks = (int)((nch * rgroups + 255) / 256);
        if (nparty == 3)
            select_fold_vec4_kernel<3, RB><<<blocks, 256, 0, st>>>(a, nch, rgroups);
        else
            select_fold_vec4_kernel<1, RB><<<blocks, 256, 0, st>>>(a, nch, rgroups);
        OGM_LAUNCH_CHECK();
        return OGM_OK;
    }
    int64_t threads_total = words * rows;
    int64_t cap = (int64_t)sm_count() * 2048;
    if (threads_total > cap) threads_total = cap;
    if (threads_total < words) threads_total = words;
    int grid = (int)((threads_total + 255) / 256);
    select_fold_kernel<<<grid, 256, 0, st>>>(a);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

static int pack_launch(int64_t rows, const int32_t* idx, int nsets, const uint32_t* const* flag_bits, int nfields,
                       const uint32_t* const* fields, const int64_t* fpitch, const int64_t* fwidth,
                       const uint32_t* r_mat, uint32_t* out, int64_t opitch, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(nfields >= 0 && nfields <= kMaxFields, OGM_ERR_ARG, "at most %d fields", kMaxFields);
    OGM_CHECK_ARG(nsets >= 1 && nsets <= kMaxSets, OGM_ERR_ARG, "1..%d share sets", kMaxSets);
    OGM_CHECK_ARG(rows >= 0 && opitch >= 0, OGM_ERR_ARG, "negative sizes");
    PackArgs a{};
    int64_t off = flag_bits ? 1 : 0;
    bool vec = true;
    for (int f = 0; f < nfields; f++) {
        OGM_CHECK_ARG(fwidth[f] >= 0, OGM_ERR_ARG, "negative field width");
        a.fwidth[f] = fwidth[f];
        a.foff[f] = off;
        off += fwidth[f];
        for (int s = 0; s < nsets; s++) {
            const uint32_t* p = fields[s * nfields + f];
            const int64_t fp = fpitch[s * nfields + f];
            OGM_CHECK_ARG(fp >= (fwidth[f] + 31) / 32, OGM_ERR_ARG, "field %d pitch below its width", f);
            a.f[s][f] = p;
            a.fpitch[s][f] = fp;
            vec = vec && (((uintptr_t)p) & 15) == 0 && (fp & 3) == 0;
        }
    }
    OGM_CHECK_ARG(opitch >= (off + 31) / 32, OGM_ERR_ARG, "output pitch too small for %lld bits",
                  (long long)off);
    if (rows == 0 || opitch == 0) return OGM_OK;
    OGM_ENSURE_INIT();
    for (int s = 0; s < nsets; s++) {
        a.flag[s] = flag_bits ? flag_bits[s] : nullptr;
        OGM_CHECK_ARG(!flag_bits || a.flag[s], OGM_ERR_ARG, "flag vector %d missing", s);
    }
    a.idx = idx;
    a.nsets = nsets;
    a.nfields = nfields;
    a.vec_fields = vec ? 1 : 0;
    a.r = r_mat;
    a.out = out;
    a.opitch = opitch;
    a.owidth = off;
    a.rows = rows;
    const bool wide = opitch >= 64 && (opitch & 3) == 0 && (((uintptr_t)out | (uintptr_t)r_mat) & 15) == 0;
    if (wide) {
        int64_t g = rows < (int64_t)sm_count() * 8 ? rows : (int64_t)sm_count() * 8;
        const int ns = vec ? nsets : 0;
        const int64_t ng = opitch / 4;
        if (ns > 0 && ng <= kPackTabChunks) {
            auto kern = ns == 1 ? pack_gather_rows_kernel<1, true> : ns == 2 ? pack_gather_rows_kernel<2, true>
                      : pack_gather_rows_kernel<3, true>;
            kern<<<(int)g, 256, (size_t)(ng * 8), as_stream(stream)>>>(a);
        } else {
            auto kern = ns == 1 ? pack_gather_rows_kernel<1> : ns == 2 ? pack_gather_rows_kernel<2>
                      : ns == 3 ? pack_gather_rows_kernel<3> : pack_gather_rows_kernel<0>;
            kern<<<(int)g, 256, 0, as_stream(stream)>>>(a);
        }
    } else {
        pack_gather_kernel<<<grid_for(rows * opitch), 256, 0, as_stream(stream)>>>(a);
    }
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

int ogm_pack_fields(int64_t rows, const uint32_t* flag_bits, int nfields, const uint32_t* const* fields,
                    const int64_t* fpitch, const int64_t* fwidth, uint32_t* out, int64_t opitch,
                    void* stream) {
    const uint32_t* flags[1] = {flag_bits};
    return pack_launch(rows, nullptr, 1, flag_bits ? flags : nullptr, nfields, fields, fpitch, fwidth, nullptr, out,
                       opitch, stream);
}

int ogm_pack_gather(int64_t rows, const int32_t* idx, int nsets, const uint32_t* const* flag_bits, int nfields,
                    const uint32_t* const* fields, const int64_t* fpitch, const int64_t* fwidth,
                    const uint32_t* r_mat, uint32_t* out, int64_t opitch, void* stream) {
    return pack_launch(rows, idx, nsets, flag_bits, nfields, fields, fpitch, fwidth, r_mat, out, opitch, stream);
}

int ogm_extract_field(const uint32_t* src, int64_t spitch, const int32_t* idx, int64_t n, int64_t bit_offset,
                      int64_t width, uint32_t* out, int64_t opitch, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(n >= 0 && width >= 0 && bit_offset >= 0, OGM_ERR_ARG, "bad extract arguments");
    OGM_CHECK_ARG(opitch >= (width + 31) / 32, OGM_ERR_ARG, "output pitch too small");
    if (n == 0 || opitch == 0) return OGM_OK;
    if (opitch >= 256) {
        int64_t g = n < (int64_t)sm_count() * 8 ? n : (int64_t)sm_count() * 8;
        extract_field_rows_kernel<<<(int)g, 256, 0, as_stream(stream)>>>(src, spitch, idx, n, bit_offset, width, out,
                                                                          opitch);
    } else {
        extract_field_kernel<<<grid_for(n * opitch), 256, 0, as_stream(stream)>>>(src, spitch, idx, n, bit_offset,
                                                                                   width, out, opitch);
    }
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

int ogm_mask_row_tails(uint32_t* mat, int64_t rows, int64_t pitch, int64_t width, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(rows >= 0 && width >= 0 && pitch >= (width + 31) / 32, OGM_ERR_ARG, "bad matrix shape");
    if (rows == 0 || (width & 31) == 0) return OGM_OK;
    mask_row_tails_kernel<<<grid_for(rows), 256, 0, as_stream(stream)>>>(mat, rows, pitch, (width + 31) / 32,
                                                                         (1u << (width & 31)) - 1u);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

int ogm_unpack_records(const void* blob, int64_t blob_bytes, int64_t nrec, const int64_t* src_off,
                       const int64_t* dst_off, const int32_t* nwords, uint32_t* arena, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(nrec >= 0 && blob_bytes >= 0, OGM_ERR_ARG, "negative sizes");
    OGM_CHECK_ARG((((uintptr_t)blob) & 3) == 0, OGM_ERR_ARG, "blob must be 4-byte aligned");
    if (nrec == 0) return OGM_OK;
    int64_t g = (nrec + 7) / 8;
    const int64_t cap = (int64_t)sm_count() * 16;
    if (g > cap) g = cap;
    unpack_records_kernel<<<(int)g, 256, 0, as_stream(stream)>>>((const uint32_t*)blob, blob_bytes, nrec, src_off,
                                                                 dst_off, nwords, arena);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

int ogm_column_bits(const uint32_t* mat, int64_t pitch, int64_t rows, uint32_t* out_bits, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(rows >= 0, OGM_ERR_ARG, "negative rows");
    if (rows == 0) return OGM_OK;
    column_bit_kernel<<<grid_for((rows + 31) / 32), 256, 0, as_stream(stream)>>>(mat, pitch, rows, out_bits);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

int64_t ogm_compact_workspace_bytes(int64_t n) { return ogm_keep_rows_workspace_bytes(n); }

// indices of the set bits, in order: the hand-written keep (ogm_fetch.cuh) with no row copies
int ogm_compact_bits(int64_t n, const uint32_t* bits, int32_t* out_idx, int64_t* out_count, void* workspace,
                     int64_t workspace_bytes, void* stream) {
    OGM_CHECK_ARG(n >= 0, OGM_ERR_ARG, "negative length");
    return ogm_keep_rows(n, bits, 0, nullptr, 0, nullptr, 0, out_idx, out_count, workspace, workspace_bytes, stream);
}

int ogm_select_many(int64_t K, int64_t X, int64_t words, int64_t pitch, const uint32_t* sel_a,
                    const uint32_t* sel_b, int64_t spitch, const uint32_t* A, const uint32_t* B, uint32_t* out,
                    int64_t opitch, void* workspace, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(K >= 0 && X >= 0 && words >= 0 && pitch >= words && opitch >= words, OGM_ERR_ARG,
                  "bad select-many shape");
    cudaStream_t st = as_stream(stream);
    if (K == 0) return OGM_OK;
    OGM_CUDA_TRY(cudaMemsetAsync(out, 0, 4 * K * opitch, st));
    if (X == 0 || words == 0) return OGM_OK;
    uint32_t* ta = (uint32_t*)workspace;
    uint32_t* tb = ta + X;
    int64_t threads_total = words * X;
    int64_t cap = (int64_t)sm_count() * 1024;
    if (threads_total > cap) threads_total = cap;
    if (threads_total < words) threads_total = words;
    for (int64_t k0 = 0; k0 < K; k0 += 32) {
        transpose_sel_kernel<<<grid_for(X), 256, 0, st>>>(sel_a, spitch, K, k0, X, ta);
        transpose_sel_kernel<<<grid_for(X), 256, 0, st>>>(sel_b, spitch, K, k0, X, tb);
        const int kn = (int)((K - k0) < 32 ? (K - k0) : 32);
        select_many_kernel<<<(int)((threads_total + 127) / 128), 128, 0, st>>>(ta, tb, A, B, X, words, pitch, kn,
                                                                              out + k0 * opitch, opitch);
    }
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

// Trio fast path: open the flag column of a shuffled three-component table,
// keep the flagged rows in order and slice their fields out (src/engine.py:
// 243-269, 321-334) -- one synchronous call instead of ~12 dispatches.
int64_t ogm_trio_open_keep_workspace_bytes(int64_t rows) {
    const int64_t w = (rows + 31) / 32;
    return ((w * 4 + 255) & ~(int64_t)255) + ((rows * 4 + 255) & ~(int64_t)255) + 256 +
           ogm_compact_workspace_bytes(rows > 0 ? rows : 1);
}

int ogm_trio_open_keep(const uint32_t* const* comps, int64_t rows, int64_t pitch, uint32_t* plain_host, int nfields,
                       const int64_t* bit_off, const int64_t* width, uint32_t* const* out, const int64_t* opitch,
                       int64_t* kept, void* workspace, int64_t workspace_bytes, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(comps && plain_host && kept && rows >= 0 && pitch >= 1 && nfields >= 0, OGM_ERR_ARG,
                  "bad open-keep arguments");
    OGM_CHECK_ARG(workspace_bytes >= ogm_trio_open_keep_workspace_bytes(rows), OGM_ERR_ARG,
                  "open-keep workspace too small");
    *kept = 0;
    if (rows == 0) return OGM_OK;
    OGM_ENSURE_INIT();
    cudaStream_t st = as_stream(stream);
    const int64_t nw = (rows + 31) / 32;
    uint8_t* w = (uint8_t*)workspace;
    uint32_t* plain = (uint32_t*)w;
    w += (nw * 4 + 255) & ~(int64_t)255;
    int32_t* idx = (int32_t*)w;
    w += (rows * 4 + 255) & ~(int64_t)255;
    int64_t* cnt = (int64_t*)w;
    w += 256;
    column_open3_kernel<<<grid_for(nw), 256, 0, st>>>(comps[0], comps[1], comps[2], pitch, rows, plain);
    OGM_LAUNCH_CHECK();
    int rc = ogm_compact_bits(rows, plain, idx, cnt, w, ogm_compact_workspace_bytes(rows), stream);
    if (rc) return rc;
    OGM_CUDA_TRY(cudaMemcpyAsync(plain_host, plain, nw * 4, cudaMemcpyDeviceToHost, st));
    OGM_CUDA_TRY(cudaStreamSynchronize(st));
    int64_t k = 0;
    for (int64_t i = 0; i < nw; i++) k += __builtin_popcount(plain_host[i]);
    *kept = k;
    bool narrow = 3 * nfields <= kMaxExtract;
    for (int f = 0; f < nfields; f++) narrow = narrow && opitch[f] < 256;
    if (narrow && k > 0 && nfields > 0) {
        ExtractJobs J{};
        int64_t most = 0;
        for (int c = 0; c < 3; c++)
            for (int f = 0; f < nfields; f++) {
                J.j[c * nfields + f] = ExtractJob{comps[c], out[c * nfields + f], bit_off[f], width[f], opitch[f]};
                most = std::max(most, k * opitch[f]);
            }
        J.idx = idx;
        J.spitch = pitch;
        J.n = k;
        if (most > 0) {
            extract_field_multi_kernel<<<dim3((unsigned)grid_for(most), (unsigned)(3 * nfields)), 256, 0, st>>>(J);
            OGM_LAUNCH_CHECK();
        }
        return OGM_OK;
    }
    for (int c = 0; c < 3; c++)
        for (int f = 0; f < nfields; f++) {
            rc = ogm_extract_field(comps[c], pitch, idx, k, bit_off[f], width[f], out[c * nfields + f], opitch[f],
                                   stream);
            if (rc) return rc;
        }
    return OGM_OK;
}

}  // extern "C"
