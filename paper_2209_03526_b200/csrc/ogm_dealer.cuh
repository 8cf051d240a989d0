// ogm_dealer.cuh -- graph outsourcing straight into device memory
// (src/graphs.py:327-400, encrypt_graph / _share_matrix).
//
// The reference draws every random share component from numpy's default
// generator: PCG64 (128-bit LCG, XSL-RR output), read through
// Generator.integers(0, 2^32, dtype=uint32), which returns the low then the
// high half of each 64-bit output (the high half buffered across calls).
// PCG64 is an LCG, so its state after k steps is a closed form (jump-ahead in
// O(log k) 128-bit multiplies): any thread can start anywhere in the stream.
// So the dealer draws the exact uint32 stream the reference would draw, on
// the device, and builds the three XOR share components of one-hot rows in
// place -- the same bytes as the host dealer, without a host-side pass or a
// PCIe copy of the 3x-expanded shares.
#pragma once

#include "ogm_common.cuh"

namespace ogm {

typedef unsigned __int128 u128;

__host__ __device__ constexpr u128 pcg64_mult() {
    return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}

// state after `delta` more LCG steps: s' = A^delta s + (A^(delta-1) + ... + 1) inc
__device__ __forceinline__ u128 pcg64_advance(u128 s, u128 inc, uint64_t delta) {
    u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg64_mult(), cur_plus = inc;
    while (delta) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return acc_mult * s + acc_plus;
}

// the same jump as a (multiplier, increment) pair, for a fixed stride
__device__ __forceinline__ void pcg64_jump(u128 inc, uint64_t delta, u128* mult, u128* plus) {
    u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg64_mult(), cur_plus = inc;
    while (delta) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    *mult = acc_mult;
    *plus = acc_plus;
}

__device__ __forceinline__ uint64_t pcg64_output(u128 s) {  // XSL-RR
    const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
    const unsigned rot = (unsigned)(s >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

// u32 stream elements [0, n) from a generator at (s0, inc) with the numpy
// buffer (has_u32, buffered): element 0 is the buffered high half when
// has_u32, then each 64-bit output contributes its low, then its high half.
// Lane l of a warp owns outputs base + l + 32 r: every step writes 32
// consecutive outputs (coalesced), and a lane moves on by one 32-step jump.
constexpr int kPcgRounds = 32;

__global__ void __launch_bounds__(256) pcg64_u32_kernel(uint64_t s_lo, uint64_t s_hi, uint64_t inc_lo,
                                                        uint64_t inc_hi, int has_u32, uint32_t buffered, int64_t n,
                                                        uint32_t* __restrict__ out) {
    const u128 s0 = ((u128)s_hi << 64) | s_lo, inc = ((u128)inc_hi << 64) | inc_lo;
    const int64_t b = has_u32 ? 1 : 0;
    if (b && blockIdx.x == 0 && threadIdx.x == 0 && n > 0) out[0] = buffered;
    const int64_t outputs = (n - b + 1) / 2;   // 64-bit outputs needed
    if (outputs <= 0) return;
    u128 jm, jp;
    pcg64_jump(inc, 32, &jm, &jp);
    const int64_t per_warp = 32 * kPcgRounds;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    const int lane = threadIdx.x & 31;
    for (int64_t wbase = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32 * per_warp; wbase < outputs;
         wbase += warps * per_warp) {
        int64_t j = wbase + lane;
        u128 s = pcg64_advance(s0, inc, (uint64_t)j + 1);   // output j is taken after j + 1 steps
        for (int r = 0; r < kPcgRounds && wbase + 32 * r < outputs; r++, j += 32) {
            if (j < outputs) {
                const uint64_t o = pcg64_output(s);
                const int64_t e = b + 2 * j;
                out[e] = (uint32_t)o;
                if (e + 1 < n) out[e + 1] = (uint32_t)(o >> 32);
            }
            s = jm * s + jp;
        }
    }
}

// The three share components of drawn rows (src/graphs.py:327-332, before
// the plaintext is folded in): row i holds drawn[i] words drawn as its
// first component at S[s1_off[i]..] and drawn[i] more as its second at
// S[s2_off[i]..]; c3 = c1 ^ c2; every word from drawn[i] to the row pitch is
// zero (k-padding slots and the 16-byte row padding).  The plaintext one-hot
// bits are XORed into c3 afterwards (ogm_deal_hot_bits).
__global__ void __launch_bounds__(256) deal_rows_kernel(const uint32_t* __restrict__ S,
                                                        const int64_t* __restrict__ s1_off,
                                                        const int64_t* __restrict__ s2_off,
                                                        const int64_t* __restrict__ drawn, int64_t rows,
                                                        int64_t pitch, uint32_t* __restrict__ c1,
                                                        uint32_t* __restrict__ c2, uint32_t* __restrict__ c3) {
    const int64_t total = rows * pitch;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
        const int64_t i = e / pitch, c = e - i * pitch;
        uint32_t a = 0, b = 0;
        if (c < __ldg(drawn + i)) {
            a = __ldg(S + __ldg(s1_off + i) + c);
            b = __ldg(S + __ldg(s2_off + i) + c);
        }
        c1[e] = a;
        c2[e] = b;
        c3[e] = a ^ b;
    }
}

// c3[word[j]] ^= mask[j]: the plaintext one-hot bits (distinct words)
__global__ void __launch_bounds__(256) deal_hot_bits_kernel(const int64_t* __restrict__ word,
                                                            const uint32_t* __restrict__ mask, int64_t n,
                                                            uint32_t* __restrict__ c3) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride)
        c3[__ldg(word + j)] ^= __ldg(mask + j);
}

}  // namespace ogm

extern "C" {

int ogm_pcg64_u32(const uint64_t* state, const uint64_t* inc, int has_uint32, uint32_t uinteger, int64_t n,
                  uint32_t* out, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(state && inc && n >= 0, OGM_ERR_ARG, "state, inc and a non-negative count are required");
    OGM_CHECK_ARG(n == 0 || out, OGM_ERR_ARG, "output is required");
    if (n == 0) return OGM_OK;
    const int64_t outputs = (n + 1) / 2 + 1;
    const int64_t per_block = 8 * 32 * kPcgRounds;
    const int64_t g = std::max<int64_t>(1, std::min<int64_t>((outputs + per_block - 1) / per_block,
                                                             (int64_t)sm_count() * 8));
    pcg64_u32_kernel<<<(int)g, 256, 0, as_stream(stream)>>>(state[0], state[1], inc[0], inc[1], has_uint32,
                                                             uinteger, n, out);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

int ogm_deal_rows(const uint32_t* words, const int64_t* s1_off, const int64_t* s2_off, const int64_t* drawn,
                  int64_t rows, int64_t pitch, uint32_t* c1, uint32_t* c2, uint32_t* c3, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(rows >= 0 && pitch >= 0, OGM_ERR_ARG, "bad share matrix shape");
    if (rows == 0 || pitch == 0) return OGM_OK;
    OGM_CHECK_ARG(s1_off && s2_off && drawn && c1 && c2 && c3, OGM_ERR_ARG, "offsets, lengths and outputs are required");
    const int64_t total = rows * pitch;
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 16));
    deal_rows_kernel<<<g, 256, 0, as_stream(stream)>>>(words, s1_off, s2_off, drawn, rows, pitch, c1, c2, c3);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

int ogm_deal_hot_bits(const int64_t* word, const uint32_t* mask, int64_t n, uint32_t* c3, void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(n >= 0, OGM_ERR_ARG, "negative count");
    if (n == 0) return OGM_OK;
    OGM_CHECK_ARG(word && mask && c3, OGM_ERR_ARG, "word indices, masks and output are required");
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 16));
    deal_hot_bits_kernel<<<g, 256, 0, as_stream(stream)>>>(word, mask, n, c3);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

}  // extern "C"
