// ogm_aes.cuh -- AES-128 for sm_100a, table-driven from shared memory.
//
// Why tables and not bitslicing: the FSS walk (src/fss.py:257-281) and the
// CTR PRF (src/prf.py:70-92) encrypt independent 16-byte blocks whose round
// keys differ per lane (left/right child key chosen by the point's bit), so
// each thread owns whole blocks.  The design point is one LDS + one PRMT per
// table lookup:
//
//  * 4 T-tables (T_r = rotl(T0, 8r), little-endian column words) are stored
//    32x replicated, one copy per lane/bank, so every lookup is bank-conflict
//    free (the smem crossbar serves one LDS per clock per SM).
//  * Entry e of (T0|T1) lives at  e*256 + {0|128} + lane*4  in region A,
//    (T2|T3) likewise in region B (+64 KiB).  The byte offset of a lookup is
//    therefore [lane*4 (+128), state byte, 0, 0] -- a single PRMT
//    (__byte_perm) of the state word with a per-lane constant -- and the LDS
//    uses [reg + imm] addressing.  128 KiB of shared memory per CTA.
//  * Columns are little-endian words, matching the byte image of the
//    reference's uint64 seeds (src/prf.py:48-53) and of its uint32 share
//    words, so no byte swapping happens on the data path.
//
// Round keys come from a functor `ks(i)` (word i of the 44-word schedule) so
// fixed PRG keys resolve to constant-bank operands and per-lane key choice
// (left vs right child) costs one LOP3 per word.
#pragma once

#include <stdint.h>

namespace ogm {

constexpr int kAesTableBytes = 128 * 1024;
constexpr int kAesRegionB = 64 * 1024;

// Host-computed tables/keys, uploaded by ogm_init().
__constant__ uint32_t c_T0[256];
__constant__ uint32_t c_prg_rk[3][44];  // src/prf.py:26-28: left, right, ctrl
__constant__ uint32_t c_prg_dlr[44];    // rk_left ^ rk_right

__device__ __forceinline__ uint32_t rotl32(uint32_t x, int s) { return __funnelshift_l(x, x, s); }

// Fill the replicated tables.  All threads of the CTA participate; caller
// must __syncthreads() before the first lookup.
__device__ __forceinline__ void aes_fill_tables(uint8_t* smem) {
    uint32_t* w = reinterpret_cast<uint32_t*>(smem);
    for (int idx = threadIdx.x; idx < 4 * 256 * 32; idx += blockDim.x) {
        int lane = idx & 31;
        int e = (idx >> 5) & 255;
        int t = idx >> 13;
        uint32_t v = c_T0[e];
        if (t) v = rotl32(v, 8 * t);
        int byte = (t >> 1) * kAesRegionB + e * 256 + (t & 1) * 128 + lane * 4;
        w[byte >> 2] = v;
    }
}

struct AesTab {
    static constexpr int kBytes = kAesTableBytes;
    __device__ __forceinline__ static void fill(uint8_t* smem) { aes_fill_tables(smem); }
    const uint8_t* base;  // shared-memory table base
    uint32_t off0;        // lane*4
    uint32_t off1;        // lane*4 + 128

    __device__ __forceinline__ explicit AesTab(const uint8_t* smem) : base(smem) {
        uint32_t lane = threadIdx.x & 31;
        off0 = lane * 4;
        off1 = lane * 4 + 128;
    }
    __device__ __forceinline__ uint32_t ld(uint32_t byteoff) const {
        return *reinterpret_cast<const uint32_t*>(base + byteoff);
    }
    // T_TBL[byte POS of x]: region, lane offset and byte position are static.
    template <int TBL, int POS>
    __device__ __forceinline__ uint32_t lut(uint32_t x) const {
        const uint32_t off = (TBL & 1) ? off1 : off0;
        return ld((TBL >> 1) * kAesRegionB + __byte_perm(x, off, 0x5504 | (POS << 4)));
    }
    __device__ __forceinline__ uint32_t t0(uint32_t x) const { return lut<0, 0>(x); }
    __device__ __forceinline__ uint32_t t1(uint32_t x) const { return lut<1, 1>(x); }
    __device__ __forceinline__ uint32_t t2(uint32_t x) const { return lut<2, 2>(x); }
    __device__ __forceinline__ uint32_t t3(uint32_t x) const { return lut<3, 3>(x); }
    // Final-round S-box column: byte r = S[byte r of x_r].  T2[.].b0, T3[.].b1,
    // T0[.].b2 and T1[.].b3 all equal S[.], so four lookups + three PRMTs.
    __device__ __forceinline__ uint32_t sub_col(uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3) const {
        uint32_t a = lut<2, 0>(x0), b = lut<3, 1>(x1), c = lut<0, 2>(x2), d = lut<1, 3>(x3);
        return __byte_perm(__byte_perm(a, b, 0x3250), __byte_perm(c, d, 0x7210), 0x7610);
    }
    // S[byte 0 of x] in the low byte (upper bytes are garbage).
    __device__ __forceinline__ uint32_t sub_b0(uint32_t x) const { return lut<2, 0>(x); }
};


// Small-work variant: the four T-tables once (4 KiB, no per-lane
// replication).  Lookups may bank-conflict (random bytes over 32 banks, ~3-4
// wavefronts), but the fill is 1024 words instead of 32768 -- for launches
// with a few thousand AES blocks (tokens, C1-sized shuffles, small domains)
// the replicated fill IS the kernel: 4 CTAs x 512 threads spent 22-35 us
// filling 128 KiB each (ncu, profiles/r01_c1_small_aes.md).
constexpr int kAesSmallBytes = 4 * 1024;

struct AesTabSmall {
    static constexpr int kBytes = kAesSmallBytes;
    __device__ __forceinline__ static void fill(uint8_t* smem) {
        uint32_t* w = reinterpret_cast<uint32_t*>(smem);
        for (int idx = threadIdx.x; idx < 1024; idx += blockDim.x) {
            const int t = idx >> 8, e = idx & 255;
            uint32_t v = c_T0[e];
            if (t) v = rotl32(v, 8 * t);
            w[idx] = v;
        }
    }
    const uint32_t* base;
    __device__ __forceinline__ explicit AesTabSmall(const uint8_t* smem)
        : base(reinterpret_cast<const uint32_t*>(smem)) {}
    template <int TBL, int POS>
    __device__ __forceinline__ uint32_t lut(uint32_t x) const {
        return base[TBL * 256 + ((x >> (8 * POS)) & 255u)];
    }
    __device__ __forceinline__ uint32_t t0(uint32_t x) const { return lut<0, 0>(x); }
    __device__ __forceinline__ uint32_t t1(uint32_t x) const { return lut<1, 1>(x); }
    __device__ __forceinline__ uint32_t t2(uint32_t x) const { return lut<2, 2>(x); }
    __device__ __forceinline__ uint32_t t3(uint32_t x) const { return lut<3, 3>(x); }
    __device__ __forceinline__ uint32_t sub_col(uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3) const {
        uint32_t a = lut<2, 0>(x0), b = lut<3, 1>(x1), c = lut<0, 2>(x2), d = lut<1, 3>(x3);
        return __byte_perm(__byte_perm(a, b, 0x3250), __byte_perm(c, d, 0x7210), 0x7610);
    }
    __device__ __forceinline__ uint32_t sub_b0(uint32_t x) const { return lut<2, 0>(x); }
};

__device__ __forceinline__ uint32_t xor5(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t e) {
    return a ^ b ^ c ^ d ^ e;
}

// Round-key functors -------------------------------------------------------

template <int K>
struct PrgKey {  // fixed PRG key K (0 left, 1 right, 2 ctrl)
    __device__ __forceinline__ uint32_t operator()(int i) const { return c_prg_rk[K][i]; }
};

struct PrgChildKey {  // left (m = 0) or right (m = ~0) child key, per lane
    uint32_t m;
    __device__ __forceinline__ uint32_t operator()(int i) const { return c_prg_rk[0][i] ^ (c_prg_dlr[i] & m); }
};

struct ParamKey {  // schedule passed by value in the kernel parameter space
    const uint32_t* rk;
    __device__ __forceinline__ uint32_t operator()(int i) const { return rk[i]; }
};

struct AesKeySched {
    uint32_t rk[44];
};

// Full AES-128 encryption of one block (4 LE column words).
template <class TAB, class KS>
__device__ __forceinline__ uint4 aes128_enc(const TAB& T, uint4 in, const KS& ks) {
    uint32_t s0 = in.x ^ ks(0), s1 = in.y ^ ks(1), s2 = in.z ^ ks(2), s3 = in.w ^ ks(3);
#pragma unroll
    for (int r = 1; r < 10; r++) {
        uint32_t n0 = xor5(T.t0(s0), T.t1(s1), T.t2(s2), T.t3(s3), ks(4 * r + 0));
        uint32_t n1 = xor5(T.t0(s1), T.t1(s2), T.t2(s3), T.t3(s0), ks(4 * r + 1));
        uint32_t n2 = xor5(T.t0(s2), T.t1(s3), T.t2(s0), T.t3(s1), ks(4 * r + 2));
        uint32_t n3 = xor5(T.t0(s3), T.t1(s0), T.t2(s1), T.t3(s2), ks(4 * r + 3));
        s0 = n0; s1 = n1; s2 = n2; s3 = n3;
    }
    // final round: SubBytes + ShiftRows + AddRoundKey; byte r of column j
    // comes from column j+r.  Pick the table whose byte r holds S[x].
    uint4 o;
    o.x = T.sub_col(s0, s1, s2, s3) ^ ks(40);
    o.y = T.sub_col(s1, s2, s3, s0) ^ ks(41);
    o.z = T.sub_col(s2, s3, s0, s1) ^ ks(42);
    o.w = T.sub_col(s3, s0, s1, s2) ^ ks(43);
    return o;
}

// Only byte 0 of the ciphertext under the fixed control key: rounds 1-8 in
// full, column 0 of round 9, one S-box lookup in round 10 (133 lookups
// instead of 160).  Returns the three PRG control/value bits
// (src/prf.py:53-56): bit0 t_left, bit1 t_right, bit2 value.
template <class TAB>
__device__ __forceinline__ uint32_t prg_ctrl_bits(const TAB& T, uint4 s) {
    PrgKey<2> ks;
    uint32_t s0 = s.x ^ ks(0), s1 = s.y ^ ks(1), s2 = s.z ^ ks(2), s3 = s.w ^ ks(3);
#pragma unroll
    for (int r = 1; r < 9; r++) {
        uint32_t n0 = xor5(T.t0(s0), T.t1(s1), T.t2(s2), T.t3(s3), ks(4 * r + 0));
        uint32_t n1 = xor5(T.t0(s1), T.t1(s2), T.t2(s3), T.t3(s0), ks(4 * r + 1));
        uint32_t n2 = xor5(T.t0(s2), T.t1(s3), T.t2(s0), T.t3(s1), ks(4 * r + 2));
        uint32_t n3 = xor5(T.t0(s3), T.t1(s0), T.t2(s1), T.t3(s2), ks(4 * r + 3));
        s0 = n0; s1 = n1; s2 = n2; s3 = n3;
    }
    uint32_t c0 = xor5(T.t0(s0), T.t1(s1), T.t2(s2), T.t3(s3), ks(36));
    return (T.sub_b0(c0) ^ ks(40) ^ s.x) & 7u;
}

// Small-work builds: one out-of-line, rolled AES per kernel instead of an
// unrolled copy per call site.  A C1-sized shuffle launch spent 155 of 212
// PC samples in "no instruction" (i-cache misses over ~50 KB of unrolled
// rounds on 16 cold SMs) -- code size, not arithmetic, was its runtime.
template <class KS>
__device__ __noinline__ uint4 aes128_enc_rolled(const AesTabSmall T, uint4 in, const KS ks) {
    uint32_t s0 = in.x ^ ks(0), s1 = in.y ^ ks(1), s2 = in.z ^ ks(2), s3 = in.w ^ ks(3);
#pragma unroll 1
    for (int r = 1; r < 10; r++) {
        uint32_t n0 = xor5(T.t0(s0), T.t1(s1), T.t2(s2), T.t3(s3), ks(4 * r + 0));
        uint32_t n1 = xor5(T.t0(s1), T.t1(s2), T.t2(s3), T.t3(s0), ks(4 * r + 1));
        uint32_t n2 = xor5(T.t0(s2), T.t1(s3), T.t2(s0), T.t3(s1), ks(4 * r + 2));
        uint32_t n3 = xor5(T.t0(s3), T.t1(s0), T.t2(s1), T.t3(s2), ks(4 * r + 3));
        s0 = n0; s1 = n1; s2 = n2; s3 = n3;
    }
    uint4 o;
    o.x = T.sub_col(s0, s1, s2, s3) ^ ks(40);
    o.y = T.sub_col(s1, s2, s3, s0) ^ ks(41);
    o.z = T.sub_col(s2, s3, s0, s1) ^ ks(42);
    o.w = T.sub_col(s3, s0, s1, s2) ^ ks(43);
    return o;
}

template <class KS>
__device__ __forceinline__ uint4 aes128_enc(const AesTabSmall& T, uint4 in, const KS& ks) {
    return aes128_enc_rolled(T, in, ks);
}

__device__ __noinline__ uint32_t prg_ctrl_bits_rolled(const AesTabSmall T, uint4 s) {
    PrgKey<2> ks;
    uint32_t s0 = s.x ^ ks(0), s1 = s.y ^ ks(1), s2 = s.z ^ ks(2), s3 = s.w ^ ks(3);
#pragma unroll 1
    for (int r = 1; r < 9; r++) {
        uint32_t n0 = xor5(T.t0(s0), T.t1(s1), T.t2(s2), T.t3(s3), ks(4 * r + 0));
        uint32_t n1 = xor5(T.t0(s1), T.t1(s2), T.t2(s3), T.t3(s0), ks(4 * r + 1));
        uint32_t n2 = xor5(T.t0(s2), T.t1(s3), T.t2(s0), T.t3(s1), ks(4 * r + 2));
        uint32_t n3 = xor5(T.t0(s3), T.t1(s0), T.t2(s1), T.t3(s2), ks(4 * r + 3));
        s0 = n0; s1 = n1; s2 = n2; s3 = n3;
    }
    uint32_t c0 = xor5(T.t0(s0), T.t1(s1), T.t2(s2), T.t3(s3), ks(36));
    return (T.sub_b0(c0) ^ ks(40) ^ s.x) & 7u;
}

__device__ __forceinline__ uint32_t prg_ctrl_bits(const AesTabSmall& T, uint4 s) { return prg_ctrl_bits_rolled(T, s); }

// Matyas-Meyer-Oseas child seed: AES_K(s) ^ s (src/prf.py:51-52).
template <class TAB, class KS>
__device__ __forceinline__ uint4 prg_child(const TAB& T, uint4 s, const KS& ks) {
    uint4 c = aes128_enc(T, s, ks);
    return make_uint4(c.x ^ s.x, c.y ^ s.y, c.z ^ s.z, c.w ^ s.w);
}

__device__ __forceinline__ uint4 xor4(uint4 a, uint4 b) {
    return make_uint4(a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w);
}
__device__ __forceinline__ uint4 and4(uint4 a, uint32_t m) {
    return make_uint4(a.x & m, a.y & m, a.z & m, a.w & m);
}

// CTR counter block (src/prf.py:82-84): the big-endian 128-bit integer
// label(4) || index(8, BE) || 0(4), plus `blk`, as LE column words.
__device__ __forceinline__ uint4 ctr_block(uint32_t label_be, uint64_t index, uint64_t blk) {
    uint64_t hi = ((uint64_t)label_be << 32) | (index >> 32);
    uint64_t lo = index << 32;
    uint64_t nlo = lo + blk;
    hi += (nlo < lo) ? 1 : 0;
    return make_uint4(__byte_perm((uint32_t)(hi >> 32), 0, 0x0123), __byte_perm((uint32_t)hi, 0, 0x0123),
                      __byte_perm((uint32_t)(nlo >> 32), 0, 0x0123), __byte_perm((uint32_t)nlo, 0, 0x0123));
}

}  // namespace ogm
