// ogm_host.cuh -- host-side helpers shared by every subsystem's C-ABI
// wrappers: error state, AES tables / key schedules (computed on the host
// from the AES definition), per-device init, launch geometry.
#pragma once

#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <mutex>

#include "oblivgm_b200.h"
#include "ogm_aes.cuh"
#include "ogm_common.cuh"

namespace ogm {

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}
const char* get_error() { return g_err; }

// ---------------------------------------------------------------------------
// host AES helpers: S-box from its definition (GF(2^8) inverse by
// exponentiation x^254, then the affine map), T0, key schedule.
// ---------------------------------------------------------------------------
static uint8_t gmul(uint8_t a, uint8_t b) {
    uint8_t p = 0;
    while (b) {
        if (b & 1) p ^= a;
        a = (uint8_t)((a << 1) ^ ((a & 0x80) ? 0x1B : 0));
        b >>= 1;
    }
    return p;
}

struct HostAes {
    uint8_t sbox[256];
    uint32_t t0[256];
    HostAes() {
        for (int x = 0; x < 256; x++) {
            uint8_t inv = 0;
            if (x) {  // x^254 = x^-1
                uint8_t r = 1, b = (uint8_t)x;
                int e = 254;
                while (e) {
                    if (e & 1) r = gmul(r, b);
                    b = gmul(b, b);
                    e >>= 1;
                }
                inv = r;
            }
            uint8_t s = inv;
            uint8_t y = s;
            for (int i = 1; i <= 4; i++) y ^= (uint8_t)((s << i) | (s >> (8 - i)));
            sbox[x] = (uint8_t)(y ^ 0x63);
        }
        for (int x = 0; x < 256; x++) {
            uint8_t s = sbox[x];
            uint8_t s2 = gmul(s, 2), s3 = gmul(s, 3);
            t0[x] = (uint32_t)s2 | ((uint32_t)s << 8) | ((uint32_t)s << 16) | ((uint32_t)s3 << 24);
        }
    }
    void expand(const uint8_t key[16], uint32_t rk[44]) const {
        uint8_t rcon = 1;
        for (int i = 0; i < 4; i++)
            rk[i] = (uint32_t)key[4 * i] | ((uint32_t)key[4 * i + 1] << 8) |
                    ((uint32_t)key[4 * i + 2] << 16) | ((uint32_t)key[4 * i + 3] << 24);
        for (int i = 4; i < 44; i++) {
            uint32_t t = rk[i - 1];
            if (i % 4 == 0) {
                t = (t >> 8) | (t << 24);
                t = (uint32_t)sbox[t & 0xff] | ((uint32_t)sbox[(t >> 8) & 0xff] << 8) |
                    ((uint32_t)sbox[(t >> 16) & 0xff] << 16) | ((uint32_t)sbox[t >> 24] << 24);
                t ^= rcon;
                rcon = gmul(rcon, 2);
            }
            rk[i] = rk[i - 4] ^ t;
        }
    }
};

static const HostAes& host_aes() {
    static HostAes h;
    return h;
}

static AesKeySched make_sched(const uint8_t* key) {
    AesKeySched s;
    host_aes().expand(key, s.rk);
    return s;
}

static uint32_t label_be(const uint8_t* label) {
    return ((uint32_t)label[0] << 24) | ((uint32_t)label[1] << 16) | ((uint32_t)label[2] << 8) | label[3];
}

// src/prf.py:26-28: the three fixed public PRG keys.
static const uint8_t kPrgKeys[3][16] = {
    {0x24, 0x3f, 0x6a, 0x88, 0x85, 0xa3, 0x08, 0xd3, 0x13, 0x19, 0x8a, 0x2e, 0x03, 0x70, 0x73, 0x44},
    {0xa4, 0x09, 0x38, 0x22, 0x29, 0x9f, 0x31, 0xd0, 0x08, 0x2e, 0xfa, 0x98, 0xec, 0x4e, 0x6c, 0x89},
    {0x45, 0x28, 0x21, 0xe6, 0x38, 0xd0, 0x13, 0x77, 0xbe, 0x54, 0x66, 0xcf, 0x34, 0xe9, 0x0c, 0x6c},
};

static std::mutex g_init_mu;
static bool g_dev_ready[64];

template <class KernelT>
static cudaError_t allow_big_smem(KernelT k, int bytes) {
    return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

// Gather kernels with no shared memory: ask for the maximum L1 carveout, or
// they inherit whatever split the previous kernel left on the SM (a
// shared-memory-heavy kernel leaves a small L1, which starves a random-row
// gather of in-flight misses: measured 2.26 -> 5.5 ms, profiles/r01_c5_plan.md).
template <class KernelT>
static cudaError_t prefer_l1(KernelT k) {
    return cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
}

int fss_init();
int engine_init();
int shuffle_init();

static int device_init() {
    int dev = 0;
    OGM_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 64 && g_dev_ready[dev]) return OGM_OK;
    std::lock_guard<std::mutex> lk(g_init_mu);
    if (dev < 64 && g_dev_ready[dev]) return OGM_OK;
    const HostAes& h = host_aes();
    uint32_t rk[3][44], dlr[44];
    for (int k = 0; k < 3; k++) h.expand(kPrgKeys[k], rk[k]);
    for (int i = 0; i < 44; i++) dlr[i] = rk[0][i] ^ rk[1][i];
    OGM_CUDA_TRY(cudaMemcpyToSymbol(c_T0, h.t0, sizeof h.t0));
    OGM_CUDA_TRY(cudaMemcpyToSymbol(c_prg_rk, rk, sizeof rk));
    OGM_CUDA_TRY(cudaMemcpyToSymbol(c_prg_dlr, dlr, sizeof dlr));
    // Random 16-byte row gathers (shuffle) otherwise pull a whole 128-byte
    // line per miss; streaming kernels request full lines anyway.
    size_t gran = 0;
    if (cudaDeviceGetLimit(&gran, cudaLimitMaxL2FetchGranularity) == cudaSuccess && gran > 32)
        OGM_CUDA_TRY(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, 32));
    int rc = fss_init();
    if (rc) return rc;
    rc = engine_init();
    if (rc) return rc;
    rc = shuffle_init();
    if (rc) return rc;
    if (dev < 64) g_dev_ready[dev] = true;
    return OGM_OK;
}

#define OGM_ENSURE_INIT()          \
    do {                           \
        int _rc = ::ogm::device_init();   \
        if (_rc) return _rc;       \
    } while (0)

constexpr int kAesThreads = 512;

// grid for the table-driven kernels: one CTA per SM, never more than the work
static int aes_grid(int64_t work_threads) {
    int64_t need = (work_threads + kAesThreads - 1) / kAesThreads;
    int64_t g = sm_count();
    if (need < g) g = need > 0 ? need : 1;
    return (int)g;
}

// AES-table kernels come in two builds: replicated 128 KiB tables (one CTA
// per SM, conflict-free lookups: the throughput path) and 4 KiB tables
// (AesTabSmall: cheap fill, some bank conflicts) for launches whose whole
// work is a few hundred CTAs' worth of 128-thread blocks, where the 32768-word
// replicated fill dominates.  Same arguments, same results.
constexpr int kAesSmallThreads = 128;
constexpr int64_t kAesSmallMaxWork = 32768;

template <class KB, class KS, class... Args>
static void aes_launch(KB big, KS small, int64_t work, int big_threads, cudaStream_t st, Args... args) {
    if (work <= kAesSmallMaxWork) {
        const int64_t g = (work + kAesSmallThreads - 1) / kAesSmallThreads;
        small<<<(int)(g > 0 ? g : 1), kAesSmallThreads, kAesSmallBytes, st>>>(args...);
    } else {
        big<<<aes_grid(work), big_threads, kAesTableBytes, st>>>(args...);
    }
}

// ---- shared-memory / mbarrier / bulk-copy (TMA) helpers -----------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

}  // namespace ogm
