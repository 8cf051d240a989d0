// ogm_lib.cu -- libogm_b200.so: the C ABI declared in include/oblivgm_b200.h.
//
// Single translation unit (the kernels live in the included .cuh files) so
// the __constant__ AES tables need no relocatable device code.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <mutex>
#include <vector>

#include "oblivgm_b200.h"
#include "ogm_host.cuh"
#include "ogm_fss.cuh"
#include "ogm_engine.cuh"
#include "ogm_shuffle.cuh"
#include "ogm_fetch.cuh"
#include "ogm_dealer.cuh"
#include "ogm_trio.cuh"
#include "ogm_measure.cuh"


using namespace ogm;

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* ogm_last_error(void) { return get_error(); }
int ogm_abi_version(void) { return 3; }
int ogm_init(void) { return device_init(); }

int ogm_prg_expand(const void* seeds, int64_t n, void* left, void* right, uint8_t* t_left,
                   uint8_t* t_right, uint8_t* value, void* stream) {
    OGM_CHECK_ARG(n >= 0, OGM_ERR_ARG, "negative seed count");
    if (n == 0) return OGM_OK;
    OGM_ENSURE_INIT();
    prg_expand_kernel<<<aes_grid(n), kFssThreads, kAesTableBytes, as_stream(stream)>>>(
        (const uint4*)seeds, n, (uint4*)left, (uint4*)right, t_left, t_right, value);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

int ogm_prf_words(const uint8_t* key, const uint8_t* label, uint64_t index, uint64_t first_word,
                  int64_t nwords, uint32_t* out, void* stream) {
    OGM_CHECK_ARG(key && label, OGM_ERR_ARG, "PRF key and label are required");
    OGM_CHECK_ARG(nwords >= 0, OGM_ERR_ARG, "negative word count");
    if (nwords == 0) return OGM_OK;
    OGM_ENSURE_INIT();
    AesKeySched k = make_sched(key);
    int64_t nblk = (int64_t)(((first_word + nwords + 3) >> 2) - (first_word >> 2));
    aes_launch(prf_words_kernel<false, AesTab>, prf_words_kernel<false, AesTabSmall>, nblk, kFssThreads,
               as_stream(stream), k, k, label_be(label), index, first_word, nwords, nwords * 32,
               (const uint32_t*)nullptr, out);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

int ogm_prf_rows(const uint8_t* key, const uint8_t* label, uint64_t index, int64_t rows, int64_t width_bits,
                 int64_t pitch, uint32_t* out, void* stream) {
    OGM_CHECK_ARG(key && label && out, OGM_ERR_ARG, "PRF key, label and output are required");
    OGM_CHECK_ARG(rows >= 0 && width_bits >= 0, OGM_ERR_ARG, "negative table shape");
    const int64_t W = (width_bits + 31) / 32;
    OGM_CHECK_ARG(pitch >= W, OGM_ERR_ARG, "pitch %lld below %lld words", (long long)pitch, (long long)W);
    if (rows == 0 || W == 0) return OGM_OK;
    OGM_ENSURE_INIT();
    AesKeySched k = make_sched(key);
    const uint32_t tail = (width_bits & 31) ? ((1u << (width_bits & 31)) - 1u) : 0xffffffffu;
    aes_launch(prf_rows_kernel<AesTab>, prf_rows_kernel<AesTabSmall>, (rows * W + 3) / 4, kFssThreads,
               as_stream(stream), k, label_be(label), index, rows, W, tail, pitch, out);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

int ogm_zero_share(const uint8_t* key_own, const uint8_t* key_prev, uint64_t counter, int64_t nbits,
                   const uint32_t* xor_into, uint32_t* out, void* stream) {
    OGM_CHECK_ARG(key_own && key_prev, OGM_ERR_ARG, "zero-share keys are required");
    OGM_CHECK_ARG(nbits >= 0, OGM_ERR_ARG, "negative bit count");
    if (nbits == 0) return OGM_OK;
    OGM_ENSURE_INIT();
    static const uint8_t kZshr[4] = {'Z', 'S', 'H', 'R'};  // src/rss.py:141
    AesKeySched k1 = make_sched(key_own), k2 = make_sched(key_prev);
    int64_t nwords = (nbits + 31) / 32;
    aes_launch(prf_words_kernel<true, AesTab>, prf_words_kernel<true, AesTabSmall>, (nwords + 3) / 4,
               kFssThreads, as_stream(stream), k1, k2, label_be(kZshr), counter, (uint64_t)0, nwords, nbits,
               xor_into, out);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

int ogm_zero_share_slice(const uint8_t* key_own, const uint8_t* key_prev, uint64_t counter, int64_t total_nbits,
                         uint64_t first_word, int64_t nwords, const uint32_t* xor_into, uint32_t* out,
                         void* stream) {
    OGM_CHECK_ARG(key_own && key_prev, OGM_ERR_ARG, "zero-share keys are required");
    OGM_CHECK_ARG(total_nbits >= 0 && nwords >= 0, OGM_ERR_ARG, "negative length");
    OGM_CHECK_ARG((int64_t)first_word + nwords <= (total_nbits + 31) / 32, OGM_ERR_ARG,
                  "slice [%llu, +%lld) outside the %lld-bit share", (unsigned long long)first_word,
                  (long long)nwords, (long long)total_nbits);
    if (nwords == 0) return OGM_OK;
    OGM_ENSURE_INIT();
    static const uint8_t kZshr[4] = {'Z', 'S', 'H', 'R'};
    AesKeySched k1 = make_sched(key_own), k2 = make_sched(key_prev);
    int64_t nblk = (int64_t)(((first_word + nwords + 3) >> 2) - (first_word >> 2));
    aes_launch(prf_words_kernel<true, AesTab>, prf_words_kernel<true, AesTabSmall>, nblk, kFssThreads,
               as_stream(stream), k1, k2, label_be(kZshr), counter, first_word, nwords, total_nbits, xor_into,
               out);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

static int fss_gen_impl(int kind, int bits, int64_t K, const uint32_t* alphas, const void* roots0,
                        const void* roots1, void* seed_cw, uint32_t* ctrl, uint8_t* out0, uint8_t* out1,
                        void* stream) {
    OGM_CHECK_ARG(kind == OGM_KIND_DPF || kind == OGM_KIND_DCF, OGM_ERR_ARG, "unknown key kind %d", kind);
    OGM_CHECK_ARG(bits >= 1 && bits <= 32, OGM_ERR_DOMAIN, "domain_bits %d outside 1..32", bits);
    OGM_CHECK_ARG(K >= 0, OGM_ERR_ARG, "negative key count");
    if (K == 0) return OGM_OK;
    OGM_ENSURE_INIT();
    if (kind == OGM_KIND_DCF)
        aes_launch(fss_gen_kernel<true, AesTab>, fss_gen_kernel<true, AesTabSmall>, K, kFssThreads, as_stream(stream),
                   bits, K, alphas, (const uint4*)roots0, (const uint4*)roots1, (uint4*)seed_cw, ctrl, out0, out1);
    else
        aes_launch(fss_gen_kernel<false, AesTab>, fss_gen_kernel<false, AesTabSmall>, K, kFssThreads,
                   as_stream(stream), bits, K, alphas, (const uint4*)roots0, (const uint4*)roots1, (uint4*)seed_cw,
                   ctrl, out0, out1);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

int ogm_fss_gen(int kind, int bits, int64_t K, const uint32_t* alphas, const void* roots0,
                const void* roots1, void* seed_cw, uint32_t* ctrl, uint8_t* final_cw, void* stream) {
    return fss_gen_impl(kind, bits, K, alphas, roots0, roots1, seed_cw, ctrl, final_cw, nullptr, stream);
}

int ogm_fss_gen_pair(int kind, int bits, int64_t K, const uint32_t* alphas, const void* roots0,
                     const void* roots1, void* seed_cw, uint32_t* ctrl, uint8_t* flags0, uint8_t* flags1,
                     void* stream) {
    OGM_CHECK_ARG(K == 0 || (flags0 && flags1), OGM_ERR_ARG, "both parties' flag outputs are required");
    return fss_gen_impl(kind, bits, K, alphas, roots0, roots1, seed_cw, ctrl, flags0, flags1, stream);
}

int ogm_fss_eval_points(int kind, int bits, int64_t K, const void* root, const void* seed_cw,
                        const uint32_t* ctrl, const uint8_t* flags, const uint32_t* points,
                        uint32_t* out_bits, void* stream) {
    OGM_CHECK_ARG(kind == OGM_KIND_DPF || kind == OGM_KIND_DCF, OGM_ERR_ARG, "unknown key kind %d", kind);
    OGM_CHECK_ARG(bits >= 1 && bits <= 32, OGM_ERR_DOMAIN, "domain_bits %d outside 1..32", bits);
    OGM_CHECK_ARG(K >= 0, OGM_ERR_ARG, "negative key count");
    if (K == 0) return OGM_OK;
    OGM_ENSURE_INIT();
    if (kind == OGM_KIND_DCF)
        fss_eval_kernel<true><<<aes_grid(K), kFssThreads, kAesTableBytes, as_stream(stream)>>>(
            bits, K, (const uint4*)root, (const uint4*)seed_cw, ctrl, flags, points, out_bits);
    else
        fss_eval_kernel<false><<<aes_grid(K), kFssThreads, kAesTableBytes, as_stream(stream)>>>(
            bits, K, (const uint4*)root, (const uint4*)seed_cw, ctrl, flags, points, out_bits);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

// Device staging cache for the host-buffer entry point (grows, never shrinks).
struct HostEvalWs {
    std::mutex mu;
    int dev = -1;
    size_t bytes = 0;
    uint8_t* buf = nullptr;
    cudaStream_t st[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
};
static HostEvalWs g_hws;

int ogm_fss_eval_points_host(int kind, int bits, int64_t K, const void* root_h, const void* seed_cw_h,
                             const uint32_t* ctrl_h, const uint8_t* flags_h, const uint32_t* points_h,
                             uint32_t* out_bits_h) {
    OGM_CHECK_ARG(kind == OGM_KIND_DPF || kind == OGM_KIND_DCF, OGM_ERR_ARG, "unknown key kind %d", kind);
    OGM_CHECK_ARG(bits >= 1 && bits <= 32, OGM_ERR_DOMAIN, "domain_bits %d outside 1..32", bits);
    OGM_CHECK_ARG(K >= 0, OGM_ERR_ARG, "negative key count");
    if (K == 0) return OGM_OK;
    OGM_ENSURE_INIT();
    std::lock_guard<std::mutex> lk(g_hws.mu);
    int dev = 0;
    OGM_CUDA_TRY(cudaGetDevice(&dev));
    // chunk of Kc keys (multiple of 32): root 16 + cw 16*bits + ctrl 12 + flags 1 + point 4 + out
    const int64_t per_key = 16 + 16 * (int64_t)bits + 12 + 1 + 4 + 1;
    int64_t Kc = ((int64_t)1 << 21);
    if (Kc > K) Kc = (K + 31) / 32 * 32;
    const size_t slot = (size_t)(Kc * per_key + 4096);
    if (g_hws.dev != dev || g_hws.bytes < 2 * slot) {
        if (g_hws.buf) cudaFree(g_hws.buf);
        if (!g_hws.st[0] || g_hws.dev != dev) {
            for (int i = 0; i < 2; i++) {
                OGM_CUDA_TRY(cudaStreamCreateWithFlags(&g_hws.st[i], cudaStreamNonBlocking));
                OGM_CUDA_TRY(cudaEventCreateWithFlags(&g_hws.done[i], cudaEventDisableTiming));
            }
        }
        g_hws.buf = nullptr;
        OGM_CUDA_TRY(cudaMalloc(&g_hws.buf, 2 * slot));
        g_hws.bytes = 2 * slot;
        g_hws.dev = dev;
    }
    const uint8_t* rh = (const uint8_t*)root_h;
    const uint8_t* ch = (const uint8_t*)seed_cw_h;
    int64_t nchunks = (K + Kc - 1) / Kc;
    for (int64_t c = 0; c < nchunks; c++) {
        const int b = (int)(c & 1);
        cudaStream_t st = g_hws.st[b];
        const int64_t k0 = c * Kc;
        const int64_t kc = (K - k0) < Kc ? (K - k0) : Kc;
        uint8_t* base = g_hws.buf + b * slot;
        uint8_t* d_root = base;
        uint8_t* d_cw = d_root + 16 * Kc;
        uint32_t* d_ctrl = (uint32_t*)(d_cw + 16 * (size_t)bits * Kc);
        uint8_t* d_flags = (uint8_t*)(d_ctrl + 3 * Kc);
        uint32_t* d_pts = (uint32_t*)(((uintptr_t)(d_flags + Kc) + 15) & ~(uintptr_t)15);
        uint32_t* d_out = (uint32_t*)(((uintptr_t)(d_pts + Kc) + 15) & ~(uintptr_t)15);
        OGM_CUDA_TRY(cudaMemcpyAsync(d_root, rh + 16 * k0, 16 * kc, cudaMemcpyHostToDevice, st));
        // a DCF walk never reads the last level's seed correction (fss_eval_kernel): not copied
        const int cw_levels = kind == OGM_KIND_DCF ? bits - 1 : bits;
        if (cw_levels > 0)
            OGM_CUDA_TRY(cudaMemcpy2DAsync(d_cw, 16 * kc, ch + 16 * k0, 16 * K, 16 * kc, cw_levels,
                                           cudaMemcpyHostToDevice, st));
        OGM_CUDA_TRY(cudaMemcpy2DAsync(d_ctrl, 4 * kc, ctrl_h + k0, 4 * K, 4 * kc, 3, cudaMemcpyHostToDevice, st));
        OGM_CUDA_TRY(cudaMemcpyAsync(d_flags, flags_h + k0, kc, cudaMemcpyHostToDevice, st));
        OGM_CUDA_TRY(cudaMemcpyAsync(d_pts, points_h + k0, 4 * kc, cudaMemcpyHostToDevice, st));
        int rc = ogm_fss_eval_points(kind, bits, kc, d_root, d_cw, d_ctrl, d_flags, d_pts, d_out, st);
        if (rc) return rc;
        // k0 is a multiple of 32 (Kc is), so the chunk's bits start on a word
        OGM_CUDA_TRY(cudaMemcpyAsync(out_bits_h + k0 / 32, d_out, 4 * ((kc + 31) / 32),
                                     cudaMemcpyDeviceToHost, st));
    }
    OGM_CUDA_TRY(cudaStreamSynchronize(g_hws.st[0]));
    OGM_CUDA_TRY(cudaStreamSynchronize(g_hws.st[1]));
    return OGM_OK;
}

int ogm_fss_full_domain(int kind, int bits, int nkeys, const void* root, const void* seed_cw,
                        const uint32_t* ctrl, const uint8_t* flags, int64_t n, uint32_t* out_words,
                        int64_t pitch, void* stream) {
    OGM_CHECK_ARG(kind == OGM_KIND_DPF || kind == OGM_KIND_DCF, OGM_ERR_ARG, "unknown key kind %d", kind);
    OGM_CHECK_ARG(bits >= 1 && bits <= 32, OGM_ERR_DOMAIN, "domain_bits %d outside 1..32", bits);
    OGM_CHECK_ARG(n >= 0 && (bits == 32 || n <= ((int64_t)1 << bits)), OGM_ERR_DOMAIN,
                  "requested %lld points from a 2^%d domain", (long long)n, bits);
    OGM_CHECK_ARG(pitch >= (n + 31) / 32, OGM_ERR_ARG, "pitch %lld below ceil(n/32)", (long long)pitch);
    if (nkeys <= 0 || n == 0) return OGM_OK;
    OGM_ENSURE_INIT();
    // leaves per thread: the deepest subtree (<= 32 leaves, never deeper
    // than the tree) that still leaves >= 64 threads per SM.  Every thread
    // walks from the root to its subtree, so filling the GPU with shallow
    // subtrees mostly repeats the walk: measured (12 DCF keys, 14 bits,
    // 10,000 points) 81 us with 1-leaf subtrees, 41 us with 8-leaf ones;
    // (12 DCF keys, 18 bits) 161 -> 127 us; small domains unchanged.
    int kk = 5;
    if (kk > bits) kk = bits;
    const int64_t words = (n + 31) / 32;
    while (kk > 0 && (int64_t)nkeys * words * (32 >> kk) < (int64_t)sm_count() * 64) kk--;
    const int64_t slots = (int64_t)nkeys * words * (32 >> kk);
    if (kind == OGM_KIND_DCF)
        aes_launch(fss_fde_kernel<true, AesTab>, fss_fde_kernel<true, AesTabSmall>, slots, kFssThreads,
                   as_stream(stream), bits, nkeys, (const uint4*)root, (const uint4*)seed_cw, ctrl, flags, n, kk,
                   out_words, pitch);
    else
        aes_launch(fss_fde_kernel<false, AesTab>, fss_fde_kernel<false, AesTabSmall>, slots, kFssThreads,
                   as_stream(stream), bits, nkeys, (const uint4*)root, (const uint4*)seed_cw, ctrl, flags, n, kk,
                   out_words, pitch);
    OGM_LAUNCH_CHECK();
    return OGM_OK;
}

}  // extern "C"
