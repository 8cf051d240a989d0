// ogm_common.cuh -- shared plumbing for the sm_100a OblivGM kernels:
// thread-local error reporting behind the C ABI, launch helpers, constants.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "oblivgm_b200.h"

namespace ogm {

// Thread-local last-error message (read through ogm_last_error()).
void set_error(const char* fmt, ...);
const char* get_error();

constexpr int kSmCountB200 = 148;

inline int sm_count() {
    static thread_local int cached = 0;
    if (!cached) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
        if (cached <= 0) cached = kSmCountB200;
    }
    return cached;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace ogm

#define OGM_CHECK_ARG(cond, code, ...)      \
    do {                                    \
        if (!(cond)) {                      \
            ::ogm::set_error(__VA_ARGS__);  \
            return (code);                  \
        }                                   \
    } while (0)

#define OGM_CUDA_TRY(expr)                                                              \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess) {                                                        \
            ::ogm::set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(_e), __FILE__, \
                             __LINE__, cudaGetErrorString(_e));                         \
            return OGM_ERR_CUDA;                                                        \
        }                                                                               \
    } while (0)

#define OGM_LAUNCH_CHECK() OGM_CUDA_TRY(cudaGetLastError())
