// ogm_engine.cuh -- secEval / combine / fetch kernels (src/engine.py, src/rss.py).
#pragma once
#include "ogm_common.cuh"
namespace ogm {
int engine_init() { return OGM_OK; }
}  // namespace ogm
