// Shared helpers for libgmask: error plumbing, launch checks, constants.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include "../../include/gmask.h"

namespace gm {

constexpr int kNumSMs = 148;  // B200

// thread-local last error, surfaced through gm_last_error()
void set_error(const std::string& msg);
gm_status fail(gm_status code, const std::string& msg);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

#define GM_CUDA_TRY(expr)                                                        \
  do {                                                                           \
    cudaError_t _e = (expr);                                                     \
    if (_e != cudaSuccess)                                                       \
      return ::gm::fail(GM_ERR_CUDA, std::string(#expr) + ": " +               \
                                        cudaGetErrorString(_e));                 \
  } while (0)

#define GM_LAUNCH_CHECK() GM_CUDA_TRY(cudaGetLastError())

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace gm
