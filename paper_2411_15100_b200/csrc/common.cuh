// Shared helpers for libgmask: error plumbing, launch checks, constants.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdlib>
#include <string>
#include <utility>

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

// Programmatic dependent launch (PDL).  The per-step kernels (apply, fill,
// accept, step, recycle) are launched with programmatic stream
// serialization: the launch, CTA rasterisation and prologue of kernel k+1
// overlap the drain of kernel k in the same stream (measured ~2 us per
// launch on B200, tools/bwprobe.cu).  Each such kernel calls pdl_trigger()
// then pdl_wait() before its first global-memory access, so every read and
// write still happens after the previous kernel has completed and its
// memory is visible — stream order is preserved.  GMASK_NO_PDL=1 disables
// the attribute (plain launches; the griddepcontrol instructions are then
// no-ops).
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("GMASK_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

struct L2Window {  // optional L2 persisting access-policy window of a launch
  void* base;
  size_t bytes;
  float hit;
};

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_w(const L2Window* win, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (win && win->base) {
    attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[na].val.accessPolicyWindow.base_ptr = win->base;
    attr[na].val.accessPolicyWindow.num_bytes = win->bytes;
    attr[na].val.accessPolicyWindow.hitRatio = win->hit;
    attr[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  return launch_pdl_w(nullptr, kernel, grid, block, smem, s, std::forward<Args>(args)...);
}

#ifdef __CUDACC__
// -inf stores into logits: streaming (.cs = evict-first in L2), so the
// masked-logits stream does not push the matcher state, arena and cache rows
// (read again next step) out of L2 — with the logits written back to back,
// every L2 miss of the latency-bound fill/accept chain otherwise queues
// behind the write stream at HBM.
__device__ __forceinline__ void st_cs_v4(void* p, uint32_t v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%1,%1,%1};" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_cs_u32(void* p, uint32_t v) {
  asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_cs_u16(void* p, uint32_t v) {
  asm volatile("st.global.cs.u16 [%0], %1;" ::"l"(p), "h"((unsigned short)v) : "memory");
}
// A 16-byte chunk of logits whose mask bits are mixed (some kept, some
// masked): load it, overwrite the masked elements with -inf and store the
// whole chunk.  Rewriting the kept elements with their own bits leaves them
// bit-identical; one full-sector store replaces up to 8 byte-masked partial
// stores, which the memory system would otherwise merge sector by sector
// (SQL-like masks: K5 48.2 -> 39.4 us/step).
// Used by K0 (per tile) and the fused apply (per warp round) when the
// mixed chunks are dense and heavily masked (gm_apply_set_blend).
template <int EB>
__device__ __forceinline__ void blend_chunk(void* p, uint32_t keep, uint32_t neg) {
  uint32_t v0, v1, v2, v3;
  asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3) : "l"(p));
  uint32_t v[4] = {v0, v1, v2, v3};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t km;  // bits of word k that keep their value
    if (EB == 4) km = ((keep >> k) & 1u) ? 0xFFFFFFFFu : 0u;
    else km = (((keep >> (2 * k)) & 1u) ? 0x0000FFFFu : 0u) | (((keep >> (2 * k + 1)) & 1u) ? 0xFFFF0000u : 0u);
    v[k] = (v[k] & km) | (neg & ~km);
  }
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3])
               : "memory");
}
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#endif

}  // namespace gm
