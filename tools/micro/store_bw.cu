// Store-bandwidth probe for the K5 apply phase: how fast can C CTAs, each
// owning a contiguous span, fill the span with -inf (16-byte streaming
// stores)?  Tells whether the fused apply (one CTA per 256-KB logits row) is
// bound per SM or by the memory system.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a store_bw.cu -o store_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void fill_span(char* base, int64_t span, uint32_t neg, int mode) {
  char* p = base + (int64_t)blockIdx.x * span;
  const int64_t chunks = span / 16;
  for (int64_t c = threadIdx.x; c < chunks; c += blockDim.x) {
    char* q = p + c * 16;
    if (mode == 0)
      asm volatile("st.global.cs.v4.u32 [%0], {%1,%1,%1,%1};" ::"l"(q), "r"(neg) : "memory");
    else
      asm volatile("st.global.v4.u32 [%0], {%1,%1,%1,%1};" ::"l"(q), "r"(neg) : "memory");
  }
}

// 32-byte stores: each thread owns 32 B per iteration
__global__ void fill_span32(char* base, int64_t span, uint32_t neg) {
  char* p = base + (int64_t)blockIdx.x * span;
  const int64_t chunks = span / 32;
  for (int64_t c = threadIdx.x; c < chunks; c += blockDim.x) {
    char* q = p + c * 32;
    asm volatile("st.global.v8.u32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(q), "r"(neg) : "memory");
  }
}

int main() {
  const int64_t total = 128ll * 128256 * 2;  // 128 bf16 rows of 128,256 logits
  char* buf;
  cudaMalloc(&buf, total + (1 << 20));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int ctas_list[] = {1, 16, 64, 128, 148, 256, 296, 512, 1024};
  const int thr_list[] = {256, 512, 1024};
  for (int mode : {0, 1, 3})
    for (int thr : thr_list)
      for (int ctas : ctas_list) {
        int64_t span = (total / ctas) & ~(int64_t)511;
        auto run = [&] {
          if (mode < 3) fill_span<<<ctas, thr>>>(buf, span, 0xff80ff80u, mode);
          else fill_span32<<<ctas, thr>>>(buf, span, 0xff80ff80u);
        };
        for (int w = 0; w < 3; ++w) run();
        cudaEventRecord(a);
        const int reps = 20;
        for (int r = 0; r < reps; ++r) run();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double us = ms * 1e3 / reps;
        const double bytes = (double)span * ctas;
        printf("{\"mode\": %d, \"threads\": %d, \"ctas\": %d, \"span_kb\": %.1f, \"us\": %.2f, \"GBps\": %.0f, \"GBps_per_cta\": %.1f}\n",
               mode, thr, ctas, span / 1024.0, us, bytes / us / 1e3, bytes / us / 1e3 / ctas);
      }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
