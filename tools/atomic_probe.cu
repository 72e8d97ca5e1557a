// Latency probe (diagnostic): cycles per dependent 64-bit atomicCAS / load
// on a device buffer, one thread, hot and cold lines.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o tools/libatomicprobe.so tools/atomic_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void probe(unsigned long long* buf, size_t n, long long* out, int mode) {
  if (threadIdx.x != 0) return;
  unsigned long long v = 0;
  long long t0 = clock64();
  const int iters = 64;
  for (int i = 0; i < iters; ++i) {
    size_t idx = mode >= 2 ? ((size_t)(v + i) * 2654435761ull % n) : (size_t)(blockIdx.x * 64 + (v & 1));
    if (mode == 0 || mode == 2) v = atomicCAS(buf + idx, ~0ull, ~0ull) & 1;  // compare fails: no write
    else { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(buf + idx) : "memory"); v &= 1; }
  }
  long long t1 = clock64();
  out[blockIdx.x] = (t1 - t0) / iters + (long long)(v & 0);
}

extern "C" int atomic_probe(void* buf, size_t n, long long* out_host, int mode, int blocks) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * blocks);
  probe<<<blocks, 32>>>((unsigned long long*)buf, n, d, mode);
  cudaMemcpy(out_host, d, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return (int)cudaGetLastError();
}
