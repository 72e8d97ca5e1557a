// Write-bandwidth probe (diagnostic, not part of the library): which store
// form streams -inf into HBM fastest on this B200?  Each variant writes
// `bytes` of 0xFF80 (bf16 -inf) into a ring of buffers, `reps` launches back
// to back, timed with CUDA events in C (no Python launch overhead).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
//        -o tools/libbwprobe.so tools/bwprobe.cu
//   python tools/bwprobe.py
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__global__ void st_v4(uint4* p, int64_t n16) {
  const uint4 v = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void st_v4_cs(uint4* p, int64_t n16) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%1,%1,%1};" ::"l"(p + i), "r"(0xFF80FF80u) : "memory");
}

__global__ void st_v8(uint4* p, int64_t n16) {  // 256-bit stores (sm_100)
  const int64_t n32 = n16 / 2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n32; i += (int64_t)gridDim.x * blockDim.x)
    asm volatile("st.global.v8.u32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p + 2 * i), "r"(0xFF80FF80u) : "memory");
}

__global__ void st_v8_evict_first(uint4* p, int64_t n16) {
  const int64_t n32 = n16 / 2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n32; i += (int64_t)gridDim.x * blockDim.x)
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p + 2 * i),
                 "r"(0xFF80FF80u) : "memory");
}

// unrolled: each thread writes 4 consecutive-warp-strided 16-B chunks per iteration
__global__ void st_v4_unroll4(uint4* p, int64_t n16) {
  const uint4 v = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    p[i] = v; p[i + stride] = v; p[i + 2 * stride] = v; p[i + 3 * stride] = v;
  }
  for (; i < n16; i += stride) p[i] = v;
}

// TMA bulk store: smem tile of -inf (16 KB) written with cp.async.bulk.global.shared
__global__ void st_tma(uint4* p, int64_t n16) {
  extern __shared__ __align__(128) uint4 tile[];
  constexpr int kTile = 16384;
  for (int i = threadIdx.x; i < kTile / 16; i += blockDim.x)
    tile[i] = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const int64_t bytes = n16 * 16;
    const int64_t ntiles = bytes / kTile;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"((char*)p + t * kTile),
                   "r"((uint32_t)__cvta_generic_to_shared(tile)), "r"(kTile) : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// PDL: allow the next launch to start now, wait for the previous grid
// (its memory visible) before storing
__global__ void st_v4_pdl(uint4* p, int64_t n16, int wait) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (wait) asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint4 v = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void copy_v4(const uint4* a, uint4* b, int64_t n16) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

}  // namespace

// variant: 0 v4, 1 v4.cs, 2 v8, 3 v8 evict_first, 4 v4 unroll4, 5 TMA bulk store, 6 copy (src = bufs[(k+1)%nbuf])
// returns microseconds per launch (mean over reps)
extern "C" float bw_probe(int variant, void** bufs, int nbuf, int64_t bytes, int reps, int blocks, int threads,
                          int graph) {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int64_t n16 = bytes / 16;
  if (variant == 5) cudaFuncSetAttribute(st_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  auto launch = [&](int k) {
    uint4* p = static_cast<uint4*>(bufs[k % nbuf]);
    switch (variant) {
      case 0: st_v4<<<blocks, threads, 0, st>>>(p, n16); break;
      case 1: st_v4_cs<<<blocks, threads, 0, st>>>(p, n16); break;
      case 2: st_v8<<<blocks, threads, 0, st>>>(p, n16); break;
      case 3: st_v8_evict_first<<<blocks, threads, 0, st>>>(p, n16); break;
      case 4: st_v4_unroll4<<<blocks, threads, 0, st>>>(p, n16); break;
      case 5: st_tma<<<blocks, threads, 16384, st>>>(p, n16); break;
      case 6: copy_v4<<<blocks, threads, 0, st>>>(static_cast<const uint4*>(bufs[(k + 1) % nbuf]), p, n16); break;
      case 7:
      case 8: {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(blocks);
        cfg.blockDim = dim3(threads);
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, st_v4_pdl, p, n16, variant == 7 ? 1 : 0);
        break;
      }
    }
  };
  for (int k = 0; k < 3; ++k) launch(k);
  cudaGraphExec_t exec = nullptr;
  if (graph) {
    cudaGraph_t g;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int k = 0; k < reps; ++k) launch(k);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    cudaGraphLaunch(exec, st);
  }
  cudaStreamSynchronize(st);
  cudaEventRecord(e0, st);
  if (graph) cudaGraphLaunch(exec, st);
  else
    for (int k = 0; k < reps; ++k) launch(k);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  if (exec) cudaGraphExecDestroy(exec);
  cudaStreamDestroy(st);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (cudaGetLastError() != cudaSuccess) return -1.0f;
  return ms * 1000.0f / reps;
}
