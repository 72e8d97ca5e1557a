// K0 — apply_token_bitmask_inplace on fp32 / fp16 / bf16 logits.
//
// Replaces XGrammar's apply kernels (xgrammar/matcher.py:58-188,
// kernels/apply_token_bitmask_inplace_{cuda.cu,triton.py}); the reference
// grammask has no apply step (REF bench.py:50-71 samples on the host).
//
// HBM-streaming design: one thread owns one 16-byte chunk of a logits row
// (8 bf16/fp16 or 4 fp32 tokens) so a warp's store instruction covers 512
// contiguous bytes.  The chunk's mask bits are a byte (or nibble) of one
// bitmask word; fully-allowed chunks cost only the (shared) bitmask read,
// fully-masked chunks are a single 128-bit store of -inf with no logits read,
// and only mixed chunks read-modify-write.  Algorithmic traffic per row is
// therefore 4*ceil(V/32) + s*M (M = masked tokens), the minimum for an
// in-place kernel.
#include "common.cuh"

namespace gm {
namespace {

__device__ __forceinline__ uint4 ld_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_v4(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// EB = bytes per element, NEG = -inf bit pattern (replicated per lane).
template <int EB>
__global__ void __launch_bounds__(256)
apply_vec_kernel(char* __restrict__ logits, int64_t n_rows, int64_t vocab,
                 int64_t lstride_bytes, const int32_t* __restrict__ bitmask,
                 int64_t bstride, const int32_t* __restrict__ indices,
                 uint32_t neg_pattern) {
  constexpr int VEC = 16 / EB;                 // tokens per 16-byte chunk
  constexpr uint32_t FULL = (VEC == 32) ? 0xFFFFFFFFu : ((1u << VEC) - 1u);
  const int64_t chunks = (vocab + VEC - 1) / VEC;
  for (int64_t i = blockIdx.y; i < n_rows; i += gridDim.y) {
    const int64_t row = indices ? (int64_t)indices[i] : i;
    char* rowp = logits + row * lstride_bytes;
    const uint32_t* brow = reinterpret_cast<const uint32_t*>(bitmask + row * bstride);
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < chunks;
         c += (int64_t)gridDim.x * blockDim.x) {
      const int64_t tok0 = c * VEC;
      const uint32_t word = __ldg(brow + (tok0 >> 5));
      uint32_t bits = (word >> (tok0 & 31)) & FULL;
      int nvalid = VEC;
      if (tok0 + VEC > vocab) {  // ragged tail: tokens >= vocab untouched
        nvalid = (int)(vocab - tok0);
        bits |= FULL & ~((1u << nvalid) - 1u);
      }
      if (bits == FULL) continue;
      char* p = rowp + tok0 * EB;
      if (nvalid == VEC && bits == 0) {
        st_v4(p, make_uint4(neg_pattern, neg_pattern, neg_pattern, neg_pattern));
        continue;
      }
      uint4 v = ld_v4(p);
      uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        if (!((bits >> j) & 1u)) {
          if (EB == 4) {
            w[j] = neg_pattern;
          } else {
            const int k = j >> 1, sh = (j & 1) * 16;
            w[k] = (w[k] & ~(0xFFFFu << sh)) | ((neg_pattern & 0xFFFFu) << sh);
          }
        }
      }
      st_v4(p, make_uint4(w[0], w[1], w[2], w[3]));
    }
  }
}

// Unaligned rows: one thread per token.
template <int EB>
__global__ void __launch_bounds__(256)
apply_scalar_kernel(char* __restrict__ logits, int64_t n_rows, int64_t vocab,
                    int64_t lstride_bytes, const int32_t* __restrict__ bitmask,
                    int64_t bstride, const int32_t* __restrict__ indices,
                    uint32_t neg_pattern) {
  for (int64_t i = blockIdx.y; i < n_rows; i += gridDim.y) {
    const int64_t row = indices ? (int64_t)indices[i] : i;
    char* rowp = logits + row * lstride_bytes;
    const int32_t* brow = bitmask + row * bstride;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < vocab;
         t += (int64_t)gridDim.x * blockDim.x) {
      if ((__ldg(brow + (t >> 5)) >> (t & 31)) & 1) continue;
      if (EB == 4) *reinterpret_cast<uint32_t*>(rowp + t * 4) = neg_pattern;
      else *reinterpret_cast<uint16_t*>(rowp + t * 2) = (uint16_t)neg_pattern;
    }
  }
}

}  // namespace
}  // namespace gm

using namespace gm;

extern "C" gm_status gm_apply_inplace(void* logits, int32_t dtype, int64_t n_rows,
                                      int64_t vocab_size, int64_t logits_stride,
                                      const int32_t* bitmask, int64_t bitmask_stride,
                                      const int32_t* indices, void* stream) {
  if (n_rows < 0 || vocab_size < 0) return fail(GM_ERR_INVALID, "negative shape");
  if (n_rows == 0 || vocab_size == 0) return GM_OK;
  if (!logits || !bitmask) return fail(GM_ERR_INVALID, "null logits/bitmask");
  int eb;
  uint32_t neg;
  switch (dtype) {
    case GM_DTYPE_F32: eb = 4; neg = 0xFF800000u; break;
    case GM_DTYPE_F16: eb = 2; neg = 0xFC00FC00u; break;
    case GM_DTYPE_BF16: eb = 2; neg = 0xFF80FF80u; break;
    default: return fail(GM_ERR_INVALID, "unknown dtype");
  }
  const int64_t lstride_bytes = logits_stride * eb;
  const bool aligned = (reinterpret_cast<uintptr_t>(logits) % 16 == 0) && (lstride_bytes % 16 == 0);
  cudaStream_t s = as_stream(stream);
  const int threads = 256;
  const int64_t per_thread = aligned ? (16 / eb) : 1;
  int64_t gx = ceil_div(ceil_div(vocab_size, per_thread), threads);
  if (gx > 65535) gx = 65535;
  const unsigned gy = (unsigned)(n_rows < 65535 ? n_rows : 65535);
  dim3 grid((unsigned)gx, gy);
  char* lp = static_cast<char*>(logits);
  if (aligned) {
    if (eb == 4) apply_vec_kernel<4><<<grid, threads, 0, s>>>(lp, n_rows, vocab_size, lstride_bytes, bitmask, bitmask_stride, indices, neg);
    else apply_vec_kernel<2><<<grid, threads, 0, s>>>(lp, n_rows, vocab_size, lstride_bytes, bitmask, bitmask_stride, indices, neg);
  } else {
    if (eb == 4) apply_scalar_kernel<4><<<grid, threads, 0, s>>>(lp, n_rows, vocab_size, lstride_bytes, bitmask, bitmask_stride, indices, neg);
    else apply_scalar_kernel<2><<<grid, threads, 0, s>>>(lp, n_rows, vocab_size, lstride_bytes, bitmask, bitmask_stride, indices, neg);
  }
  GM_LAUNCH_CHECK();
  return GM_OK;
}
