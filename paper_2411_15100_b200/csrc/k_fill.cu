// K2 — batched fill_next_token_bitmask.
//
// Replaces Matcher.fill_next_token_mask / _fill_cached / _resolve_dependents
// / _closed_facts (REF matcher.py:377-444, 219-237).  Per request the mask is
//     universe AND  OR_{stacks s} ( acc_row[key(s)] OR walked_dependents(s) )
// plus the EOS bit iff some stack is terminable, with bits >= V zero
// (REF matcher.py:388-390, 411-412).  This is the reference's Algorithm-1 set
// algebra with the dense accepted row as the stored form, so the expand is a
// pure streaming OR of L2-resident rows.
//
// One CTA per request row.  Phase 1: the CTA's threads each walk one
// context-dependent token of one stack against the request's full stack
// (device arena chain), setting bits of a shared-memory row.  Phase 2: all
// threads stream the output row with 128-bit loads/stores, OR-ing the cached
// rows of every stack top, the shared dependent row and the universe.
#include "device.cuh"

namespace gm {

constexpr int kFillThreads = 256;
constexpr int kDepS = 16;
constexpr int kDepF = 64;
constexpr int kMaxTopsInFill = 32;

__global__ void __launch_bounds__(kFillThreads)
fill_kernel(DevPool P, const int32_t* __restrict__ slots, int32_t n, uint32_t* __restrict__ bitmask,
            int64_t bstride, const int32_t* __restrict__ rows, uint8_t* __restrict__ need_apply) {
  extern __shared__ uint32_t dep_acc[];  // [W]
  __shared__ int32_t s_key[kMaxTopsInFill];
  __shared__ int32_t s_dep0[kMaxTopsInFill + 1];
  __shared__ int s_term, s_partial;
  const int32_t i = blockIdx.x;
  if (i >= n) return;
  const int32_t slot = slots[i];
  const int64_t row = rows ? (int64_t)rows[i] : (int64_t)i;
  const DevBinding* B = P.binding[slot];
  const DevGrammar& G = B->g;
  const DevVocab& Vc = B->v;
  const DevCache& C = B->c;
  const int32_t W = Vc.W;
  const int32_t h = P.head[slot];
  const int32_t meta = P.meta[(size_t)slot * P.H + h];
  const int ntops = meta & 0xFFFF;
  const bool terminated = (meta >> 16) & 1;
  const int2* tops = slot_tops(P, slot, h);

  for (int32_t w = threadIdx.x; w < W; w += blockDim.x) dep_acc[w] = 0u;
  if (threadIdx.x == 0) {
    int term = 0, total = 0;
    if (terminated) atomicOr(P.err, kErrTerminated);
    for (int s = 0; s < ntops && s < kMaxTopsInFill; ++s) {
      const int2 t = tops[s];
      s_key[s] = G.key_of_node[t.y];
      s_dep0[s] = total;
      const int32_t kk = s_key[s];
      total += kk >= 0 ? C.dep_off[kk + 1] - C.dep_off[kk] : 0;
      // terminable: POP(node) && every chain frame POP (term bit)
      if (!terminated && (G.node_flags[t.y] & GM_NODE_POP)) {
        const int32_t hh = t.x;
        if (hh < 0 || key_term(arena_load(P.arena, hh))) term = 1;
      }
    }
    s_dep0[ntops < kMaxTopsInFill ? ntops : kMaxTopsInFill] = total;
    s_term = term;
    s_partial = 0;
  }
  __syncthreads();
  const int nt = terminated ? 0 : (ntops < kMaxTopsInFill ? ntops : kMaxTopsInFill);

  // Phase 1: dependent-token walks, one thread per (stack, dependent token).
  const int32_t total_deps = s_dep0[nt];
  for (int32_t q = threadIdx.x; q < total_deps; q += blockDim.x) {
    int s = 0;
    while (s + 1 < nt && s_dep0[s + 1] <= q) ++s;
    const int32_t kk = s_key[s];
    const int32_t tid = C.dep_ids[C.dep_off[kk] + (q - s_dep0[s])];
    if ((dep_acc[tid >> 5] >> (tid & 31)) & 1u) continue;  // already allowed by another stack
    const int2 t = tops[s];
    const int32_t o0 = __ldg(Vc.off + tid);
    const int len = __ldg(Vc.off + tid + 1) - o0;
    const uint8_t* tok = Vc.bytes + o0;
    Walker<kDepS, kDepF> w;
    w.reset();
    w.add(t.x < 0 ? -1 : -2 - t.x, t.y);
    for (int b = 0; b < len; ++b) {
      if (w.nf > kDepF / 2) w.intern_all(P.arena);
      bool pb = false;
      if (!w.template step<kDepS>(G, P.arena, tok[b], &pb)) break;
    }
    if (w.err) atomicOr(P.err, w.err);
    if (w.n > 0) atomicOr(dep_acc + (tid >> 5), 1u << (tid & 31));
  }
  __syncthreads();

  // Phase 2: expand.  128-bit vectors when the row is 16-byte aligned.
  uint32_t* out = bitmask + row * bstride;
  const int32_t eos_w = Vc.eos >> 5;
  const uint32_t eos_bit = s_term ? (1u << (Vc.eos & 31)) : 0u;
  const uint32_t tail = (Vc.V & 31) ? ((1u << (Vc.V & 31)) - 1u) : 0xFFFFFFFFu;
  bool partial = false;
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(out) & 15) == 0) && (W % 4 == 0);
  if (vec_ok) {
    const int32_t W4 = W >> 2;
    for (int32_t w4 = threadIdx.x; w4 < W4; w4 += blockDim.x) {
      uint4 acc = reinterpret_cast<const uint4*>(dep_acc)[w4];
      for (int s = 0; s < nt; ++s) {
        const int32_t kk = s_key[s];
        if (kk < 0) continue;
        const uint4 r = __ldg(reinterpret_cast<const uint4*>(C.acc_rows + (size_t)kk * W) + w4);
        acc.x |= r.x; acc.y |= r.y; acc.z |= r.z; acc.w |= r.w;
      }
      const uint4 u = __ldg(reinterpret_cast<const uint4*>(Vc.universe) + w4);
      uint32_t v[4] = {acc.x & u.x, acc.y & u.y, acc.z & u.z, acc.w & u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int32_t w = w4 * 4 + e;
        if (w == eos_w) v[e] |= eos_bit;
        if (w == W - 1) v[e] &= tail;
        const uint32_t full = (w == W - 1) ? tail : 0xFFFFFFFFu;
        partial |= (v[e] != full);
      }
      reinterpret_cast<uint4*>(out)[w4] = make_uint4(v[0], v[1], v[2], v[3]);
    }
  } else {
    for (int32_t w = threadIdx.x; w < W; w += blockDim.x) {
      uint32_t acc = dep_acc[w];
      for (int s = 0; s < nt; ++s) {
        const int32_t kk = s_key[s];
        if (kk >= 0) acc |= __ldg(C.acc_rows + (size_t)kk * W + w);
      }
      acc &= __ldg(Vc.universe + w);
      if (w == eos_w) acc |= eos_bit;
      const uint32_t full = (w == W - 1) ? tail : 0xFFFFFFFFu;
      if (w == W - 1) acc &= tail;
      partial |= (acc != full);
      out[w] = acc;
    }
  }
  if (need_apply) {
    if (partial) s_partial = 1;
    __syncthreads();
    if (threadIdx.x == 0) need_apply[i] = (uint8_t)s_partial;
  }
}

gm_status launch_fill(const DevPool& P, const int32_t* slots, int32_t n, int32_t* bitmask,
                      int64_t bstride, const int32_t* rows, uint8_t* need_apply, int32_t W,
                      cudaStream_t s) {
  if (n <= 0) return GM_OK;
  const size_t smem = (size_t)W * 4;
  static bool attr_set = false;
  if (!attr_set) {
    GM_CUDA_TRY(cudaFuncSetAttribute(fill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr_set = true;
  }
  if (smem > 200 * 1024) return fail(GM_ERR_INVALID, "vocabulary too large for fill kernel");
  fill_kernel<<<n, kFillThreads, smem, s>>>(P, slots, n, reinterpret_cast<uint32_t*>(bitmask), bstride,
                                            rows, need_apply);
  GM_LAUNCH_CHECK();
  return GM_OK;
}

}  // namespace gm
