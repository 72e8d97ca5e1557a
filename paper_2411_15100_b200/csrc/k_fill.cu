// K2 — batched fill_next_token_bitmask.
//
// Replaces Matcher.fill_next_token_mask / _fill_cached / _resolve_dependents
// / _closed_facts (REF matcher.py:377-444, 219-237).  Per request the mask is
//     universe AND  OR_{stacks s} ( acc_row[key(s)] OR walked_dependents(s) )
// plus the EOS bit iff some stack is terminable, with bits >= V zero
// (REF matcher.py:388-390, 411-412).  This is the reference's Algorithm-1 set
// algebra with the dense accepted row as the stored form, so the expand is a
// pure streaming OR of rows.
//
// One CTA per request row, designed for a cold L2 (the model's forward pass
// evicts everything between decode steps), i.e. for few dependent round
// trips: the slot header (one 256-byte record) gives keys, dependent ranges
// and the EOS fact; the grammar tables are staged into shared memory in one
// coalesced copy; each dependent token (id + bytes, contiguous per key) is
// walked by one thread against the request's full stack, setting bits of a
// shared-memory row; finally all threads stream the output row with 128-bit
// loads/stores.
#include "device.cuh"

namespace gm {

constexpr int kFillThreads = 256;
constexpr int kDepS = 16;
constexpr int kDepF = 64;

__global__ void __launch_bounds__(kFillThreads)
fill_kernel(DevPool P, const int32_t* __restrict__ slots, int32_t n, uint32_t* __restrict__ bitmask,
            int64_t bstride, const int32_t* __restrict__ rows, uint8_t* __restrict__ need_apply, int32_t Wmax) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* dep_acc = reinterpret_cast<uint32_t*>(smem);         // [Wmax]
  uint8_t* tables = smem + (((size_t)Wmax * 4 + 15) & ~(size_t)15);   // staged grammar blob
  __shared__ SlotHdr s_hdr;
  __shared__ int s_partial, s_nt;
  __shared__ int32_t s_key[32], s_lo[32], s_hi[32];
  __shared__ int2 s_top[32];
  const int32_t i = blockIdx.x;
  if (i >= n) return;
  const int32_t slot = __ldg(slots + i);
  const int64_t row = rows ? (int64_t)__ldg(rows + i) : (int64_t)i;

  // header: 256 bytes, one coalesced load
  if (threadIdx.x < 16)
    reinterpret_cast<int4*>(&s_hdr)[threadIdx.x] = reinterpret_cast<const int4*>(P.hdr + slot)[threadIdx.x];
  if (threadIdx.x == 0) s_partial = 0;
  __syncthreads();
  const DevBinding* B = s_hdr.binding;
  const DevVocab& Vc = B->v;
  const DevCache& C = B->c;
  const int32_t W = Vc.W;
  const bool terminated = s_hdr.flags & 1;
  if (threadIdx.x == 0) {
    int nt = s_hdr.ntops;
    if (terminated) {
      atomicOr(P.err, kErrTerminated);
      nt = 0;
    } else if (nt >= 0) {
      for (int s = 0; s < nt; ++s) {
        s_key[s] = s_hdr.key[s];
        s_lo[s] = s_hdr.dep_lo[s];
        s_hi[s] = s_hdr.dep_hi[s];
        s_top[s] = s_hdr.top[s];
      }
    } else {  // more stacks than the header holds: read the ring entry
      const int32_t h = P.head[slot];
      nt = P.meta[(size_t)slot * P.H + h] & 0xFFFF;
      const int2* tops = slot_tops(P, slot, h);
      for (int s = 0; s < nt; ++s) {
        const int32_t k = B->g.key_of_node[tops[s].y];
        s_key[s] = k;
        s_lo[s] = k >= 0 ? C.dep_off[k] : 0;
        s_hi[s] = k >= 0 ? C.dep_off[k + 1] : 0;
        s_top[s] = tops[s];
      }
    }
    s_nt = nt;
  }
  __syncthreads();
  const int nt = s_nt;
  int total = 0;
  for (int s = 0; s < nt; ++s) total += s_hi[s] - s_lo[s];

  for (int32_t w = threadIdx.x; w < W; w += blockDim.x) dep_acc[w] = 0u;
  DevGrammar G = B->g;
  if (total) G = stage_grammar(B->g, tables);
  __syncthreads();

  // Phase 1: dependent-token walks, one thread per (stack, dependent token).
  for (int32_t q = threadIdx.x; q < total; q += blockDim.x) {
    int s = 0, base = 0;
    while (q - base >= s_hi[s] - s_lo[s]) {
      base += s_hi[s] - s_lo[s];
      ++s;
    }
    const int4 ent = __ldg(C.dep_ent + s_lo[s] + (q - base));
    const int32_t tid = ent.x;
    if ((dep_acc[tid >> 5] >> (tid & 31)) & 1u) continue;  // already allowed by another stack
    const uint8_t* tok = C.dep_bytes + ent.y;
    const int2 t = s_top[s];
    Walker<kDepS, kDepF> w;
    w.reset();
    w.add(t.x < 0 ? -1 : -2 - t.x, t.y);
    for (int b = 0; b < ent.z; ++b) {
      if (w.nf > kDepF / 2) w.intern_all(P.arena);
      bool pb = false;
      if (!w.template step<kDepS>(G, P.arena, __ldg(tok + b), &pb)) break;
    }
    if (w.err) atomicOr(P.err, w.err);
    if (w.n > 0) atomicOr(dep_acc + (tid >> 5), 1u << (tid & 31));
  }
  __syncthreads();

  // Phase 2: expand.  128-bit vectors when the row is 16-byte aligned.
  uint32_t* out = bitmask + row * bstride;
  const int32_t eos_w = Vc.eos >> 5;
  const uint32_t eos_bit = (!terminated && (s_hdr.flags & 2)) ? (1u << (Vc.eos & 31)) : 0u;
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
        partial |= (v[e] != ((w == W - 1) ? tail : 0xFFFFFFFFu));
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
      if (w == W - 1) acc &= tail;
      partial |= (acc != ((w == W - 1) ? tail : 0xFFFFFFFFu));
      out[w] = acc;
    }
  }
  if (need_apply) {
    if (partial) s_partial = 1;
    __syncthreads();
    if (threadIdx.x == 0) need_apply[i] = (uint8_t)s_partial;
  }
}

gm_status launch_fill(const DevPool& P, const int32_t* slots, int32_t n, int32_t* bitmask, int64_t bstride,
                      const int32_t* rows, uint8_t* need_apply, int32_t Wmax, cudaStream_t s) {
  if (n <= 0) return GM_OK;
  const size_t smem = (((size_t)Wmax * 4 + 15) & ~(size_t)15) + kStageBytes;
  static bool attr_set = false;
  if (!attr_set) {
    GM_CUDA_TRY(cudaFuncSetAttribute(fill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    attr_set = true;
  }
  if (smem > 220 * 1024) return fail(GM_ERR_INVALID, "vocabulary too large for fill kernel");
  fill_kernel<<<n, kFillThreads, smem, s>>>(P, slots, n, reinterpret_cast<uint32_t*>(bitmask), bstride, rows,
                                            need_apply, Wmax);
  GM_LAUNCH_CHECK();
  return GM_OK;
}

}  // namespace gm
