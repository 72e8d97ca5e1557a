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
// One CTA per request row, built for a cold L2 (the model's forward pass
// evicts it between decode steps), i.e. for as few dependent HBM round trips
// as possible:
//   1. the 512-byte slot header (pointers, cache keys, dependent ranges, EOS
//      fact, tops and their ancestor-chain arena keys) — one coalesced load;
//   2. TMA bulk copies bring the accepted row of every top and the universe
//      row into shared memory while the binding blob (walker tables) is
//      staged the same way and each dependent record (id + length + 16 inline
//      bytes) is fetched;
//   3. one thread per dependent token (spread across warps) walks it against
//      the request's full stack (tables in smem, pops served from the header's
//      ancestor chain), setting bits of a shared-memory row;
//   4. rows, dependent bits and universe are merged from shared memory and
//      stored with 128-bit stores.
#include "device.cuh"

namespace gm {

constexpr int kFillThreads = 512;
constexpr int kTmaRows = 4;     // tops whose rows are TMA-staged (more: direct loads)
constexpr int kDepS = 16;
constexpr int kDepF = 64;
constexpr int kDepR = 4;    // register walker: stacks
constexpr int kDepRF = 24;  // register walker: local frames

// K3 tail: mask one logits row in place from the finished mask words in
// shared memory (coalesced 16-byte chunks, -inf only where masked, logits
// never read; mixed chunks store just their masked elements).
__device__ __forceinline__ void apply_row(char* __restrict__ rowp, const uint32_t* __restrict__ words, int64_t vocab,
                                          int eb, uint32_t neg) {
  const int vec = 16 / eb;
  const uint32_t full = (1u << vec) - 1u;
  const int64_t chunks = (vocab + vec - 1) / vec;
  for (int64_t c = threadIdx.x; c < chunks; c += blockDim.x) {
    const int64_t tok0 = c * vec;
    uint32_t keep = (words[tok0 >> 5] >> (tok0 & 31)) & full;
    if (tok0 + vec > vocab) keep |= full & ~((1u << (vocab - tok0)) - 1u);
    if (keep == full) continue;
    char* p = rowp + tok0 * eb;
    if (keep == 0) {
      asm volatile("st.global.v4.u32 [%0], {%1,%1,%1,%1};" ::"l"(p), "r"(neg) : "memory");
    } else {
      uint32_t m = ~keep & full;
      while (m) {
        const int j = __ffs(m) - 1;
        m &= m - 1;
        if (eb == 4) *reinterpret_cast<uint32_t*>(p + j * 4) = neg;
        else *reinterpret_cast<uint16_t*>(p + j * 2) = (uint16_t)neg;
      }
    }
  }
}

template <bool APPLY>
__global__ void __launch_bounds__(kFillThreads)
fill_kernel(DevPool P, const int32_t* __restrict__ slots, int32_t n, uint32_t* __restrict__ bitmask,
            int64_t bstride, const int32_t* __restrict__ rows, uint8_t* __restrict__ need_apply, int32_t Wmax,
            char* __restrict__ logits, int64_t lstride_bytes, int64_t ap_vocab, int ap_eb, uint32_t ap_neg) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t* dep_acc = reinterpret_cast<uint32_t*>(smem);                    // [Wmax]
  uint8_t* tables = smem + (((size_t)Wmax * 4 + 15) & ~(size_t)15);        // staged blob
  __shared__ SlotHdr hd;
  __shared__ int s_partial, s_nt;
  __shared__ int32_t s_key[32], s_lo[32], s_hi[32];
  __shared__ int2 s_top[32];
  const int32_t i = blockIdx.x;
  if (i >= n) return;
  trace_mark(P, 1, 0);
  unsigned long long t_start = 0;
  if (P.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  const int32_t slot = __ldg(slots + i);
  const int64_t row = rows ? (int64_t)__ldg(rows + i) : (int64_t)i;
  load_header(P, slot, &hd);
  __syncthreads();
  trace_mark(P, 1, 1);
  const int32_t W = hd.W;
  const bool terminated = hd.flags & 1;
  if (threadIdx.x == 0) {
    s_partial = 0;
    int nt = hd.ntops;
    if (terminated) {
      atomicOr(P.err, kErrTerminated);
      nt = 0;
    } else if (nt >= 0) {
      for (int s = 0; s < nt; ++s) {
        s_key[s] = hd.key[s];
        s_lo[s] = hd.dep_lo[s];
        s_hi[s] = hd.dep_hi[s];
        s_top[s] = hd.top[s];
      }
    } else {  // more stacks than the header holds: read the ring entry
      const int32_t h = P.head[slot];
      nt = P.meta[(size_t)slot * P.H + h] & 0xFFFF;
      const int2* tops = slot_tops(P, slot, h);
      const DevGrammar Gg = blob_view(hd.blob);
      for (int s = 0; s < nt; ++s) {
        const int4 ni = Gg.node_info[tops[s].y];
        s_key[s] = ni.x;
        s_lo[s] = ni.y;
        s_hi[s] = ni.z;
        s_top[s] = tops[s];
      }
    }
    s_nt = nt;
  }
  for (int32_t w = threadIdx.x; w < W; w += blockDim.x) dep_acc[w] = 0u;
  __syncthreads();
  trace_mark(P, 1, 2);
  const int nt = s_nt;

  // Stage the accepted rows of every top and the universe into shared memory
  // with TMA bulk copies; they land while the dependent walks run.
  const bool vec = (!bitmask || (reinterpret_cast<uintptr_t>(bitmask + row * bstride) & 15) == 0) && (W % 4 == 0);
  const bool tma = vec && nt <= kTmaRows;
  const int32_t W4 = W >> 2;
  const size_t row_bytes = ((size_t)W * 4 + 15) & ~(size_t)15;
  uint8_t* rows_s = tables + kStageBytes;  // [kTmaRows + 1][row_bytes]
  __shared__ __align__(8) unsigned long long rows_bar;
  __shared__ int s_nrows;
  if (tma && threadIdx.x == 0) {
    int nr = 0;
    for (int s = 0; s < nt; ++s) nr += s_key[s] >= 0;
    s_nrows = nr;
    mbar_init(&rows_bar, (uint32_t)((nr + 1) * (size_t)W * 4));
    int k = 0;
    for (int s = 0; s < nt; ++s) {
      if (s_key[s] < 0) continue;
      bulk_g2s(rows_s + (size_t)k * row_bytes, hd.acc_rows + (size_t)s_key[s] * W, (uint32_t)W * 4, &rows_bar);
      ++k;
    }
    bulk_g2s(rows_s + (size_t)kTmaRows * row_bytes, hd.universe, (uint32_t)W * 4, &rows_bar);
  }

  trace_mark(P, 1, 3);
  int total = 0;
  for (int s = 0; s < nt; ++s) total += s_hi[s] - s_lo[s];
  (void)total;
  if (P.trace && blockIdx.x == 0 && threadIdx.x == 0) {
    P.trace[16 + 8] = (unsigned long long)total;
    P.trace[16 + 9] = (unsigned long long)(nt > 0 ? s_key[0] : -1);
    P.trace[16 + 10] = (unsigned long long)nt;
  }
  if (total) {
    const DevGrammar G = stage_blob(hd.blob, hd.blob_bytes, tables);
    trace_mark(P, 1, 4);
    const uint8_t* rec_base = reinterpret_cast<const uint8_t*>(hd.dep_ent);
    // warp-major assignment: consecutive dependents go to different warps, so
    // a handful of walks run in parallel instead of diverging inside one warp
    const int32_t nw = blockDim.x >> 5;
    const int32_t q0 = (threadIdx.x & 31) * nw + (threadIdx.x >> 5);
    for (int32_t q = q0; q < total; q += blockDim.x) {
      int s = 0, base = 0;
      while (q - base >= s_hi[s] - s_lo[s]) {
        base += s_hi[s] - s_lo[s];
        ++s;
      }
      const int4* rec = hd.dep_ent + 2 * (size_t)(s_lo[s] + (q - base));
      const int4 e = __ldg(rec), inl = __ldg(rec + 1);
      const int32_t tid = e.x;
      if ((dep_acc[tid >> 5] >> (tid & 31)) & 1u) continue;  // already allowed by another stack
      const int2 t = s_top[s];
      const uint8_t* far = rec_base + e.z;  // bytes beyond the inline 16
      const bool tr = P.trace && blockIdx.x == 0 && q == 0;
      long long c0 = tr ? clock64() : 0;
      // fast path: register walker; general walker only on spill
      RWalker<kDepR, kDepRF> rw;
      rw.init(hd.chain_h, hd.chain_k, hd.nchain);
      rw.add(rw.ref_of_handle(t.x), t.y);
      for (int b = 0; b < e.y && rw.n > 0 && !rw.spill; ++b) {
        bool pb = false;
        rw.step(G, P.arena, rec_byte(inl, far, b), &pb);
        if (tr && b < 12) {
          const long long c1 = clock64();
          P.trace[32 + b] = (unsigned long long)(c1 - c0) | ((unsigned long long)rw.n << 48);
          c0 = c1;
        }
      }
      if (tr) P.trace[44] = (unsigned long long)e.y | ((unsigned long long)rw.spill << 16) |
                            ((unsigned long long)hd.nchain << 32);
      bool ok;
      if (!rw.spill) {
        if (rw.err) atomicOr(P.err, rw.err);
        ok = rw.n > 0;
      } else {
        Walker<kDepS, kDepF> w;
        w.reset();
        w.external(hd.chain_h, hd.chain_k, hd.nchain);
        w.add(t.x < 0 ? -1 : -2 - t.x, t.y);
        for (int b = 0; b < e.y; ++b) {
          if (w.nf > kDepF / 2) w.intern_all(P.arena);
          bool pb = false;
          if (!w.template step<kDepS>(G, P.arena, rec_byte(inl, far, b), &pb)) break;
        }
        if (w.err) atomicOr(P.err, w.err);
        ok = w.n > 0;
      }
      if (ok) atomicOr(dep_acc + (tid >> 5), 1u << (tid & 31));
    }
  }
  trace_mark(P, 1, 5);
  __syncthreads();
  trace_mark(P, 1, 6);

  // Merge and store.
  uint32_t* out = bitmask ? bitmask + row * bstride : nullptr;
  const int32_t eos_w = hd.eos >> 5;
  const uint32_t eos_bit = (!terminated && (hd.flags & 2)) ? (1u << (hd.eos & 31)) : 0u;
  const uint32_t tail = (hd.V & 31) ? ((1u << (hd.V & 31)) - 1u) : 0xFFFFFFFFu;
  bool partial = false;
  if (tma) {
    mbar_wait(&rows_bar, 0);
    const int nr = s_nrows;
    const uint4* univ = reinterpret_cast<const uint4*>(rows_s + (size_t)kTmaRows * row_bytes);
    for (int32_t w4 = threadIdx.x; w4 < W4; w4 += blockDim.x) {
      uint4 a = reinterpret_cast<const uint4*>(dep_acc)[w4];
      for (int k = 0; k < nr; ++k) {
        const uint4 r = reinterpret_cast<const uint4*>(rows_s + (size_t)k * row_bytes)[w4];
        a.x |= r.x; a.y |= r.y; a.z |= r.z; a.w |= r.w;
      }
      const uint4 u = univ[w4];
      uint32_t v[4] = {a.x & u.x, a.y & u.y, a.z & u.z, a.w & u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int32_t w = w4 * 4 + e;
        if (w == eos_w) v[e] |= eos_bit;
        if (w == W - 1) v[e] &= tail;
        partial |= (v[e] != ((w == W - 1) ? tail : 0xFFFFFFFFu));
      }
      const uint4 fin = make_uint4(v[0], v[1], v[2], v[3]);
      if (out) reinterpret_cast<uint4*>(out)[w4] = fin;
      if (APPLY) reinterpret_cast<uint4*>(dep_acc)[w4] = fin;  // own slot only
    }
  } else {
    for (int32_t w = threadIdx.x; w < W; w += blockDim.x) {
      uint32_t a = dep_acc[w];
      for (int s = 0; s < nt; ++s) {
        const int32_t kk = s_key[s];
        if (kk >= 0) a |= __ldg(hd.acc_rows + (size_t)kk * W + w);
      }
      a &= __ldg(hd.universe + w);
      if (w == eos_w) a |= eos_bit;
      if (w == W - 1) a &= tail;
      partial |= (a != ((w == W - 1) ? tail : 0xFFFFFFFFu));
      if (out) out[w] = a;
      if (APPLY) dep_acc[w] = a;
    }
  }
  trace_mark(P, 1, 7);
  if (need_apply || APPLY) {
    if (partial) s_partial = 1;
    __syncthreads();
    if (need_apply && threadIdx.x == 0) need_apply[i] = (uint8_t)s_partial;
  }
  if (APPLY && s_partial) apply_row(logits + row * lstride_bytes, dep_acc, ap_vocab, ap_eb, ap_neg);
  if (P.trace && threadIdx.x == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    P.trace[64 + 2 * blockIdx.x] = t1 - t_start;
    P.trace[64 + 2 * blockIdx.x + 1] = (unsigned long long)total | ((unsigned long long)nt << 32);
  }
}

template <bool APPLY>
static gm_status fill_attrs() {
  GM_CUDA_TRY(cudaFuncSetAttribute(fill_kernel<APPLY>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  // small shared carveout: the dependent walkers' local state must hit L1
  GM_CUDA_TRY(cudaFuncSetAttribute(fill_kernel<APPLY>, cudaFuncAttributePreferredSharedMemoryCarveout, 25));
  return GM_OK;
}

static size_t fill_smem(int32_t Wmax) {
  const size_t row_bytes = ((size_t)Wmax * 4 + 15) & ~(size_t)15;
  return row_bytes + kStageBytes + (kTmaRows + 1) * row_bytes;
}

gm_status launch_fill(const DevPool& P, const int32_t* slots, int32_t n, int32_t* bitmask, int64_t bstride,
                      const int32_t* rows, uint8_t* need_apply, int32_t Wmax, cudaStream_t s) {
  if (n <= 0) return GM_OK;
  const size_t smem = fill_smem(Wmax);
  if (smem > 220 * 1024) return fail(GM_ERR_INVALID, "vocabulary too large for the fill kernel");
  static gm_status attrs = fill_attrs<false>();
  if (attrs) return attrs;
  fill_kernel<false><<<n, kFillThreads, smem, s>>>(P, slots, n, reinterpret_cast<uint32_t*>(bitmask), bstride, rows,
                                                   need_apply, Wmax, nullptr, 0, 0, 2, 0u);
  GM_LAUNCH_CHECK();
  return GM_OK;
}

// K3: fill + apply in one kernel (no bitmask round trip, one launch).
gm_status launch_fill_apply(const DevPool& P, const int32_t* slots, int32_t n, int32_t* bitmask, int64_t bstride,
                            const int32_t* rows, int32_t Wmax, void* logits, int32_t eb, uint32_t neg,
                            int64_t vocab, int64_t lstride_bytes, cudaStream_t s) {
  if (n <= 0) return GM_OK;
  const size_t smem = fill_smem(Wmax);
  if (smem > 220 * 1024) return fail(GM_ERR_INVALID, "vocabulary too large for the fill kernel");
  static gm_status attrs = fill_attrs<true>();
  if (attrs) return attrs;
  fill_kernel<true><<<n, kFillThreads, smem, s>>>(P, slots, n, reinterpret_cast<uint32_t*>(bitmask), bstride, rows,
                                                  nullptr, Wmax, static_cast<char*>(logits), lstride_bytes, vocab,
                                                  eb, neg);
  GM_LAUNCH_CHECK();
  return GM_OK;
}

}  // namespace gm
