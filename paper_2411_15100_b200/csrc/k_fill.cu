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
#include <cstring>

#include "accept.cuh"

namespace gm {

constexpr int kFillThreads = 512;
// The fused apply's mixed-chunk policy is decided per cache key at build
// (gm_cache_create: K0's thresholds, gm_apply_set_blend, over the key's
// accepted row) and rides in the slot header (flag 4).
// (Measured and rejected: a per-warp-round decision inside the apply loop,
// K5 SQL 43.9 -> 37.9 us/step but XML 19.7 -> 23.0 and JSON +0.7 from the
// per-round ballots; per-row statistics gathered by the merge, +0.3-0.6 us
// on JSON even sampled 1 word in 8.)
constexpr int kTmaRows = 4;     // tops whose rows are TMA-staged (more: direct loads)
constexpr int kDepS = 16;
constexpr int kDepF = 64;
#ifndef GM_DEP_R
#define GM_DEP_R 1
#endif
constexpr int kDepR = GM_DEP_R;  // register walker: stacks
#ifndef GM_DEP_RF
#define GM_DEP_RF 24
#endif
constexpr int kDepRF = GM_DEP_RF;  // register walker: local frames
#ifndef GM_PREFETCH_ROWS
#define GM_PREFETCH_ROWS 0
#endif
constexpr bool kPrefetchRows = GM_PREFETCH_ROWS;  // K5: issue row TMAs from the accept walk
#ifdef GM_NO_DEFER_INTERN
constexpr bool kDeferIntern = false;
#else
constexpr bool kDeferIntern = true;  // K5: fresh frames' CASes by warp 2, verified at the end
#endif
// per-CTA timeline stamps (GMASK_TRACE=1 at run time) exist only in builds
// with -DGM_TIMELINE (tools/trace.sh): the untaken branches cost ~0.2 us/step
#ifdef GM_TIMELINE
constexpr bool kTimeline = true;
#else
constexpr bool kTimeline = false;
#endif


// K3/K5 tail: mask one logits row in place from the finished mask words in
// shared memory (coalesced 16-byte chunks, -inf only where masked, logits
// never read; mixed chunks store just their masked elements, or — rows of
// keys the per-key policy flagged, apply_row_blend2 — are loaded, blended and
// stored whole).  EB = bytes per logit as a template parameter: the chunk
// arithmetic is shifts and masks.  (Measured and rejected: K0's warp-tile scheme here,
// 0.3 us/step slower — the block-contiguous chunk order streams better from
// one SM.)
template <int EB>
__device__ __forceinline__ void apply_row_t(char* __restrict__ rowp, const uint32_t* __restrict__ words,
                                            int64_t tok_lo, int64_t tok_hi, uint32_t neg) {
  // words[] holds the mask from token tok_lo (a multiple of 128) on.  The
  // per-chunk work is kept minimal: no tail test (the ragged last chunk is
  // handled apart), word index and shift from the chunk index, the chunk
  // pointer advanced by a constant (XML K5 16.94 -> 16.81 us/step).
  constexpr int vec = 16 / EB;
  constexpr int cpw = 32 / vec;  // chunks per mask word
  constexpr uint32_t full = (1u << vec) - 1u;
  const int32_t lim = (int32_t)(tok_hi - tok_lo);  // tokens of this span (< 2^31)
  const int32_t whole = lim / vec;                 // chunks entirely inside the span
  char* base = rowp + tok_lo * EB;
  const int32_t stride = (int32_t)blockDim.x;
  char* p = base + (int64_t)threadIdx.x * 16;
  const int64_t pstep = (int64_t)stride * 16;
  for (int32_t c = threadIdx.x; c < whole; c += stride, p += pstep) {
    const uint32_t keep = (words[c / cpw] >> ((c % cpw) * vec)) & full;
    if (keep == full) continue;
    if (keep == 0) {
      st_cs_v4(p, neg);
    } else {  // mixed: only the masked elements
      uint32_t m = ~keep & full;
      while (m) {
        const int j = __ffs(m) - 1;
        m &= m - 1;
        if (EB == 4) st_cs_u32(p + j * 4, neg);
        else st_cs_u16(p + j * 2, neg);
      }
    }
  }
  if (whole * vec < lim && threadIdx.x == (unsigned)(whole % stride)) {  // the ragged last chunk
    const int32_t t0 = whole * vec;
    const uint32_t keep = ((words[t0 >> 5] >> (t0 & 31)) & full) | (full & ~((1u << (lim - t0)) - 1u));
    uint32_t m = ~keep & full;
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      if (EB == 4) st_cs_u32(base + (int64_t)t0 * EB + j * 4, neg);
      else st_cs_u16(base + (int64_t)t0 * EB + j * 2, neg);
    }
  }
}

// The blended apply (2-byte logits), out of line: only rows the per-key
// policy picks call it, and the inline element-store path keeps its code
// layout.  Each thread takes kBlendU chunks per round and issues all their
// loads before any blend: one load in flight per thread left a heavy SQL row
// (every 16-byte chunk mixed) at ~22 us on one SM, bound by load latency
// (K5 SQL 34.0 -> 26.1 us/step with 4 chunks per round, 24.9 with 8).
#ifndef GM_BLEND_U
#define GM_BLEND_U 8
#endif
constexpr int kBlendU = GM_BLEND_U;
__device__ __noinline__ void apply_row_blend2(char* rowp, const uint32_t* words, int64_t tok_lo, int64_t tok_hi,
                                              uint32_t neg) {
  constexpr int vec = 8;
  constexpr uint32_t full = 0xFFu;
  const int32_t lim = (int32_t)(tok_hi - tok_lo);
  const int32_t chunks = (lim + vec - 1) / vec;
  char* base = rowp + tok_lo * 2;
  const int32_t step = (int32_t)blockDim.x;
  for (int32_t c0 = threadIdx.x; c0 < chunks; c0 += kBlendU * step) {
    uint32_t keep[kBlendU];
    uint4 v[kBlendU];
#pragma unroll
    for (int u = 0; u < kBlendU; ++u) {  // masks, then every load of the round
      const int32_t c = c0 + u * step;
      keep[u] = full;
      if (c < chunks) {
        const int32_t t0 = c * vec;
        keep[u] = (words[t0 >> 5] >> (t0 & 31)) & full;
        if (t0 + vec > lim) keep[u] |= full & ~((1u << (lim - t0)) - 1u);
        else if (keep[u] != 0u && keep[u] != full)
          asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                       : "l"(base + (int64_t)t0 * 2));
      }
    }
#pragma unroll
    for (int u = 0; u < kBlendU; ++u) {
      const int32_t c = c0 + u * step;
      if (c >= chunks || keep[u] == full) continue;
      const int32_t t0 = c * vec;
      char* p = base + (int64_t)t0 * 2;
      if (keep[u] == 0u) {
        st_cs_v4(p, neg);
      } else if (t0 + vec <= lim) {  // blend the loaded chunk, one full store
        uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t km = (((keep[u] >> (2 * k)) & 1u) ? 0x0000FFFFu : 0u) |
                              (((keep[u] >> (2 * k + 1)) & 1u) ? 0xFFFF0000u : 0u);
          w[k] = (w[k] & km) | (neg & ~km);
        }
        asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]),
                     "r"(w[3])
                     : "memory");
      } else {  // the span's last chunk: element stores
        uint32_t m = ~keep[u] & full;
        while (m) {
          const int j = __ffs(m) - 1;
          m &= m - 1;
          st_cs_u16(p + j * 2, neg);
        }
      }
    }
  }
}

__device__ __forceinline__ void apply_row(char* __restrict__ rowp, const uint32_t* __restrict__ words, int64_t tok_lo,
                                          int64_t tok_hi, int eb, uint32_t neg, bool blend = false) {
  // the blend path out of line: the element-store loop stays as tight as
  // without it (measured +0.3 us/step on JSON with a runtime flag in the loop)
  if (eb == 4) apply_row_t<4>(rowp, words, tok_lo, tok_hi, neg);
  else if (blend) apply_row_blend2(rowp, words, tok_lo, tok_hi, neg);
  else apply_row_t<2>(rowp, words, tok_lo, tok_hi, neg);
}

// Caller index of a top's parent frame within the callers of the top's
// rule (selects the dependents' one-level context class; kRootCaller for a
// top on the root frame, -1 if unknown) and, with two-level classes, the
// grandparent frame's caller index.
__device__ __forceinline__ void context_of(const DevPool& P, const SlotHdr& hd, const DevGrammar& G, int2 t, int& cj,
                                           int& cj2) {
  cj = kRootCaller;  // the root frame: nothing below it
  cj2 = -1;
  if (t.x < 0) return;
  cj = -1;
  const bool on_chain = hd.nchain > 0 && hd.chain_h[0] == t.x;
  const unsigned long long pk = on_chain ? hd.chain_k[0] : arena_load(P.arena, t.x);
  if (pk >= kTombKey) return;
  const int32_t pn = key_node(pk);
  const int32_t* cr = G.callers + (size_t)G.node_rule[t.y] * kMaxCallers;
  for (int j = 0; j < kRootCaller; ++j) {
    const int32_t c = cr[j];
    if (c < 0) break;
    if (c == pn) { cj = j; break; }
  }
  if (cj < 0 || !G.ctx2) return;
  const int32_t h2 = key_parent(pk);
  if (h2 < 0) {
    cj2 = kRootCaller;  // pn's frame is the bottom one
    return;
  }
  const unsigned long long k2 =
      (on_chain && hd.nchain > 1 && hd.chain_h[1] == h2) ? hd.chain_k[1] : arena_load(P.arena, h2);
  if (k2 >= kTombKey) return;
  const int32_t pn2 = key_node(k2);
  const int32_t* cr2 = G.callers + (size_t)G.node_rule[pn] * kMaxCallers;
  for (int j = 0; j < kRootCaller; ++j) {
    const int32_t c = cr2[j];
    if (c < 0) break;
    if (c == pn2) { cj2 = j; break; }
  }
}

// General and overflow tiers of a dependent walk (rare: the register walker
// spilled).  Walker (<= kDepS stacks, local frames) first, then BigWalk
// (<= kWideCap stacks in the pool's global scratch lanes).  Both look frames
// up by handle, so while a deferred commit's CASes may still be in flight
// (K5) they walk a private copy of the chain rewritten to real handles.
#ifdef GM_DEP_GENERAL_NOINLINE  // measured: the call ABI costs ~3 us/step (K5, JSON)
__device__ __noinline__
#else
__device__ __forceinline__
#endif
bool walk_dep_general(const DevPool* Pp, int32_t slot, const SlotHdr* hd,
                                              const DevGrammar* Gp, int32_t th, int32_t node, int4 e, int4 inl,
                                              const uint8_t* far, const SpecOut* spec, uint32_t* err_out) {
  const DevPool& P = *Pp;
  const DevGrammar& G = *Gp;
  int32_t ch_h[kChain];
  unsigned long long ch_k[kChain];
  const int nc = hd->nchain;
  for (int i = 0; i < nc; ++i) {
    ch_h[i] = hd->chain_h[i];
    ch_k[i] = hd->chain_k[i];
  }
  if (spec && spec->n > 0 && !spec_realize(P.arena, *spec, ch_h, ch_k, nc, &th)) {
    *err_out |= kErrArena;
    return false;
  }
  {
    Walker<kDepS, kDepF> w;
    w.reset();
    w.external(ch_h, ch_k, nc);
    w.add(th < 0 ? -1 : -2 - th, node);
    for (int b = 0; b < e.y; ++b) {
      if (w.nf > kDepF / 2) w.intern_all(P.arena);
      bool pb = false;
      if (!w.template step<kDepS>(G, P.arena, rec_byte(inl, far, b), &pb)) break;
    }
    if (__builtin_expect(!(w.err & kErrCap), 1)) {
      *err_out |= w.err;
      return w.n > 0;
    }
  }
#ifdef GM_DIAG_NO_DEP_BIGWALK
  *err_out |= kErrCap;
  return false;
#endif
  BigWalk bw;
  bw.acquire(P.ovf, (uint32_t)slot * 131u + threadIdx.x);
  bw.start();
  bw.add(th, node);
  for (int b = 0; b < e.y && bw.n > 0 && !bw.err; ++b) {
    bool pb = false;
    bw.step(G, P.arena, rec_byte(inl, far, b), &pb);
  }
  const bool ok = bw.n > 0 && !bw.err;
  *err_out |= bw.err;
  bw.release();
  return ok;
}

// Dependent record di of top t (context indices cj, cj2): decided by its
// context class when possible.  Returns 0 when nothing is left to do (out of
// this split's range, already allowed, rejected, or accepted — bit set in
// dep_acc), 1 when it needs a walk against the request's full stack.
__device__ __forceinline__ int dep_decide(const DevGrammar& G, int32_t di, const int4& e, int cj, int cj2,
                                          uint32_t* dep_acc, int32_t w_lo, int32_t tok_lo, int32_t tok_hi) {
  // two-level class word fetched alongside the record (not after it)
  const uint32_t c2w = cj2 >= 0 ? __ldg(G.ctx2 + (size_t)di * kMaxCallers + cj) : 0u;
  const int32_t tid = e.x;
  if (tid < tok_lo || tid >= tok_hi) return 0;  // another split's token
  uint32_t* acc_w = dep_acc + ((tid >> 5) - w_lo);
  const uint32_t bit = 1u << (tid & 31);
  if (*acc_w & bit) return 0;  // already allowed by another stack
  if (cj >= 0) {
    uint32_t cls = ((uint32_t)e.w >> (2 * cj)) & 3u;
    if (cls == kCtxDeeper && cj2 >= 0)  // two-level class from the grandparent frame
      cls = (c2w >> (2 * cj2)) & 3u;
    if (cls == kCtxReject) return 0;
    if (cls == kCtxAccept) {
      atomicOr(acc_w, bit);
      return 0;
    }
  }
  return 1;
}

// Walk dependent record di (first int4 e) from top t; on success its bit is
// set in dep_acc.  Register walker; general / overflow walkers on spill.
__device__ __forceinline__ void dep_walk(const DevPool& P, int32_t slot, const SlotHdr& hd, const DevGrammar& G,
                                         int32_t di, const int4& e, int2 t, uint32_t* dep_acc, int32_t w_lo,
                                         const SpecOut* spec, int* s_err) {
  const int4 inl = __ldg(hd.dep_ent + 2 * (size_t)di + 1);
  const uint8_t* far = reinterpret_cast<const uint8_t*>(hd.tokrec) + e.z;  // bytes beyond the inline 16
  RWalker<kDepR, kDepRF> rw;
  rw.init(hd.chain_h, hd.chain_k, hd.nchain);
  rw.add(rw.ref_of_handle(t.x), t.y);
  for (int b = 0; b < e.y && rw.n > 0 && !rw.spill; ++b) {
    bool pb = false;
    rw.template step<true>(G, P.arena, rec_byte(inl, far, b), &pb);
  }
  bool ok;
  uint32_t err = 0;
  if (__builtin_expect(!rw.spill, 1)) {
    err = rw.err;
    ok = rw.n > 0;
  } else {
#ifdef GM_DIAG_NO_GENERAL
    err = kErrCap;
    ok = false;
#else
    ok = walk_dep_general(&P, slot, &hd, &G, t.x, t.y, e, inl, far, spec, &err);
#endif
  }
  if (err) {
    slot_error(P, slot, err);
    *s_err = 1;
  }
  if (ok) atomicOr(dep_acc + ((e.x >> 5) - w_lo), 1u << (e.x & 31));
}

// K3/K5 apply overlapped with the dependent walks: the apply warps mask
// every token whose bit is 0 in `base` (cached rows | dependents decided so
// far, AND universe) and that is not `pend`ing a walk; thread `ti` of `nt`.
template <int EB>
__device__ __forceinline__ void apply_row_keep(char* __restrict__ rowp, const uint32_t* __restrict__ base,
                                               const uint32_t* __restrict__ pend, int64_t tok_lo, int64_t tok_hi,
                                               uint32_t neg, int ti, int nthr) {
  constexpr int vec = 16 / EB;
  constexpr uint32_t full = (1u << vec) - 1u;
  const int32_t lim = (int32_t)(tok_hi - tok_lo);
  const int32_t chunks = (lim + vec - 1) / vec;
  char* bp = rowp + tok_lo * EB;
  for (int32_t c = ti; c < chunks; c += nthr) {
    const int32_t t0 = c * vec;
    const int32_t w = t0 >> 5, sh = t0 & 31;
    uint32_t keep = ((base[w] | pend[w]) >> sh) & full;
    const bool tail = t0 + vec > lim;
    if (tail) keep |= full & ~((1u << (lim - t0)) - 1u);
    if (keep == full) continue;
    char* q = bp + t0 * EB;
    if (keep == 0) {
      st_cs_v4(q, neg);
    } else {
      uint32_t m = ~keep & full;
      while (m) {
        const int j = __ffs(m) - 1;
        m &= m - 1;
        if (EB == 4) st_cs_u32(q + j * 4, neg);
        else st_cs_u16(q + j * 2, neg);
      }
    }
  }
}

constexpr int kFillTops = 32;
constexpr int kWalkQueue = 512;
#ifndef GM_OVERLAP_APPLY
#define GM_OVERLAP_APPLY 0  // measured: K5 b2b +0.6 us, cold -2 us (tools/variants J/K/L)
#endif
#ifndef GM_WALK_DIV
#define GM_WALK_DIV 2  // overlap: 1/GM_WALK_DIV of the warps walk, the rest apply
#endif  // overlap: dependent walks queued per CTA (more: walked at once)  // tops per pass of the fill's per-top arrays (wide sets: several passes)

// Tops b0 .. b0+kFillTops of the slot's current ring entry into the fill's
// per-top arrays (key, dependent range, top); returns how many.
__device__ __forceinline__ int load_ring_tops(const DevPool& P, int32_t slot, const SlotHdr& hd, int b0, int32_t* key,
                                              int32_t* lo, int32_t* hi, int2* top) {
  const int32_t h = P.head[slot];
  const int n = P.meta[(size_t)slot * P.H + h] & 0xFFFF;
  const int2* tops = ring_tops(P, slot, h, n);
  const DevGrammar Gg = blob_view(hd.blob);
  const int nb = min(kFillTops, n - b0);
  for (int s = 0; s < nb; ++s) {
    const int2 t = tops[b0 + s];
    const int4 ni = Gg.node_info[t.y];
    key[s] = ni.x;
    lo[s] = ni.y;
    hi[s] = ni.z;
    top[s] = t;
  }
  return nb;
}

// Grid: (requests, splits).  A request's mask is cut into `splits` word
// ranges (multiples of 4 words, i.e. 128 tokens) and each CTA owns one: it
// merges only its slice of the rows, walks only the dependents whose token
// falls in it, stores its slice of the bitmask and masks its slice of the
// logits row.  Header and tables are read by every CTA of the request (one
// round trip each, L2-shared); everything proportional to the vocabulary
// shrinks by the split factor, so small batches still fill the 148 SMs.
// Fused step (ACCEPT): before the fill, thread 0 accepts the request's
// sampled token (K4 semantics, new state written straight into the shared
// header) and optionally restarts a request that just terminated; the fill
// then runs from that state — one launch and one header/table load per
// decode step instead of two.
struct StepArgs {
  const int32_t* tokens;  // null: no accept (first step)
  uint8_t* accepted;
  int32_t recycle;
};

// Token ids carried in the launch parameters (the native decode loop passes
// the host's sampled ids by value: no H2D copy on the step's path).
// Sized to the batch (64 / 128 / 256 / 512 requests): the launch's
// parameter block stays small — above 4 KB of parameters the driver takes a
// slower path (measured: host issue +3 us per step with 512-entry arrays).
constexpr int kParamTokens = 512;
template <int N>
struct TokParams {
  int32_t v[N];     // token ids (when has_tok)
  int32_t slot[N];  // slot ids: the header load needs no global round trip first
  int32_t has_tok;
};

template <bool APPLY, bool ACCEPT>
__device__ __forceinline__ void
fill_body(DevPool P, const int32_t* __restrict__ slots, int32_t n, uint32_t* __restrict__ bitmask,
          int64_t bstride, const int32_t* __restrict__ rows, uint8_t* __restrict__ need_apply, int32_t Wp,
          char* __restrict__ logits, int64_t lstride_bytes, int64_t ap_vocab, int ap_eb, uint32_t ap_neg,
          StepArgs SA, const int32_t* ptok, const int32_t* pslot = nullptr) {
  extern __shared__ __align__(16) uint8_t smem[];
  const size_t part_bytes = ((size_t)Wp * 4 + 15) & ~(size_t)15;
  uint32_t* dep_acc = reinterpret_cast<uint32_t*>(smem);  // [Wp] this CTA's words
  uint8_t* tables = smem + part_bytes;                    // staged blob
  uint8_t* rows_s = tables + kStageBytes;                 // [kTmaRows + 1][part_bytes]
  uint32_t* pend = reinterpret_cast<uint32_t*>(rows_s + (size_t)(kTmaRows + 1) * part_bytes);  // [Wp] walks pending
  __shared__ SlotHdr hd;
  __shared__ int s_partial, s_nt, s_nrows;
  __shared__ int32_t s_key[32], s_lo[32], s_hi[32];
  __shared__ int2 s_top[32];
  __shared__ int s_cj[32], s_cj2[32];
  __shared__ __align__(8) unsigned long long rows_bar;
  __shared__ __align__(8) unsigned long long blob_bar;
  pdl_trigger();
  // the pool's launch hint (immutable grammar blob of the binding every
  // slot shares): staged before the grid dependency wait and the header
  const bool hinted = P.hint_blob != nullptr && blockIdx.x < n;
  if (hinted && threadIdx.x == 0) {
    mbar_init(&blob_bar, (uint32_t)P.hint_blob_bytes);
    bulk_g2s(tables, P.hint_blob, (uint32_t)P.hint_blob_bytes, &blob_bar);
  }
  unsigned long long t_launch = 0;  // diagnostics: CTA resident (before the grid-dependency wait)
  if (kTimeline && P.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_launch));
  pdl_wait();
  const int32_t i = blockIdx.x;
  if (i >= n) return;
  const int32_t split = blockIdx.y, n_split = gridDim.y;
  trace_mark(P, 1, 0);
  unsigned long long t_start = 0, t_hdr = 0, t_setup = 0, t_ctx = 0, t_walks = 0, t_walk = 0, walk_info = 0;
  unsigned long long acc_ts[4] = {0, 0, 0, 0};  // accept: commit start, frames interned, ring written
  unsigned long long t_pref = 0, t_pre = 0;  // accept: frames interned, header state built
  if (kTimeline && P.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  const int32_t slot = pslot ? pslot[i] : __ldg(slots + i);
  const int64_t row = rows ? (int64_t)__ldg(rows + i) : (int64_t)i;
  __shared__ RingPos rp;
  __shared__ int4 s_rec[2];
  __shared__ int s_just_term, s_dirty, s_walked, s_acc, s_err, s_wide, s_nwalk;
  __shared__ int2 s_wq[kWalkQueue];  // overlap: queued dependent walks (record index, top)
  __shared__ SpecOut s_spec;  // K5: fresh frames whose interning is deferred (warp 2, checked at the end)
  int32_t tok = -1;
  const bool do_acc = ACCEPT && (SA.tokens || ptok);
  if (do_acc) {
    // volatile load: `tokens` may be pinned host memory written by the host
    // between graph replays (zero-copy H2D, graph.py), never cached
    if (ptok) tok = ptok[i];
    else asm volatile("ld.global.cv.s32 %0, [%1];" : "=r"(tok) : "l"(SA.tokens + i));
    load_header_ring(P, slot, &hd, &rp);
    // token record from the hinted vocabulary, in the header's round trip
    if (hinted && threadIdx.x < 2 && tok >= 0 && tok < P.hint_V)
      s_rec[threadIdx.x] = __ldg(P.hint_tokrec + 2 * (size_t)tok + threadIdx.x);
  } else {
    load_header(P, slot, &hd);
  }
  __syncthreads();
  // the hint is usable iff this slot is bound to it; otherwise drain the
  // early copy and stage the slot's own blob
  const bool hint_ok = hinted && hd.blob == P.hint_blob && hd.blob_bytes == P.hint_blob_bytes &&
                       hd.tokrec == P.hint_tokrec && hd.V == P.hint_V;
  if (hinted) mbar_wait(&blob_bar, 0);
  trace_mark(P, 1, 1);
  if (kTimeline && P.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_hdr));
  DevGrammar Gs{};
  unsigned long long t_acc = 0;
  const bool vec = (!bitmask || (reinterpret_cast<uintptr_t>(bitmask + row * bstride) & 15) == 0) && (hd.W % 4 == 0);
  __shared__ int s_pref;  // K5: cache rows already in flight (count), -1 none, -2 issued but stale
  if (do_acc) {  // launched with one split: one accept per request
    const bool in_range = tok >= 0 && tok < hd.V;
    if (hint_ok) {
      Gs = blob_view(tables);
    } else {
      if (threadIdx.x < 2 && in_range) s_rec[threadIdx.x] = __ldg(hd.tokrec + 2 * (size_t)tok + threadIdx.x);
      Gs = stage_blob(hd.blob, hd.blob_bytes, tables);  // barrier inside
    }
    if (kTimeline && P.trace && i == 0 && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      P.trace[49] = t;
      P.trace[50] = (unsigned long long)hd.blob_bytes;
    }
    if (threadIdx.x == 0) {
      int acc = 0;
      s_spec.n = 0;
      const bool was_term = hd.flags & 1;
      if (!in_range) {  // REF matcher.py:278-279
        slot_error(P, slot, kErrInvalid);
        acc = kAccErr;
      } else {
        const int4 e = s_rec[0], inl = s_rec[1];
        const uint8_t* far = reinterpret_cast<const uint8_t*>(hd.tokrec) + e.z;
#ifdef GM_TRACE_PROBES
        if (kTimeline && P.trace && i == 0 && hd.ntops > 0) {  // diagnostic: dry walk of the same token, timed
          unsigned long long t0, t1;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
          auto clk = []() { long long t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t) :: "memory"); return t; };
          {  // load-latency probes: generic load of the staged table, its 2nd load, a plain smem load
            const volatile uint8_t* bc = Gs.byte_class;
            long long a0 = clk();
            uint32_t v0 = bc[rec_byte(inl, far, 0)];
            asm volatile("" :: "r"(v0) : "memory");
            long long a1 = clk();
            uint32_t v1 = bc[(v0 + 7) & 255];
            asm volatile("" :: "r"(v1) : "memory");
            long long a2 = clk();
            const volatile int32_t* sk = s_key;
            uint32_t v2 = sk[(v1 + 3) & 31];
            asm volatile("" :: "r"(v2) : "memory");
            long long a3 = clk();
            const volatile int32_t* fst = Gs.fast;
            uint32_t v3 = fst[(v2 + v1) & 63];
            asm volatile("" :: "r"(v3) : "memory");
            long long a4 = clk();
            P.trace[46] = (unsigned long long)(a1 - a0) | ((unsigned long long)(a2 - a1) << 16) |
                          ((unsigned long long)(a3 - a2) << 32) | ((unsigned long long)(a4 - a3) << 48);
            P.trace[47] = v0 + v1 + v2 + v3;
          }
          RWalker<kAccR, kAccRF> rw;
#pragma unroll 1
          for (int it = 0; it < 2; ++it) {
            long long c0 = clock64();
            rw.init(hd.chain_h, hd.chain_k, hd.nchain);
            for (int s = 0; s < hd.ntops && s < kAccR; ++s) rw.add(rw.ref_of_handle(hd.top[s].x), hd.top[s].y);
            long long c1 = clock64();
            P.trace[54 + 5 * it] = (unsigned long long)(c1 - c0);
            for (int b = 0; b < e.y && rw.n > 0 && !rw.spill; ++b) {
              bool pb = false;
              rw.step(Gs, P.arena, rec_byte(inl, far, b), &pb);
              const long long c2 = clock64();
              if (b < 4) P.trace[55 + 5 * it + b] = (unsigned long long)(c2 - c1);
              c1 = c2;
            }
          }
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
          P.trace[51] = t1 - t0;
          P.trace[52] = (unsigned long long)rw.n | ((unsigned long long)e.y << 32);
          P.trace[53] = (unsigned long long)rw.nload | ((unsigned long long)rw.nf << 16) |
                        ((unsigned long long)rw.spill << 32) | ((unsigned long long)hd.nchain << 40) |
                        ((unsigned long long)(hd.top[0].x == hd.chain_h[0]) << 48);
          P.trace[49] = t1;
        }
#endif
        // as soon as the walk has the new tops, start the TMA copies of their
        // cache rows + the universe (the fill needs them) so they overlap
        // the interning and the header publish
        s_pref = -1;
        auto prefetch_rows = [&](const auto& rw) {
          if (kTimeline && P.trace) {
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_walk));
            walk_info = (unsigned long long)e.y | ((unsigned long long)rw.n << 16) | ((unsigned long long)rw.nf << 24);
          }
          if (!vec || rw.n > kTmaRows || !kPrefetchRows) return;
          struct StampPref {  // diagnostics: end of the row prefetch issue
            unsigned long long& t; bool on;
            __device__ ~StampPref() { if (on) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); }
          } stamp_pref{t_pref, kTimeline && P.trace != nullptr};
          const int32_t Wr = hd.W;
          int32_t keys[kTmaRows];
          int nr = 0;
#pragma unroll
          for (int q = 0; q < kTmaRows; ++q) {
            keys[q] = -1;
            if (q < rw.n) {
              keys[q] = Gs.node_info[rw.node[q]].x;
              nr += keys[q] >= 0;
            }
          }
          mbar_init(&rows_bar, (uint32_t)((nr + 1) * (size_t)Wr * 4));
          int k = 0;
#pragma unroll
          for (int q = 0; q < kTmaRows; ++q) {
            if (keys[q] < 0) continue;
            bulk_g2s(rows_s + (size_t)k * part_bytes, hd.acc_rows + (size_t)keys[q] * Wr, (uint32_t)Wr * 4, &rows_bar);
            ++k;
          }
          bulk_g2s(rows_s + (size_t)kTmaRows * part_bytes, hd.universe, (uint32_t)Wr * 4, &rows_bar);
          s_pref = nr;
        };
        if (kTimeline && P.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_pre));
        acc = accept_one(P, slot, rp, hd, Gs, e.y, [&](int64_t b) { return rec_byte(inl, far, (int)b); },
                         tok == hd.eos, e.x != 0, &hd, prefetch_rows, (kTimeline && P.trace) ? acc_ts : nullptr,
                         kDeferIntern ? &s_spec : nullptr);
        if (!(acc & kAccOk) && s_pref >= 0) s_pref = -2;  // walked but not committed: state unchanged, rows stale
      }
      SA.accepted[i] = (uint8_t)acc;
      s_acc = acc;
      s_just_term = !was_term && (hd.flags & 1);
      const bool restart = SA.recycle && (hd.flags & 1);
      if (restart) restart_slot(P, slot, Gs, &hd);
      s_dirty = (acc & kAccOk) || restart;
      if (kTimeline && P.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_acc));
      if (kTimeline && P.trace && i == 0) P.trace[48] = t_acc;
    }
    __syncthreads();
    // publish the new header state (one 16-byte store per lane of warp 0)
    if (s_dirty && threadIdx.x < 32) store_header_state_warp(P, slot, hd, threadIdx.x);
  }
  // deferred interning: warp 2 issues the fresh frames' CASes now and checks
  // their results only at the end of the kernel
  unsigned long long spec_old = kEmptyKey;
  const int spec_lane = (int)threadIdx.x - 64;
  const bool spec_mine = do_acc && spec_lane >= 0 && spec_lane < s_spec.n;
  if (spec_mine)
    spec_old = atomicCAS(P.arena.keys + s_spec.slot[spec_lane], kEmptyKey, s_spec.key[spec_lane]);
  const int32_t W = hd.W;
  const int32_t per = ((W + 3) / 4 + n_split - 1) / n_split * 4;  // words per split
  const int32_t w_lo = min(W, split * per), w_hi = min(W, w_lo + per), nw = w_hi - w_lo;
  const bool terminated = hd.flags & 1;
  const int pref = do_acc ? s_pref : -1;
  // the setup runs on warp 3's lane 0: its mbarrier init fences (MEMBAR)
  // would otherwise wait for the header/ring stores thread 0 just issued
  // (warp 1 computes contexts, warp 2 carries the deferred CASes)
  const unsigned setup_thread = blockDim.x > 96 ? 96u : 0u;
  if (threadIdx.x == setup_thread) {
    s_partial = 0;
    s_wide = 0;
    int nt = hd.ntops;
    if (terminated) {  // a request that terminated in this very step gets an empty row, no error
      // (REF matcher.py:379-381: fill on a terminated matcher raises); K5's
      // accept already reported a terminated slot
      if (split == 0 && !do_acc) slot_error(P, slot, kErrTerminated);
      nt = 0;
    } else if (nt >= 0) {
      // issue the row copies first: they are the longest-latency loads
      if (pref >= 0) {
        s_nrows = pref;  // issued during the accept (K5, one split: w_lo = 0, nw = W)
      } else if (vec && nt <= kTmaRows && nw > 0 && pref == -1) {
        int nr = 0;
        for (int s = 0; s < nt; ++s) nr += hd.key[s] >= 0;
        s_nrows = nr;
        mbar_init(&rows_bar, (uint32_t)((nr + 1) * (size_t)nw * 4));
        int k = 0;
        for (int s = 0; s < nt; ++s) {
          if (hd.key[s] < 0) continue;
          bulk_g2s(rows_s + (size_t)k * part_bytes, hd.acc_rows + (size_t)hd.key[s] * W + w_lo, (uint32_t)nw * 4,
                   &rows_bar);
          ++k;
        }
        bulk_g2s(rows_s + (size_t)kTmaRows * part_bytes, hd.universe + w_lo, (uint32_t)nw * 4, &rows_bar);
      }
      for (int s = 0; s < nt; ++s) {
        s_key[s] = hd.key[s];
        s_lo[s] = hd.dep_lo[s];
        s_hi[s] = hd.dep_hi[s];
        s_top[s] = hd.top[s];
      }
    } else {  // more stacks than the header holds: read the ring entry
      const int32_t h = P.head[slot];
      nt = P.meta[(size_t)slot * P.H + h] & 0xFFFF;
      if (nt > kFillTops) s_wide = nt;  // wide set: kFillTops tops per pass below
      nt = load_ring_tops(P, slot, hd, 0, s_key, s_lo, s_hi, s_top);
    }
    s_nt = nt;
  }
  // K5: the dependents' context indices from the new header, by warp 1 while
  // thread 0 issues the row copies (one phase and one barrier fewer)
  const bool early_ctx = do_acc && hd.ntops >= 0 && !terminated;
  if (early_ctx && threadIdx.x >= 32 && (int)threadIdx.x < 32 + hd.ntops) {
    const int st = threadIdx.x - 32;
    int cj, cj2;
    context_of(P, hd, Gs, hd.top[st], cj, cj2);
    s_cj[st] = cj;
    s_cj2[st] = cj2;
  }
  for (int32_t w = threadIdx.x; w < nw; w += blockDim.x) dep_acc[w] = 0u;
  if (threadIdx.x == 0) {
    s_walked = 0;
    s_err = 0;
    s_nwalk = 0;
  }
  __syncthreads();
  const SpecOut* spec = do_acc ? &s_spec : nullptr;
  trace_mark(P, 1, 2);
  if (kTimeline && P.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_setup));
  int nt = s_nt;
  const bool tma = pref >= 0 || (vec && hd.ntops >= 0 && nt <= kTmaRows && nw > 0 && !terminated && pref == -1);
  if (pref == -2) mbar_wait(&rows_bar, 0);  // drain the stale prefetch before leaving
  // K3/K5: the apply starts before the dependent walks finish.  The walks
  // that context classes cannot decide are queued (their tokens marked
  // pending); half of the warps walk them while the other half mask every
  // token that is neither allowed by the rows / decided dependents nor
  // pending, then the few pending tokens that stayed rejected are masked.
  // Wide sets (several passes) keep the serial order.
  const bool overlap = GM_OVERLAP_APPLY && APPLY && !s_wide;
  const int32_t n_warps = blockDim.x >> 5;
  const int32_t walk_warps = overlap ? n_warps / GM_WALK_DIV : n_warps;
  if (overlap)
    for (int32_t w = threadIdx.x; w < nw; w += blockDim.x) pend[w] = 0u;

  trace_mark(P, 1, 3);
  // one pass over the tops' dependents — several for a wide set (more than
  // kFillTops stacks), each OR-ing its tops' rows into dep_acc
  int total = 0;
  DevGrammar Gd = do_acc ? Gs : hint_ok ? blob_view(tables) : Gs;  // staged below when needed
  bool staged = do_acc || hint_ok;
  for (int b0 = 0;;) {
  total = 0;
  for (int s = 0; s < nt; ++s) total += s_hi[s] - s_lo[s];
  if (kTimeline && P.trace && i == 0 && split == 0 && threadIdx.x == 0) {
    P.trace[16 + 8] = (unsigned long long)total;
    P.trace[16 + 9] = (unsigned long long)(nt > 0 ? s_key[0] : -1);
    P.trace[16 + 10] = (unsigned long long)nt;
  }
  if (total) {
    if (!staged) {
      Gd = stage_blob(hd.blob, hd.blob_bytes, tables);  // barrier inside (total is CTA-uniform)
      staged = true;
    }
    // caller index of each top's parent frame within the callers of the
    // top's rule: selects the dependents' one-level context class
    if (!early_ctx) {
      if ((int)threadIdx.x < nt) {
        int cj, cj2;
        context_of(P, hd, Gd, s_top[threadIdx.x], cj, cj2);
        s_cj[threadIdx.x] = cj;
        s_cj2[threadIdx.x] = cj2;
      }
      __syncthreads();
    }
    trace_mark(P, 1, 4);
    if (kTimeline && P.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_ctx));
    const int32_t tok_lo = w_lo * 32, tok_hi = w_hi * 32;
    // warp-major assignment: consecutive dependents go to different warps, so
    // a handful of walks run in parallel instead of diverging inside one warp
    const int32_t q0 = (threadIdx.x & 31) * n_warps + (threadIdx.x >> 5);
    // the next record is loaded before this one is resolved (the loop is
    // latency-bound for keys with thousands of dependents)
    auto locate = [&](int32_t q, int& s) -> int32_t {  // top of dependent q, its record index
      int base = 0;
      s = 0;
      while (q - base >= s_hi[s] - s_lo[s]) {
        base += s_hi[s] - s_lo[s];
        ++s;
      }
      return s_lo[s] + (q - base);
    };
    int s_next = 0;
    int32_t di_next = q0 < total ? locate(q0, s_next) : 0;
    int4 e_next = q0 < total ? __ldg(hd.dep_ent + 2 * (size_t)di_next) : make_int4(0, 0, 0, 0);
    for (int32_t q = q0; q < total; q += blockDim.x) {
      const int s = s_next;
      const int32_t di = di_next;
      const int4 e = e_next;
      if (q + (int32_t)blockDim.x < total) {
        di_next = locate(q + blockDim.x, s_next);
        e_next = __ldg(hd.dep_ent + 2 * (size_t)di_next);
      }
      if (!dep_decide(Gd, di, e, s_cj[s], s_cj2[s], dep_acc, w_lo, tok_lo, tok_hi)) continue;
      if (kTimeline && P.trace) atomicAdd(&s_walked, 1 | (e.y << 16));  // diagnostics: walks, bytes
      if (overlap) {  // queue the walk, mark the token pending
        const int k = atomicAdd(&s_nwalk, 1);
        if (k < kWalkQueue) {
          s_wq[k] = make_int2(di, s);
          atomicOr(pend + ((e.x >> 5) - w_lo), 1u << (e.x & 31));
          continue;
        }
      }
      dep_walk(P, slot, hd, Gd, di, e, s_top[s], dep_acc, w_lo, spec, &s_err);
    }
  }
  if (!s_wide) break;
  // wide set: this pass's rows into dep_acc, then the next kFillTops tops
  __syncthreads();
  for (int32_t w = threadIdx.x; w < nw; w += blockDim.x) {
    uint32_t a = dep_acc[w];
    for (int s = 0; s < nt; ++s)
      if (s_key[s] >= 0) a |= __ldg(hd.acc_rows + (size_t)s_key[s] * W + w_lo + w);
    dep_acc[w] = a;
  }
  b0 += kFillTops;
  __syncthreads();
  if (b0 >= s_wide) {
    nt = 0;  // every row is in dep_acc already
    break;
  }
  if (threadIdx.x == setup_thread) s_nt = load_ring_tops(P, slot, hd, b0, s_key, s_lo, s_hi, s_top);
  __syncthreads();
  nt = s_nt;
  }
  trace_mark(P, 1, 5);
  __syncthreads();

  uint32_t* out = bitmask ? bitmask + row * bstride : nullptr;
  const int32_t eos_w = hd.eos >> 5;
  const uint32_t eos_bit = (!terminated && (hd.flags & 2)) ? (1u << (hd.eos & 31)) : 0u;
  const uint32_t tail = (hd.V & 31) ? ((1u << (hd.V & 31)) - 1u) : 0xFFFFFFFFu;
  const int64_t vocab = ap_vocab < (int64_t)W * 32 ? ap_vocab : (int64_t)W * 32;
  const int64_t t_lo = (int64_t)w_lo * 32, t_hi = (int64_t)w_hi * 32 < vocab ? (int64_t)w_hi * 32 : vocab;
  uint32_t* base = reinterpret_cast<uint32_t*>(rows_s);  // overlap: rows | decided dependents, AND universe
  if (overlap) {
    const int32_t warp = threadIdx.x >> 5;
    if (warp < walk_warps) {  // walk warps: the queued walks, warp-major
      const int nq = min(s_nwalk, kWalkQueue);
      for (int32_t k = (threadIdx.x & 31) * walk_warps + warp; k < nq; k += walk_warps * 32) {
        const int2 wq = s_wq[k];
        const int4 e = __ldg(hd.dep_ent + 2 * (size_t)wq.x);
        dep_walk(P, slot, hd, Gd, wq.x, e, s_top[wq.y], dep_acc, w_lo, spec, &s_err);
      }
    } else {  // apply warps: base words, then mask all but allowed and pending tokens
      const int ti = (int)threadIdx.x - walk_warps * 32, nthr = (int)blockDim.x - walk_warps * 32;
      if (tma) {
        mbar_wait(&rows_bar, 0);
        const int nr = s_nrows;
        const uint4* univ = reinterpret_cast<const uint4*>(rows_s + (size_t)kTmaRows * part_bytes);
        for (int32_t w4 = ti; w4 < (nw >> 2); w4 += nthr) {
          uint4 a = reinterpret_cast<const uint4*>(dep_acc)[w4];
          for (int k = 0; k < nr; ++k) {
            const uint4 r = reinterpret_cast<const uint4*>(rows_s + (size_t)k * part_bytes)[w4];
            a.x |= r.x; a.y |= r.y; a.z |= r.z; a.w |= r.w;
          }
          const uint4 u = univ[w4];
          uint32_t v[4] = {a.x & u.x, a.y & u.y, a.z & u.z, a.w & u.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int32_t w = w_lo + w4 * 4 + e;
            if (w == eos_w) v[e] |= eos_bit;
            if (w == W - 1) v[e] &= tail;
          }
          reinterpret_cast<uint4*>(base)[w4] = make_uint4(v[0], v[1], v[2], v[3]);
        }
      } else {
        for (int32_t w = w_lo + ti; w < w_hi; w += nthr) {
          uint32_t a = dep_acc[w - w_lo];
          for (int s = 0; s < nt; ++s)
            if (s_key[s] >= 0) a |= __ldg(hd.acc_rows + (size_t)s_key[s] * W + w);
          a &= __ldg(hd.universe + w);
          if (w == eos_w) a |= eos_bit;
          if (w == W - 1) a &= tail;
          base[w - w_lo] = a;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");  // apply warps only: base complete
      if (t_hi > t_lo) {
        char* rowp = logits + row * lstride_bytes;
        if (ap_eb == 4) apply_row_keep<4>(rowp, base, pend, t_lo, t_hi, ap_neg, ti, nthr);
        else apply_row_keep<2>(rowp, base, pend, t_lo, t_hi, ap_neg, ti, nthr);
      }
    }
    __syncthreads();
  }
  trace_mark(P, 1, 6);
  // a walk error this step: the request's flag says so (bit 1) next to
  // whether its token was accepted (bit 0); the slot's error word says which
  if (do_acc && threadIdx.x == 0 && s_err) SA.accepted[i] = (uint8_t)(s_acc | kAccErr);
  if (kTimeline && P.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_walks));

  // Merge and store this CTA's words.
  bool partial = false;
  if (overlap) {
    // final = base | walked dependents; the pending tokens that stayed
    // rejected are the apply's last stores
    char* rowp = logits + row * lstride_bytes;
    for (int32_t w = threadIdx.x; w < nw; w += blockDim.x) {
      const int32_t wg = w_lo + w;
      const uint32_t f = base[w] | dep_acc[w];
      partial |= (f != ((wg == W - 1) ? tail : 0xFFFFFFFFu));
      if (out) out[wg] = f;
      uint32_t m = pend[w] & ~f;
      while (m) {
        const int j = __ffs(m) - 1;
        m &= m - 1;
        const int64_t t = (int64_t)wg * 32 + j;
        if (t < t_hi) {
          if (ap_eb == 4) st_cs_u32(rowp + t * 4, ap_neg);
          else st_cs_u16(rowp + t * 2, ap_neg);
        }
      }
    }
  } else if (tma) {
    mbar_wait(&rows_bar, 0);
    const int nr = s_nrows;
    const uint4* univ = reinterpret_cast<const uint4*>(rows_s + (size_t)kTmaRows * part_bytes);
    for (int32_t w4 = threadIdx.x; w4 < (nw >> 2); w4 += blockDim.x) {
      uint4 a = reinterpret_cast<const uint4*>(dep_acc)[w4];
      for (int k = 0; k < nr; ++k) {
        const uint4 r = reinterpret_cast<const uint4*>(rows_s + (size_t)k * part_bytes)[w4];
        a.x |= r.x; a.y |= r.y; a.z |= r.z; a.w |= r.w;
      }
      const uint4 u = univ[w4];
      uint32_t v[4] = {a.x & u.x, a.y & u.y, a.z & u.z, a.w & u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int32_t w = w_lo + w4 * 4 + e;
        if (w == eos_w) v[e] |= eos_bit;
        if (w == W - 1) v[e] &= tail;
        partial |= (v[e] != ((w == W - 1) ? tail : 0xFFFFFFFFu));
      }
      const uint4 fin = make_uint4(v[0], v[1], v[2], v[3]);
      if (out) reinterpret_cast<uint4*>(out + w_lo)[w4] = fin;
      if (APPLY) reinterpret_cast<uint4*>(dep_acc)[w4] = fin;  // own slot only
    }
  } else {
    for (int32_t w = w_lo + threadIdx.x; w < w_hi; w += blockDim.x) {
      uint32_t a = dep_acc[w - w_lo];
      for (int s = 0; s < nt; ++s) {
        const int32_t kk = s_key[s];
        if (kk >= 0) a |= __ldg(hd.acc_rows + (size_t)kk * W + w);
      }
      a &= __ldg(hd.universe + w);
      if (w == eos_w) a |= eos_bit;
      if (w == W - 1) a &= tail;
      partial |= (a != ((w == W - 1) ? tail : 0xFFFFFFFFu));
      if (out) out[w] = a;
      if (APPLY) dep_acc[w - w_lo] = a;
    }
  }
  trace_mark(P, 1, 7);
  unsigned long long t_merge = 0;
  if (kTimeline && P.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_merge));
  if (need_apply || (APPLY && !overlap)) {
    if (partial) s_partial = 1;
    __syncthreads();
    if (need_apply && threadIdx.x == 0) need_apply[i] = (uint8_t)s_partial;  // launched with one split
  }
  // serial order (wide sets): apply from the final words.  An all-allowed
  // row still masks logits columns in [V, vocab) (their bits are zero, as
  // gm_apply_inplace treats them)
  if (APPLY && !overlap && (s_partial || ap_vocab > (int64_t)hd.V)) {
    // the per-key mixed-chunk policy (header flag 4, decided at cache build)
    const bool blend = hd.flags & 4;
    if (t_hi > t_lo) apply_row(logits + row * lstride_bytes, dep_acc, t_lo, t_hi, ap_eb, ap_neg, blend);
  }
  if (do_acc && threadIdx.x >= 64 && threadIdx.x < 96 && s_spec.n > 0) {  // warp 2: verify the deferred commit
    const bool bad = spec_mine && spec_old != kEmptyKey && spec_old != s_spec.key[spec_lane];
    if (__any_sync(0xFFFFFFFFu, bad) && threadIdx.x == 64 && !spec_fixup(P, slot, s_spec, hd))
      SA.accepted[i] = (uint8_t)(s_acc | kAccErr);
  }
  if (kTimeline && P.trace && threadIdx.x == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    const int64_t c = (int64_t)i * n_split + split;
    if (16 * c + 16 <= 16 * (int64_t)P.capacity) {  // per-CTA timeline (absolute %globaltimer stamps)
      unsigned long long* tr = P.trace + 64 + 16 * c;
      if (P.trace_ring > 0) {  // GMASK_TRACE=2: ring of the last trace_ring launches (back-to-back analysis)
        unsigned long long* cnt = P.trace + 64 + 16 * (int64_t)P.capacity * (1 + P.trace_ring) + c;
        const unsigned long long k = (*cnt)++;
        tr = P.trace + 64 + 16 * (int64_t)P.capacity * (1 + (int64_t)(k % P.trace_ring)) + 16 * c;
        t_pref = t_launch;
      }
      tr[0] = t_start; tr[1] = t_hdr; tr[2] = t_acc; tr[3] = t_setup;
      tr[4] = t_ctx; tr[5] = t_walks; tr[6] = t_merge; tr[7] = t1;
      tr[8] = t_walk;                // accept: register walk done (0: no walk / general path)
      tr[9] = walk_info;             // token bytes | stacks << 16 | walker frames << 24
      tr[10] = (unsigned long long)total | ((unsigned long long)nt << 32) |
               ((unsigned long long)(s_walked & 0xFFFF) << 40);  // dependents, tops, dependents walked
      tr[11] = acc_ts[0];            // accept: frames interned (publish starts)
      tr[12] = t_pre;                // accept_one entered
      tr[13] = t_pref;               // row prefetch issued
      tr[14] = acc_ts[2];            // commit entered (after on_walk)
      tr[15] = acc_ts[3];            // ring entry written (header state next)
    }
    if (c == 0) P.trace[63] = (unsigned long long)n_split;
  }
}

template <bool APPLY, bool ACCEPT>
__global__ void __maxnreg__(128)
fill_kernel(DevPool P, const int32_t* __restrict__ slots, int32_t n, uint32_t* __restrict__ bitmask,
            int64_t bstride, const int32_t* __restrict__ rows, uint8_t* __restrict__ need_apply, int32_t Wp,
            char* __restrict__ logits, int64_t lstride_bytes, int64_t ap_vocab, int ap_eb, uint32_t ap_neg,
            StepArgs SA) {
  fill_body<APPLY, ACCEPT>(P, slots, n, bitmask, bstride, rows, need_apply, Wp, logits, lstride_bytes, ap_vocab,
                           ap_eb, ap_neg, SA, nullptr);
}

// K5 with the token ids in the launch parameters (__grid_constant__: read
// in place from the parameter bank)
template <bool APPLY, int N>
__global__ void __maxnreg__(128)
step_ptok_kernel(DevPool P, const int32_t* __restrict__ slots, int32_t n, uint32_t* __restrict__ bitmask,
                 int64_t bstride, const int32_t* __restrict__ rows, int32_t Wp, char* __restrict__ logits,
                 int64_t lstride_bytes, int64_t ap_vocab, int ap_eb, uint32_t ap_neg, StepArgs SA,
                 const __grid_constant__ TokParams<N> tp) {
  fill_body<APPLY, true>(P, slots, n, bitmask, bstride, rows, nullptr, Wp, logits, lstride_bytes, ap_vocab, ap_eb,
                         ap_neg, SA, tp.has_tok ? tp.v : nullptr, tp.slot);
}

template <bool APPLY, bool ACCEPT>
static gm_status fill_attrs() {
  GM_CUDA_TRY(cudaFuncSetAttribute(fill_kernel<APPLY, ACCEPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   220 * 1024));
  // small shared carveout: the dependent walkers' local state must hit L1
  GM_CUDA_TRY(cudaFuncSetAttribute(fill_kernel<APPLY, ACCEPT>, cudaFuncAttributePreferredSharedMemoryCarveout, 25));
  return GM_OK;
}

// Splits per request: enough CTAs to cover the SMs once,
// at most kMaxSplits; one when the caller wants the per-row need_apply flag.
constexpr int kMaxSplits = 8;
static int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e && *e ? std::atoi(e) : dflt;
}

static int fill_splits(int32_t n, bool need_apply) {
  if (need_apply) return 1;
  static const int forced = env_int("GMASK_FILL_SPLITS", 0);  // diagnostics
  if (forced > 0) return forced > kMaxSplits ? kMaxSplits : forced;
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // one CTA per SM: the walkers' local state needs the L1 a second
  // resident CTA would take (measured: two per SM is slower)
  int s = sms / (n > 0 ? n : 1);
  return s < 1 ? 1 : (s > kMaxSplits ? kMaxSplits : s);
}

// threads per fill CTA: 512 for one CTA per request; with splits the CTAs
// are smaller so two fit per SM (GMASK_FILL_THREADS overrides, diagnostics)
static int fill_threads(int splits) {
  static const int forced = env_int("GMASK_FILL_THREADS", 0);
  if (forced > 0) return forced;
  return splits > 1 ? 256 : kFillThreads;
}

static int32_t split_words(int32_t Wmax, int splits) { return ((Wmax + 3) / 4 + splits - 1) / splits * 4; }

static size_t fill_smem(int32_t Wp) {
  const size_t part = ((size_t)Wp * 4 + 15) & ~(size_t)15;
  return part + kStageBytes + (kTmaRows + 2) * part;
}

gm_status launch_fill(const DevPool& P, const int32_t* slots, int32_t n, int32_t* bitmask, int64_t bstride,
                      const int32_t* rows, uint8_t* need_apply, int32_t Wmax, cudaStream_t s) {
  if (n <= 0) return GM_OK;
  const int splits = fill_splits(n, need_apply != nullptr);
  const int32_t Wp = split_words(Wmax, splits);
  const size_t smem = fill_smem(Wp);
  if (smem > 220 * 1024) return fail(GM_ERR_INVALID, "vocabulary too large for the fill kernel");
  static gm_status attrs = fill_attrs<false, false>();
  if (attrs) return attrs;
  const L2Window win{P.l2_base, P.l2_bytes, P.l2_hit};
  GM_CUDA_TRY(launch_pdl_w(&win, fill_kernel<false, false>, dim3(n, splits), dim3(fill_threads(splits)), smem, s, P, slots, n,
                         reinterpret_cast<uint32_t*>(bitmask), bstride, rows, need_apply, Wp, nullptr, (int64_t)0,
                         (int64_t)0, 2, 0u, StepArgs{nullptr, nullptr, 0}));
  return GM_OK;
}

// K3: fill + apply in one kernel (no bitmask round trip, one launch).
gm_status launch_fill_apply(const DevPool& P, const int32_t* slots, int32_t n, int32_t* bitmask, int64_t bstride,
                            const int32_t* rows, int32_t Wmax, void* logits, int32_t eb, uint32_t neg,
                            int64_t vocab, int64_t lstride_bytes, cudaStream_t s) {
  if (n <= 0) return GM_OK;
  const int splits = fill_splits(n, false);
  const int32_t Wp = split_words(Wmax, splits);
  const size_t smem = fill_smem(Wp);
  if (smem > 220 * 1024) return fail(GM_ERR_INVALID, "vocabulary too large for the fill kernel");
  static gm_status attrs = fill_attrs<true, false>();
  if (attrs) return attrs;
  const L2Window win{P.l2_base, P.l2_bytes, P.l2_hit};
  GM_CUDA_TRY(launch_pdl_w(&win, fill_kernel<true, false>, dim3(n, splits), dim3(fill_threads(splits)), smem, s, P, slots, n,
                         reinterpret_cast<uint32_t*>(bitmask), bstride, rows, nullptr, Wp, static_cast<char*>(logits),
                         lstride_bytes, vocab, (int)eb, neg, StepArgs{nullptr, nullptr, 0}));
  return GM_OK;
}

// K5: accept the sampled tokens, then fill (and, with logits, apply) the next
// masks — one launch per decode step.  One CTA per request (no splits: the
// accept must run once per request).
gm_status launch_step(const DevPool& P, const int32_t* slots, int32_t n, const int32_t* tokens, uint8_t* accepted,
                      int32_t recycle, int32_t* bitmask, int64_t bstride, const int32_t* rows, int32_t Wmax,
                      void* logits, int32_t eb, uint32_t neg, int64_t vocab, int64_t lstride_bytes, cudaStream_t s) {
  if (n <= 0) return GM_OK;
  const size_t smem = fill_smem(split_words(Wmax, 1));
  if (smem > 220 * 1024) return fail(GM_ERR_INVALID, "vocabulary too large for the fill kernel");
  const StepArgs sa{tokens, accepted, recycle};
  const L2Window win{P.l2_base, P.l2_bytes, P.l2_hit};
  uint32_t* bm = reinterpret_cast<uint32_t*>(bitmask);
  if (logits) {
    static gm_status attrs = fill_attrs<true, true>();
    if (attrs) return attrs;
    GM_CUDA_TRY(launch_pdl_w(&win, fill_kernel<true, true>, dim3(n, 1), dim3(fill_threads(1)), smem, s, P, slots, n, bm, bstride,
                           rows, nullptr, split_words(Wmax, 1), static_cast<char*>(logits), lstride_bytes, vocab,
                           (int)eb, neg, sa));
  } else {
    static gm_status attrs = fill_attrs<false, true>();
    if (attrs) return attrs;
    GM_CUDA_TRY(launch_pdl_w(&win, fill_kernel<false, true>, dim3(n, 1), dim3(fill_threads(1)), smem, s, P, slots, n, bm,
                           bstride, rows, nullptr, split_words(Wmax, 1), nullptr, (int64_t)0, (int64_t)0, 2, 0u, sa));
  }
  GM_LAUNCH_CHECK();
  return GM_OK;
}

// K5 from the native decode loop: token ids by value (n <= kParamTokens).
template <bool APPLY, int N>
static gm_status ptok_attrs() {
  GM_CUDA_TRY(cudaFuncSetAttribute(step_ptok_kernel<APPLY, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  GM_CUDA_TRY(cudaFuncSetAttribute(step_ptok_kernel<APPLY, N>, cudaFuncAttributePreferredSharedMemoryCarveout, 25));
  return GM_OK;
}

template <int N>
static gm_status launch_step_ptok_n(const DevPool& P, const int32_t* host_slots, int32_t n, const int32_t* host_tokens,
                                    const int32_t* device_tokens, uint8_t* accepted, int32_t recycle, int32_t* bitmask,
                                    int64_t bstride, int32_t Wmax, void* logits, int32_t eb, uint32_t neg,
                                    int64_t vocab, int64_t lstride_bytes, size_t smem, cudaStream_t s) {
  TokParams<N> tp;
  std::memset(&tp, 0, sizeof(tp));
  if (host_tokens) std::memcpy(tp.v, host_tokens, (size_t)n * 4);
  std::memcpy(tp.slot, host_slots, (size_t)n * 4);
  tp.has_tok = host_tokens != nullptr;
  const int32_t* slots = nullptr;  // the kernel reads tp.slot
  const StepArgs sa{host_tokens ? nullptr : device_tokens, accepted, recycle};
  const L2Window win{P.l2_base, P.l2_bytes, P.l2_hit};
  uint32_t* bm = reinterpret_cast<uint32_t*>(bitmask);
  if (logits) {
    static gm_status attrs = ptok_attrs<true, N>();
    if (attrs) return attrs;
    GM_CUDA_TRY(launch_pdl_w(&win, step_ptok_kernel<true, N>, dim3(n, 1), dim3(fill_threads(1)), smem, s, P, slots, n,
                             bm, bstride, (const int32_t*)nullptr, split_words(Wmax, 1), static_cast<char*>(logits),
                             lstride_bytes, vocab, (int)eb, neg, sa, tp));
  } else {
    static gm_status attrs = ptok_attrs<false, N>();
    if (attrs) return attrs;
    GM_CUDA_TRY(launch_pdl_w(&win, step_ptok_kernel<false, N>, dim3(n, 1), dim3(fill_threads(1)), smem, s, P, slots, n,
                             bm, bstride, (const int32_t*)nullptr, split_words(Wmax, 1), (char*)nullptr, (int64_t)0,
                             (int64_t)0, 2, 0u, sa, tp));
  }
  return GM_OK;
}

// K5 with the slot ids (and, when host_tokens is non-null, the token ids)
// by value in the launch parameters; with host_tokens null the tokens come
// from device_tokens (nullable: no accept, first step).
gm_status launch_step_ptok(const DevPool& P, const int32_t* host_slots, int32_t n, const int32_t* host_tokens,
                           const int32_t* device_tokens, uint8_t* accepted, int32_t recycle, int32_t* bitmask,
                           int64_t bstride, int32_t Wmax, void* logits, int32_t eb, uint32_t neg, int64_t vocab,
                           int64_t lstride_bytes, cudaStream_t s) {
  if (n <= 0) return GM_OK;
  if (n > kParamTokens) return fail(GM_ERR_INVALID, "batch too large for parameter-passed slot / token ids");
  const size_t smem = fill_smem(split_words(Wmax, 1));
  if (smem > 220 * 1024) return fail(GM_ERR_INVALID, "vocabulary too large for the fill kernel");
#define GM_PTOK(N)                                                                                                  \
  return launch_step_ptok_n<N>(P, host_slots, n, host_tokens, device_tokens, accepted, recycle, bitmask, bstride, \
                               Wmax, logits, eb, neg, vocab, lstride_bytes, smem, s)
  if (n <= 64) GM_PTOK(64);
  if (n <= 128) GM_PTOK(128);
  if (n <= 256) GM_PTOK(256);
  GM_PTOK(kParamTokens);
#undef GM_PTOK
}

}  // namespace gm
