// K1 / K1b — adaptive token-mask cache build.
//
// Replaces build_mask_cache (REF cache.py:516-574), whose inner loop sweeps
// every (reachable stack top, token) pair through the byte-level automaton
// (REF cache.py:88-193) and refines context-dependent tokens through the
// follow automaton (REF cache.py:241-333, 551-560).
//
// One thread classifies one (cache key, token) pair.  Threads of a warp take
// consecutive tokens of the lexicographically sorted vocabulary, so their
// walks share prefixes and stay converged on the same table rows (the
// reference exploits the same order with checkpoint rollback).  A token is
//   ACC  if some run consumes all its bytes without popping the key's frame,
//   DEP  if every run dies but some run popped past the frame at depth d and
//        the remainder tok[d:] can still start a legal continuation of the
//        key's rule (K1b: follow-DFA walk, fused into the same thread),
//   REJ  otherwise.
// Classification bits go straight into dense per-key rows (accepted row and
// dependent row, ceil(V/32) words each) with atomicOr; the rows stay
// L2-resident during the build.
#include "device.cuh"

namespace gm {

constexpr int kBuildS = 16;   // stacks per walk
constexpr int kBuildF = 96;   // walker-local frames

__global__ void __launch_bounds__(128)
cache_build_kernel(DevGrammar G, DevVocab Vc, DevArena A, DevOverflow O, int32_t key_begin,
                   const int32_t* __restrict__ key_list, uint32_t* __restrict__ acc_rows,
                   uint32_t* __restrict__ dep_rows, uint32_t* __restrict__ err_out) {
  const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= Vc.n_sorted) return;
  const int32_t k = blockIdx.y;  // row k: key key_list[k] (position sharding) or key_begin + k
  const int32_t key_node = G.cache_keys[key_list ? __ldg(key_list + k) : key_begin + k];
  const int32_t tid = __ldg(Vc.sorted_ids + j);
  const int32_t o0 = __ldg(Vc.off + tid);
  const int len = __ldg(Vc.off + tid + 1) - o0;
  const uint8_t* tok = Vc.bytes + o0;

  uint64_t pops = 0;     // bit d: popped past the frame before byte d
  bool far_pop = false;  // popped at depth >= 64 (treated as "allowed", sound)
  bool alive_end = false;
  uint32_t err = 0;
  {
    Walker<kBuildS, kBuildF> w;
    w.reset();
    w.add(-1, key_node);
    for (int i = 0; i < len; ++i) {
      if (w.nf > kBuildF / 2) w.intern_all(A);
      bool pb = false;
      const int alive = w.template step<kBuildS>(G, A, tok[i], &pb);
      if (pb) {
        if (i < 64) pops |= 1ull << i;
        else far_pop = true;
      }
      if (!alive) break;
    }
    alive_end = w.n > 0;
    err = w.err;
  }
  if (err & kErrCap) {
    // more than kBuildS stacks (ambiguous grammar): redo the walk in the
    // overflow tier, up to the reference's 4096-state cap (REF cache.py:
    // 58, 137-138)
    pops = 0;
    far_pop = false;
    BigWalk bw;
    bw.acquire(O, (uint32_t)j * 7u + (uint32_t)k);
    bw.start();
    bw.add(-1, key_node);
    for (int i = 0; i < len && bw.n > 0 && !bw.err; ++i) {
      bool pb = false;
      bw.step(G, A, tok[i], &pb);
      if (pb) {
        if (i < 64) pops |= 1ull << i;
        else far_pop = true;
      }
    }
    alive_end = bw.n > 0 && !bw.err;
    err = bw.err;
    bw.release();
  }
  if (err) atomicOr(err_out, err);
  const uint32_t bit = 1u << (tid & 31);
  const size_t word = (size_t)k * Vc.W + (tid >> 5);
  if (alive_end) {
    atomicOr(acc_rows + word, bit);
    return;
  }
  if (!pops && !far_pop) return;
  bool keep = far_pop;
  const int32_t rid = G.node_rule[key_node];
  while (!keep && pops) {
    const int d = __ffsll((long long)pops) - 1;
    pops &= pops - 1;
    keep = follow_allows(G, rid, tok + d, len - d);
  }
  if (keep) atomicOr(dep_rows + word, bit);
}

// Dependent-row compaction: per key, the number of dependent tokens.
__global__ void row_popcount_kernel(const uint32_t* __restrict__ rows, int32_t W, int32_t n,
                                    int64_t* __restrict__ out) {
  const int32_t k = blockIdx.x;
  if (k >= n) return;
  int64_t c = 0;
  for (int32_t w = threadIdx.x; w < W; w += blockDim.x) c += __popc(rows[(size_t)k * W + w]);
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __shared__ int64_t part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += part[i];
    out[k] = t;
  }
}

// Mixed-chunk statistics of each accepted row for 2-byte logits (16-byte
// chunk = 8 tokens = one byte of a mask word): out[k] = mixed chunks << 32 |
// their masked elements.  The fused apply's per-key policy (node_info.w bit
// 30, header flag 4) is decided from it on the host.
__global__ void row_mixstats_kernel(const uint32_t* __restrict__ rows, int32_t W, int32_t n,
                                    int64_t* __restrict__ out) {
  const int32_t k = blockIdx.x;
  if (k >= n) return;
  unsigned long long mix = 0, nel = 0;
  for (int32_t w = threadIdx.x; w < W; w += blockDim.x) {
    const uint32_t x = rows[(size_t)k * W + w];
    for (int b = 0; b < 4; ++b) {
      const uint32_t c = (x >> (8 * b)) & 0xFFu;
      if (c != 0u && c != 0xFFu) {
        ++mix;
        nel += 8 - __popc(c);
      }
    }
  }
  unsigned long long v = (mix << 32) | nel;
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __shared__ unsigned long long part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += part[i];
    out[k] = (int64_t)t;
  }
}

// Sorted id lists of the dependent rows (REF cache.py:400-402 sorts them).
// One CTA per key: every thread counts the set bits of a contiguous run of
// words, a block-wide exclusive scan gives each run its output offset, and
// the run is written in order — one pass over the row instead of a serial
// warp walk (82 us -> a few us for JSON at 128k).
constexpr int kCompactThreads = 256;
__global__ void __launch_bounds__(kCompactThreads)
dep_compact_kernel(const uint32_t* __restrict__ rows, int32_t W, int32_t n, const int32_t* __restrict__ dep_off,
                   int32_t* __restrict__ dep_ids) {
  const int32_t k = blockIdx.x;
  if (k >= n) return;
  const uint32_t* row = rows + (size_t)k * W;
  const int32_t per = (W + kCompactThreads - 1) / kCompactThreads;
  const int32_t w0 = min(W, (int32_t)threadIdx.x * per), w1 = min(W, w0 + per);
  int cnt = 0;
  for (int32_t w = w0; w < w1; ++w) cnt += __popc(__ldg(row + w));
  // block exclusive scan of cnt
  __shared__ int warp_sum[kCompactThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_sum[warp] = incl;
  __syncthreads();
  int before = 0;
  for (int j = 0; j < warp; ++j) before += warp_sum[j];
  int pos = dep_off[k] + before + incl - cnt;
  for (int32_t w = w0; w < w1; ++w) {
    uint32_t bits = __ldg(row + w);
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      dep_ids[pos++] = w * 32 + b;
    }
  }
}

// Dependent records: the vocabulary's 32-byte token record (length, offset
// of the full bytes in the vocabulary's record buffer, 16 inline bytes) with
// the token id in word 0 and word 3 cleared for the context classes.
__global__ void dep_records_kernel(const int32_t* __restrict__ ids, int64_t n_dep, const int4* __restrict__ tokrec,
                                   int4* __restrict__ rec) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_dep) return;
  const int32_t t = ids[i];
  int4 r0 = tokrec[2 * (size_t)t];
  r0.x = t;
  r0.w = 0;
  rec[2 * i] = r0;
  rec[2 * i + 1] = tokrec[2 * (size_t)t + 1];
}

// One-level context classes of the dependent tokens (compile time).  A
// dependent token of key n dies inside n's rule but for branches that pop
// past n's frame, so its fate depends on the frames below.  For every
// caller c of n's rule (a return node that can sit directly below that
// frame) walk the token from the two-frame stack [c | n]:
//   survives                      -> accepted whatever lies below c
//   dies, no branch pops past c   -> rejected whatever lies below c
//   some branch pops past c       -> needs the request's deeper stack
// and, for keys of the root rule, from [n] alone (the root frame: popping
// past it ends the walk).  The classes are packed 2 bits per caller index
// into the record's 4th word; the fill then walks only the "deeper" ones and
// unknown callers.  An exact refinement of the reference's context-dependent
// set (REF matcher.py:219-237 resolves every one of them by a full walk).
// One thread per dependent entry.
__device__ uint32_t context_class(const DevGrammar& G, int32_t caller, int32_t node, const int4& e, const int4& inl,
                                  const uint8_t* far) {
  const DevArena A{nullptr, 0, nullptr};  // only local frames are touched
  RWalker<8, 48> rw;
  rw.init(nullptr, nullptr, 0);
  rw.add(caller < 0 ? -1 : rw.push(G, A, -1, caller), node);
  bool popped = false;
  for (int b = 0; b < e.y && rw.n > 0 && !rw.spill; ++b) {
    bool pb = false;
    rw.step(G, A, rec_byte(inl, far, b), &pb);
    popped |= pb;
  }
  if (rw.spill || rw.err) return kCtxUnknown;
  if (rw.n > 0) return kCtxAccept;
  return (popped && caller >= 0) ? kCtxDeeper : kCtxReject;
}

__global__ void dep_context_kernel(DevGrammar G, const int32_t* __restrict__ dep_off, int32_t n_keys, int64_t n_dep,
                                   int4* __restrict__ rec, const uint8_t* __restrict__ tok_base) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_dep) return;
  int32_t lo = 0, hi = n_keys - 1;  // key k: dep_off[k] <= i < dep_off[k+1]
  while (lo < hi) {
    const int32_t mid = (lo + hi + 1) >> 1;
    if (dep_off[mid] <= i) lo = mid;
    else hi = mid - 1;
  }
  const int32_t node = G.cache_keys[lo];
  const int32_t rule = G.node_rule[node];
  const int32_t* cr = G.callers + (size_t)rule * kMaxCallers;
  const int4 e = rec[2 * i], inl = rec[2 * i + 1];
  const uint8_t* far = tok_base + e.z;
  uint32_t w = 0;
  for (int j = 0; j < kRootCaller && cr[j] >= 0; ++j) w |= context_class(G, cr[j], node, e, inl, far) << (2 * j);
  if (rule == G.node_rule[G.start_node]) w |= context_class(G, -1, node, e, inl, far) << (2 * kRootCaller);
  rec[2 * i].w = (int32_t)w;
}

// Two-level context classes: for a dependent whose one-level class at
// caller c1 is "deeper", walk it from [c2 | c1 | n] for every caller c2 of
// c1's rule (and from [c1 | n] with c1's frame at the bottom when c1's rule
// is the root rule, index kRootCaller): accept / reject / still deeper.
// ctx2[dep * kMaxCallers + j] packs the classes over c2 for caller j.  The
// fill uses them when the request's stack has the matching grandparent
// frame, so most "deeper" dependents need no walk at all.
__device__ uint32_t context_class2(const DevGrammar& G, int32_t c2, int32_t c1, int32_t node, const int4& e,
                                   const int4& inl, const uint8_t* far) {
  const DevArena A{nullptr, 0, nullptr};
  RWalker<8, 48> rw;
  rw.init(nullptr, nullptr, 0);
  const int32_t f2 = c2 < 0 ? -1 : rw.push(G, A, -1, c2);
  rw.add(rw.push(G, A, f2, c1), node);
  bool popped = false;
  for (int b = 0; b < e.y && rw.n > 0 && !rw.spill; ++b) {
    bool pb = false;
    rw.step(G, A, rec_byte(inl, far, b), &pb);
    popped |= pb;
  }
  if (rw.spill || rw.err) return kCtxUnknown;
  if (rw.n > 0) return kCtxAccept;
  return (popped && c2 >= 0) ? kCtxDeeper : kCtxReject;
}

__global__ void dep_context2_kernel(DevGrammar G, const int32_t* __restrict__ dep_off, int32_t n_keys, int64_t n_dep,
                                    const int4* __restrict__ rec, const uint8_t* __restrict__ tok_base,
                                    uint32_t* __restrict__ ctx2) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_dep) return;
  int32_t lo = 0, hi = n_keys - 1;
  while (lo < hi) {
    const int32_t mid = (lo + hi + 1) >> 1;
    if (dep_off[mid] <= i) lo = mid;
    else hi = mid - 1;
  }
  const int32_t node = G.cache_keys[lo];
  const int32_t* cr = G.callers + (size_t)G.node_rule[node] * kMaxCallers;
  const int4 e = rec[2 * i], inl = rec[2 * i + 1];
  const uint8_t* far = tok_base + e.z;
  const int32_t root_rule = G.node_rule[G.start_node];
  for (int j = 0; j < kMaxCallers; ++j) {
    uint32_t w = 0;
    const int32_t c1 = j < kRootCaller ? cr[j] : -1;
    if (c1 >= 0 && (((uint32_t)e.w >> (2 * j)) & 3u) == kCtxDeeper) {
      const int32_t r1 = G.node_rule[c1];
      const int32_t* cr2 = G.callers + (size_t)r1 * kMaxCallers;
      for (int j2 = 0; j2 < kRootCaller && cr2[j2] >= 0; ++j2)
        w |= context_class2(G, cr2[j2], c1, node, e, inl, far) << (2 * j2);
      if (r1 == root_rule) w |= context_class2(G, -1, c1, node, e, inl, far) << (2 * kRootCaller);
    }
    ctx2[i * kMaxCallers + j] = w;
  }
}

}  // namespace gm

using namespace gm;

namespace gm {
gm_status launch_cache_build(const DevGrammar& G, const DevVocab& V, const DevArena& A, const DevOverflow& O,
                             int32_t key_begin, const int32_t* key_list, int32_t n, uint32_t* acc, uint32_t* dep,
                             uint32_t* err, cudaStream_t s) {
  if (n <= 0 || V.n_sorted == 0) return GM_OK;
  const int threads = 128;
  for (int32_t k0 = 0; k0 < n; k0 += 65535) {
    const int32_t kn = (n - k0) < 65535 ? (n - k0) : 65535;
    dim3 grid((unsigned)ceil_div(V.n_sorted, threads), (unsigned)kn);
    cache_build_kernel<<<grid, threads, 0, s>>>(G, V, A, O, key_begin + k0, key_list ? key_list + k0 : nullptr,
                                                acc + (size_t)k0 * V.W,
                                                dep + (size_t)k0 * V.W, err);
    GM_LAUNCH_CHECK();
  }
  return GM_OK;
}
gm_status launch_row_popcount(const uint32_t* rows, int32_t W, int32_t n, int64_t* out, cudaStream_t s) {
  if (n <= 0) return GM_OK;
  row_popcount_kernel<<<n, 256, 0, s>>>(rows, W, n, out);
  GM_LAUNCH_CHECK();
  return GM_OK;
}
gm_status launch_row_mixstats(const uint32_t* rows, int32_t W, int32_t n, int64_t* out, cudaStream_t s) {
  if (n <= 0) return GM_OK;
  row_mixstats_kernel<<<n, 256, 0, s>>>(rows, W, n, out);
  GM_LAUNCH_CHECK();
  return GM_OK;
}
gm_status launch_dep_records(const int32_t* ids, int64_t n_dep, const int4* tokrec, int4* rec, cudaStream_t s) {
  if (n_dep <= 0) return GM_OK;
  dep_records_kernel<<<(unsigned)ceil_div(n_dep, 256), 256, 0, s>>>(ids, n_dep, tokrec, rec);
  GM_LAUNCH_CHECK();
  return GM_OK;
}
gm_status launch_dep_context(const DevGrammar& G, const int32_t* dep_off, int32_t n_keys, int64_t n_dep, int4* rec,
                             const uint8_t* tok_base, cudaStream_t s) {
  if (n_dep <= 0) return GM_OK;
  dep_context_kernel<<<(unsigned)ceil_div(n_dep, 128), 128, 0, s>>>(G, dep_off, n_keys, n_dep, rec, tok_base);
  GM_LAUNCH_CHECK();
  return GM_OK;
}
gm_status launch_dep_context2(const DevGrammar& G, const int32_t* dep_off, int32_t n_keys, int64_t n_dep,
                              const int4* rec, const uint8_t* tok_base, uint32_t* ctx2, cudaStream_t s) {
  if (n_dep <= 0) return GM_OK;
  dep_context2_kernel<<<(unsigned)ceil_div(n_dep, 64), 64, 0, s>>>(G, dep_off, n_keys, n_dep, rec, tok_base, ctx2);
  GM_LAUNCH_CHECK();
  return GM_OK;
}
gm_status launch_dep_compact(const uint32_t* rows, int32_t W, int32_t n, const int32_t* off,
                             int32_t* ids, cudaStream_t s) {
  if (n <= 0) return GM_OK;
  dep_compact_kernel<<<n, kCompactThreads, 0, s>>>(rows, W, n, off, ids);
  GM_LAUNCH_CHECK();
  return GM_OK;
}
}  // namespace gm
