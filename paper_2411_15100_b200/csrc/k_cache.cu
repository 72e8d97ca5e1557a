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
cache_build_kernel(DevGrammar G, DevVocab Vc, DevArena A, int32_t key_begin,
                   uint32_t* __restrict__ acc_rows, uint32_t* __restrict__ dep_rows,
                   uint32_t* __restrict__ err_out) {
  const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= Vc.n_sorted) return;
  const int32_t k = blockIdx.y;
  const int32_t key_node = G.cache_keys[key_begin + k];
  const int32_t tid = __ldg(Vc.sorted_ids + j);
  const int32_t o0 = __ldg(Vc.off + tid);
  const int len = __ldg(Vc.off + tid + 1) - o0;
  const uint8_t* tok = Vc.bytes + o0;

  Walker<kBuildS, kBuildF> w;
  w.reset();
  w.add(-1, key_node);
  uint64_t pops = 0;     // bit d: popped past the frame before byte d
  bool far_pop = false;  // popped at depth >= 64 (treated as "allowed", sound)
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
  if (w.err) atomicOr(err_out, w.err);
  const uint32_t bit = 1u << (tid & 31);
  const size_t word = (size_t)k * Vc.W + (tid >> 5);
  if (w.n > 0) {
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

// Sorted id lists of the dependent rows (REF cache.py:400-402 sorts them).
// One warp per key walks the row in order; ballot + prefix keeps it ordered.
__global__ void dep_compact_kernel(const uint32_t* __restrict__ rows, int32_t W, int32_t n,
                                   const int32_t* __restrict__ dep_off, int32_t* __restrict__ dep_ids) {
  const int32_t k = blockIdx.x;
  if (k >= n || threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  int32_t base = dep_off[k];
  for (int32_t w0 = 0; w0 < W; w0 += 32) {
    const int32_t w = w0 + lane;
    uint32_t bits = w < W ? rows[(size_t)k * W + w] : 0u;
    const int cnt = __popc(bits);
    int incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
      int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    int pos = base + incl - cnt;
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      dep_ids[pos++] = w * 32 + b;
    }
    base += __shfl_sync(0xffffffffu, incl, 31);
  }
}

// One-level context classes of the dependent tokens (compile time).  A
// dependent token of key n dies inside n's rule but for branches that pop
// past n's frame, so its fate depends on the frames below.  For every
// caller c of n's rule (a return node that can sit directly below that
// frame) walk the token from the two-frame stack [c | n]:
//   survives                      -> accepted whatever lies below c
//   dies, no branch pops past c   -> rejected whatever lies below c
//   some branch pops past c       -> needs the request's deeper stack
// The class is or-ed into the record's 4th word (2 bits per caller index);
// the fill then walks only the "deeper" ones (and unknown callers).
// This is an exact refinement of the reference's context-dependent set
// (REF matcher.py:219-237 resolves every one of them by a full walk).
__global__ void dep_context_kernel(DevGrammar G, const int4* __restrict__ tasks, int64_t n_tasks,
                                   uint8_t* __restrict__ dep) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n_tasks) return;
  const int4 tk = tasks[q];  // (entry, caller index, key node, caller node or -1 = root)
  int4* rec = reinterpret_cast<int4*>(dep + (size_t)tk.x * 32);
  const int4 e = rec[0], inl = rec[1];
  const uint8_t* far = dep + e.z;
  const DevArena A{nullptr, 0, nullptr};  // only local frames are touched
  RWalker<8, 48> rw;
  rw.init(nullptr, nullptr, 0);
  // caller -1: the root frame, popping past it ends the walk
  rw.add(tk.w < 0 ? -1 : rw.push(G, A, -1, tk.w), tk.z);
  bool popped = false;
  for (int b = 0; b < e.y && rw.n > 0 && !rw.spill; ++b) {
    bool pb = false;
    rw.step(G, A, rec_byte(inl, far, b), &pb);
    popped |= pb;
  }
  uint32_t cls = kCtxUnknown;
  if (!rw.spill && !rw.err)
    cls = rw.n > 0 ? kCtxAccept : ((popped && tk.w >= 0) ? kCtxDeeper : kCtxReject);
  if (cls) atomicOr(reinterpret_cast<int*>(&rec->w), (int)(cls << (2 * tk.y)));
}

}  // namespace gm

using namespace gm;

namespace gm {
gm_status launch_cache_build(const DevGrammar& G, const DevVocab& V, const DevArena& A,
                             int32_t key_begin, int32_t n, uint32_t* acc, uint32_t* dep,
                             uint32_t* err, cudaStream_t s) {
  if (n <= 0 || V.n_sorted == 0) return GM_OK;
  const int threads = 128;
  for (int32_t k0 = 0; k0 < n; k0 += 65535) {
    const int32_t kn = (n - k0) < 65535 ? (n - k0) : 65535;
    dim3 grid((unsigned)ceil_div(V.n_sorted, threads), (unsigned)kn);
    cache_build_kernel<<<grid, threads, 0, s>>>(G, V, A, key_begin + k0, acc + (size_t)k0 * V.W,
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
gm_status launch_dep_context(const DevGrammar& G, const int4* tasks, int64_t n_tasks, uint8_t* dep, cudaStream_t s) {
  if (n_tasks <= 0) return GM_OK;
  dep_context_kernel<<<(unsigned)ceil_div(n_tasks, 128), 128, 0, s>>>(G, tasks, n_tasks, dep);
  GM_LAUNCH_CHECK();
  return GM_OK;
}
gm_status launch_dep_compact(const uint32_t* rows, int32_t W, int32_t n, const int32_t* off,
                             int32_t* ids, cudaStream_t s) {
  if (n <= 0) return GM_OK;
  dep_compact_kernel<<<n, 32, 0, s>>>(rows, W, n, off, ids);
  GM_LAUNCH_CHECK();
  return GM_OK;
}
}  // namespace gm
