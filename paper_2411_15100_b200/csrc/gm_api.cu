// Host side of the C ABI: object lifetimes, uploads, the sorted vocabulary
// index, cache assembly and the matcher pool.  All compute is in the
// k_*.cu kernels; nothing here runs on the per-step path except argument
// marshalling and kernel launches.
#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>
#include <mutex>
#include <set>
#include <unordered_map>
#include <vector>

#include "device.cuh"

namespace gm {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
gm_status fail(gm_status code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

// kernel launchers (k_*.cu)
gm_status launch_cache_build(const DevGrammar&, const DevVocab&, const DevArena&, const DevOverflow&, int32_t,
                             const int32_t*, int32_t, uint32_t*, uint32_t*, uint32_t*, cudaStream_t);
gm_status launch_pool_errors(const DevPool&, const int32_t*, int32_t, uint32_t*, int32_t, cudaStream_t);
gm_status launch_collect(const DevPool&, const int32_t*, int32_t, uint32_t*, uint32_t*, cudaStream_t);
gm_status launch_arena_count(const DevArena&, unsigned long long*, cudaStream_t);
gm_status launch_row_popcount(const uint32_t*, int32_t, int32_t, int64_t*, cudaStream_t);
gm_status launch_dep_compact(const uint32_t*, int32_t, int32_t, const int32_t*, int32_t*, cudaStream_t);
gm_status launch_dep_records(const int32_t*, int64_t, const int4*, int4*, cudaStream_t);
gm_status launch_dep_context(const DevGrammar&, const int32_t*, int32_t, int64_t, int4*, const uint8_t*, cudaStream_t);
gm_status launch_dep_context2(const DevGrammar&, const int32_t*, int32_t, int64_t, const int4*, const uint8_t*,
                              uint32_t*, cudaStream_t);
gm_status launch_fill(const DevPool&, const int32_t*, int32_t, int32_t*, int64_t, const int32_t*,
                      uint8_t*, int32_t, cudaStream_t);
gm_status launch_fill_apply(const DevPool&, const int32_t*, int32_t, int32_t*, int64_t, const int32_t*, int32_t,
                            void*, int32_t, uint32_t, int64_t, int64_t, cudaStream_t);
gm_status launch_l2_touch(void* base, size_t bytes, const L2Window& win);
int32_t apply_blend_policy();
gm_status launch_row_mixstats(const uint32_t*, int32_t, int32_t, int64_t*, cudaStream_t);
gm_status launch_step_ptok(const DevPool&, const int32_t*, int32_t, const int32_t*, const int32_t*, uint8_t*, int32_t,
                           int32_t*, int64_t, int32_t, void*, int32_t, uint32_t, int64_t, int64_t, cudaStream_t);
gm_status launch_step(const DevPool&, const int32_t*, int32_t, const int32_t*, uint8_t*, int32_t, int32_t*, int64_t,
                      const int32_t*, int32_t, void*, int32_t, uint32_t, int64_t, int64_t, cudaStream_t);
gm_status launch_accept_tokens(const DevPool&, const int32_t*, const int32_t*, int32_t, uint8_t*, cudaStream_t);
gm_status launch_accept_bytes(const DevPool&, int32_t, const uint8_t*, int64_t, uint8_t*, cudaStream_t);
gm_status launch_reset(const DevPool&, int32_t, const DevBinding*, int32_t, int32_t, cudaStream_t);
gm_status launch_rollback(const DevPool&, const int32_t*, const int32_t*, int32_t, cudaStream_t);
gm_status launch_recycle(const DevPool&, const int32_t*, int32_t, cudaStream_t);
gm_status launch_fork(const DevPool&, int32_t, int32_t, cudaStream_t);
gm_status launch_probe(const DevPool&, int32_t, int32_t*, int2*, int32_t, uint32_t*, cudaStream_t);

// RAII-less device buffer list: every object frees what it allocated.
struct DevAllocs {
  std::vector<void*> ptrs;
  template <class T>
  gm_status alloc(T** p, size_t count) {
    void* q = nullptr;
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc(&q, count * sizeof(T));
    if (e != cudaSuccess) return fail(GM_ERR_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    ptrs.push_back(q);
    *p = static_cast<T*>(q);
    return GM_OK;
  }
  template <class T>
  gm_status upload(T** p, const T* host, size_t count) {
    gm_status st = alloc(p, count);
    if (st) return st;
    if (count) GM_CUDA_TRY(cudaMemcpy(*p, host, count * sizeof(T), cudaMemcpyHostToDevice));
    return GM_OK;
  }
  void release() {
    for (void* p : ptrs) cudaFree(p);
    ptrs.clear();
  }
};

// Overflow-walker lanes (DevOverflow): `lanes` scratch sets of two
// kWideCap stack buffers + a kHashCap dedupe table each.
static gm_status alloc_overflow(int32_t lanes, DevOverflow* O, std::vector<void*>* owned) {
  *O = DevOverflow{};
  if (lanes <= 0) return GM_OK;
  void *bufs, *hk, *hg, *gen, *lock;
  GM_CUDA_TRY(cudaMalloc(&bufs, (size_t)lanes * 2 * kWideCap * sizeof(int2)));
  GM_CUDA_TRY(cudaMalloc(&hk, (size_t)lanes * kHashCap * 8));
  GM_CUDA_TRY(cudaMalloc(&hg, (size_t)lanes * kHashCap * 4));
  GM_CUDA_TRY(cudaMalloc(&gen, (size_t)lanes * 4));
  GM_CUDA_TRY(cudaMalloc(&lock, (size_t)lanes * 4));
  GM_CUDA_TRY(cudaMemset(hg, 0, (size_t)lanes * kHashCap * 4));
  GM_CUDA_TRY(cudaMemset(gen, 0, (size_t)lanes * 4));
  GM_CUDA_TRY(cudaMemset(lock, 0, (size_t)lanes * 4));
  for (void* q : {bufs, hk, hg, gen, lock}) owned->push_back(q);
  *O = DevOverflow{static_cast<int2*>(bufs), static_cast<unsigned long long*>(hk), static_cast<uint32_t*>(hg),
                   static_cast<uint32_t*>(gen), static_cast<int32_t*>(lock), lanes};
  return GM_OK;
}

static int32_t env_i32(const char* name, int32_t dflt) {
  const char* e = getenv(name);
  return e && *e ? (int32_t)atoi(e) : dflt;
}

// Scratch for cache builds, per host thread (builds on one thread are
// serial: gm_cache_build_rows syncs its stream): an arena for the walkers'
// interned frames, cleared before every build, and overflow lanes.
struct BuildScratch {
  DevArena arena{nullptr, 0, nullptr};
  DevOverflow ovf{};
  uint64_t builds = 0;
  std::vector<void*> owned;
  ~BuildScratch() {
    for (void* q : owned) cudaFree(q);
  }
};
static thread_local BuildScratch g_build;
static gm_status build_scratch(BuildScratch** out, cudaStream_t s) {
  BuildScratch& b = g_build;
  if (!b.arena.keys) {
    const uint32_t cap = 1u << 22;
    unsigned long long* keys = nullptr;
    uint32_t* err = nullptr;
    GM_CUDA_TRY(cudaMalloc(&keys, sizeof(unsigned long long) * cap));
    b.owned.push_back(keys);
    GM_CUDA_TRY(cudaMalloc(&err, sizeof(uint32_t)));
    b.owned.push_back(err);
    b.arena = DevArena{keys, cap - 1, err};
    gm_status st = alloc_overflow(env_i32("GMASK_BUILD_OVF_LANES", 64), &b.ovf, &b.owned);
    if (st) return st;
  }
  // The arena only holds hash-consed (parent, node, term) tuples, valid for
  // any grammar; the walkers intern rarely (local-frame overflow, overflow
  // tier), so it is cleared every 64 builds instead of every build (a 32 MB
  // memset measured +0.7 ms per schema compile).
  if (b.builds++ % 64 == 0)
    GM_CUDA_TRY(cudaMemsetAsync(b.arena.keys, 0xFF, sizeof(unsigned long long) * ((size_t)b.arena.mask + 1), s));
  GM_CUDA_TRY(cudaMemsetAsync(b.arena.err, 0, 4, s));
  *out = &b;
  return GM_OK;
}

static gm_status err_bits_to_status(uint32_t bits, const char* where) {
  if (!bits) return GM_OK;
  std::string w(where);
  if (bits & kErrCap) return fail(GM_ERR_STATE_CAP, w + ": stack set exceeded cap of " + std::to_string(kWideCap));
  if (bits & kErrArena) return fail(GM_ERR_ARENA_FULL, w + ": device stack arena is full");
  if (bits & kErrTerminated) return fail(GM_ERR_TERMINATED, w + ": matcher is terminated");
  if (bits & (1u << GM_ERR_ROLLBACK)) return fail(GM_ERR_ROLLBACK, w + ": cannot roll back beyond history");
  if ((bits & kErrInvalid) && !(bits & 0xF0000000u)) return fail(GM_ERR_INVALID, w + ": token id out of range");
  return fail(GM_ERR_INVALID, w + ": device error (flags 0x" + [&] {
                char b[16];
                snprintf(b, sizeof b, "%x", bits);
                return std::string(b);
              }() + ")");
}

}  // namespace gm

using namespace gm;

// ---------------------------------------------------------------------------
struct gm_vocab {
  DevAllocs mem;
  DevVocab dev;
  std::vector<uint32_t> universe_host;
  std::vector<uint8_t> bytes_host;
  std::vector<int64_t> off_host;
};

struct gm_grammar {
  DevAllocs mem;
  DevGrammar dev;
  std::vector<int32_t> keys;
  std::vector<uint8_t> blob_host;     // grammar blob (BlobHdr + walker tables)
  std::vector<int32_t> key_of_node;
  std::vector<int32_t> node_rule;
};

struct gm_cache {
  DevAllocs mem;
  DevBinding host_binding;
  DevBinding* binding;  // device copy
  int32_t n_keys;
  int32_t n_blend_keys = 0;  // keys whose rows the fused apply blends (policy at build)
};

struct gm_pool {
  DevAllocs mem;
  DevPool dev;
  std::vector<const gm_cache*> slot_cache;           // binding of each slot (null: never bound)
  std::unordered_map<const gm_cache*, int32_t> bound;  // slots per binding
  uint8_t* scratch_bytes;  // accept_bytes staging
  int64_t scratch_cap;
  int32_t* scratch_i32;    // probe outputs
  int32_t max_w;
  uint32_t* gc_mark = nullptr;  // collector bitmaps (arena slots / 32 words each)
  uint32_t* gc_need = nullptr;
  unsigned long long* counts = nullptr;
};

// Pools that may hold bindings to a cache: gm_cache_release unbinds the
// cache from each, so a pool's launch hint never names released memory (a
// freed cache's host struct or device buffers can be reused by the next
// allocation).
static std::mutex g_pools_mu;
static std::set<gm_pool*> g_pools;

extern "C" {
static void refresh_hint(gm_pool* p);

const char* gm_last_error(void) { return g_last_error.c_str(); }
const char* gm_version(void) { return "gmask-b200 0.1 (sm_100a)"; }

// ---------------------------------------------------------------------------
// Vocabulary: REF vocab.py:111-134 (tokens/specials/eos), 227-234 (sorted
// index, ties by id), matcher.py:141-144 (universe).

gm_status gm_vocab_create(const uint8_t* bytes, const int64_t* offsets, int32_t V, const int32_t* special,
                          int32_t n_special, int32_t eos_id, gm_vocab** out) {
  if (V <= 0 || !offsets || !out) return fail(GM_ERR_INVALID, "bad vocabulary arguments");
  if (eos_id < 0 || eos_id >= V) return fail(GM_ERR_INVALID, "eos_id outside vocabulary");
  if (offsets[V] > INT32_MAX) return fail(GM_ERR_INVALID, "vocabulary bytes exceed 2 GiB");
  std::vector<uint8_t> is_special(V, 0);
  for (int32_t i = 0; i < n_special; ++i) {
    if (special[i] < 0 || special[i] >= V) return fail(GM_ERR_INVALID, "special token id outside vocabulary");
    is_special[special[i]] = 1;
  }
  is_special[eos_id] = 1;
  const int32_t W = (V + 31) / 32;
  std::vector<int32_t> off32(V + 1);
  for (int32_t i = 0; i <= V; ++i) off32[i] = (int32_t)offsets[i];
  std::vector<uint8_t> reject(V, 0);
  std::vector<uint32_t> universe(W, 0);
  std::vector<int32_t> ids;
  ids.reserve(V);
  for (int32_t t = 0; t < V; ++t) {
    const bool empty = offsets[t + 1] == offsets[t];
    reject[t] = (is_special[t] || empty) ? 1 : 0;
    if (!reject[t]) {
      universe[t >> 5] |= 1u << (t & 31);
      ids.push_back(t);
    }
  }
  std::sort(ids.begin(), ids.end(), [&](int32_t a, int32_t b) {
    const uint8_t* pa = bytes + offsets[a];
    const uint8_t* pb = bytes + offsets[b];
    const int64_t la = offsets[a + 1] - offsets[a], lb = offsets[b + 1] - offsets[b];
    const int c = std::memcmp(pa, pb, (size_t)std::min(la, lb));
    if (c != 0) return c < 0;
    if (la != lb) return la < lb;
    return a < b;
  });
  // 32-byte token records (reject, len, far offset, 0) + 16 inline bytes,
  // followed by all token bytes; far offset is relative to the buffer start
  const size_t rec_bytes = (size_t)V * 32;
  std::vector<uint8_t> recbuf(rec_bytes + (size_t)offsets[V] + 16, 0);
  for (int32_t t = 0; t < V; ++t) {
    const int64_t o0 = offsets[t], len = offsets[t + 1] - o0;
    int32_t hdr4[4] = {reject[t], (int32_t)len, (int32_t)(rec_bytes + o0), 0};
    std::memcpy(recbuf.data() + (size_t)t * 32, hdr4, 16);
    std::memcpy(recbuf.data() + (size_t)t * 32 + 16, bytes + o0, (size_t)std::min<int64_t>(len, 16));
  }
  if (offsets[V]) std::memcpy(recbuf.data() + rec_bytes, bytes, (size_t)offsets[V]);
  gm_vocab* v = new gm_vocab();
  gm_status st;
  uint8_t* d_rec;
  uint8_t* d_bytes;
  int32_t *d_off, *d_sorted;
  uint32_t* d_univ;
  uint8_t* d_rej;
  if ((st = v->mem.upload(&d_bytes, bytes, (size_t)offsets[V])) ||
      (st = v->mem.upload(&d_off, off32.data(), off32.size())) ||
      (st = v->mem.upload(&d_sorted, ids.data(), ids.size())) ||
      (st = v->mem.upload(&d_univ, universe.data(), universe.size())) ||
      (st = v->mem.upload(&d_rej, reject.data(), reject.size())) ||
      (st = v->mem.upload(&d_rec, recbuf.data(), recbuf.size()))) {
    v->mem.release();
    delete v;
    return st;
  }
  v->dev = DevVocab{V, W, (int32_t)ids.size(), eos_id, d_bytes, d_off, d_sorted, d_univ, d_rej,
                    reinterpret_cast<const int4*>(d_rec)};
  v->universe_host = std::move(universe);
  v->bytes_host.assign(bytes, bytes + offsets[V]);
  v->off_host.assign(offsets, offsets + V + 1);
  *out = v;
  return GM_OK;
}

void gm_vocab_release(gm_vocab* v) {
  if (!v) return;
  v->mem.release();
  delete v;
}
int32_t gm_vocab_size(const gm_vocab* v) { return v ? v->dev.V : 0; }
const int32_t* gm_vocab_universe(const gm_vocab* v) {
  return v ? reinterpret_cast<const int32_t*>(v->dev.universe) : nullptr;
}

// ---------------------------------------------------------------------------
gm_status gm_grammar_create(const gm_grammar_tables* t, gm_grammar** out) {
  if (!t || !out) return fail(GM_ERR_INVALID, "null tables");
  if (t->n_nodes <= 0 || t->n_classes <= 0 || t->n_rules <= 0) return fail(GM_ERR_INVALID, "empty automaton");
  if (t->start_node < 0 || t->start_node >= t->n_nodes) return fail(GM_ERR_INVALID, "bad start node");
  for (int b = 0; b < 256; ++b)
    if (t->byte_class[b] >= t->n_classes) return fail(GM_ERR_INVALID, "byte class out of range");
  const int64_t n_idx = (int64_t)t->n_nodes * t->n_classes;
  if (t->trans_off[0] != 0 || t->trans_off[n_idx] != t->n_trans) return fail(GM_ERR_INVALID, "bad transition CSR");
  for (int32_t i = 0; i < t->n_trans; ++i) {
    const int32_t d = t->trans[2 * i];
    const uint32_t pk = (uint32_t)t->trans[2 * i + 1];
    const uint32_t poff = pk & 0xFFFFFF, plen = pk >> 24;
    if (d < 0 || d >= t->n_nodes || poff + plen > (uint32_t)t->n_push)
      return fail(GM_ERR_INVALID, "transition out of range");
  }
  std::vector<int32_t> key_of_node(t->n_nodes, -1);
  for (int32_t k = 0; k < t->n_keys; ++k) {
    const int32_t nd = t->cache_keys[k];
    if (nd < 0 || nd >= t->n_nodes) return fail(GM_ERR_INVALID, "cache key out of range");
    key_of_node[nd] = k;
  }
  // walker tables in one contiguous 16-byte aligned blob (staged into shared
  // memory by the fill/accept kernels)
  std::vector<uint8_t> blob(sizeof(BlobHdr), 0);
  auto put = [&](const void* src, size_t bytes) {
    size_t off = (blob.size() + 15) & ~size_t(15);
    blob.resize(off + ((bytes + 15) & ~size_t(15)), 0);
    if (bytes) std::memcpy(blob.data() + off, src, bytes);
    return off;
  };
  const size_t o_bc = put(t->byte_class, 256);
  const size_t o_flags = put(t->node_flags, (size_t)t->n_nodes);
  const size_t o_toff = put(t->trans_off, ((size_t)n_idx + 1) * 4);
  const size_t o_trans = put(t->trans, (size_t)t->n_trans * 8);
  const size_t o_pool = put(t->push_pool, (size_t)t->n_push * 4);
  const size_t o_kon = put(key_of_node.data(), key_of_node.size() * 4);
  const size_t o_rule = put(t->node_rule, (size_t)t->n_nodes * 4);
  // single-stack fast path: for (node, class) the whole byte step when it is
  // a plain DFA move (node cannot pop, exactly one transition, no push, the
  // target is not a spent final): target >= 0; -1 = dies; -2 = general step
  //
  // A node that can pop (its rule may be complete) still gets a fast entry
  // for a class no continuation after the pop can consume: FOLLOW(rule) =
  // the classes with a transition at a return node that can sit below a
  // frame of the rule, plus FOLLOW of that node's rule when it can pop too
  // (fixpoint).  Such entries are encoded -3 - target (kFastPopDies: dies)
  // and taken only above the bottom frame, so the synthetic-bottom walks of
  // the cache build still see their pop-past-bottom flag.  Identifier and
  // number runs inside nested rules (SQL, arithmetic) become table moves.
  const int32_t C = t->n_classes;
  std::vector<std::vector<int32_t>> returns(t->n_rules);
  for (int32_t i = 0; i < t->n_trans; ++i) {
    const int32_t d = t->trans[2 * i];
    const uint32_t pk = (uint32_t)t->trans[2 * i + 1];
    const uint32_t poff = pk & 0xFFFFFF, plen = pk >> 24;
    for (uint32_t k = 0; k < plen; ++k) {
      const int32_t r = t->node_rule[k + 1 < plen ? t->push_pool[poff + k + 1] : d];
      if (r >= 0 && r < t->n_rules) returns[r].push_back(t->push_pool[poff + k]);
    }
  }
  std::vector<std::vector<char>> follow(t->n_rules, std::vector<char>((size_t)C, 0));
  for (bool changed = true; changed;) {
    changed = false;
    for (int32_t r = 0; r < t->n_rules; ++r)
      for (const int32_t ret : returns[r]) {
        const int32_t rr = t->node_rule[ret];
        for (int32_t c = 0; c < C; ++c) {
          if (follow[r][c]) continue;
          const int64_t idx = (int64_t)ret * C + c;
          const bool f = t->trans_off[idx + 1] > t->trans_off[idx] ||
                         ((t->node_flags[ret] & GM_NODE_POP) && rr >= 0 && rr < t->n_rules && follow[rr][c]);
          if (f) { follow[r][c] = 1; changed = true; }
        }
      }
  }
  std::vector<int32_t> fast((size_t)n_idx);
  for (int32_t u = 0; u < t->n_nodes; ++u)
    for (int32_t c = 0; c < C; ++c) {
      const int64_t idx = (int64_t)u * C + c;
      const int32_t t0 = t->trans_off[idx], t1 = t->trans_off[idx + 1];
      const bool pops = t->node_flags[u] & GM_NODE_POP;
      const int32_t ru = t->node_rule[u];
      if (pops && (ru < 0 || ru >= t->n_rules || follow[ru][c])) {
        fast[(size_t)idx] = -2;
        continue;
      }
      int32_t d = -2;  // plain move target, -1 dies, -2 general
      if (t1 == t0) {
        d = -1;
      } else if (t1 - t0 == 1) {
        const int32_t dd = t->trans[2 * t0];
        const uint32_t plen = (uint32_t)t->trans[2 * t0 + 1] >> 24;
        if (plen == 0 && !(t->node_flags[dd] & GM_NODE_DEAD_END)) d = dd;
      }
      fast[(size_t)idx] = !pops ? d : d >= 0 ? -3 - d : d == -1 ? kFastPopDies : -2;
    }
  const size_t o_fast = put(fast.data(), fast.size() * 4);
  // callers[rule]: the return nodes a push run leaves directly below a frame
  // of that rule (the frame under a pushed p_{i+1} holds p_i; under the
  // run's target, the last pushed node).  Frames only ever get parents this
  // way, so the set is exact; a rule with more than kRootCaller callers keeps
  // the first ones and the fill walks for the rest.
  std::vector<int32_t> callers((size_t)t->n_rules * kMaxCallers, -1);
  std::vector<int32_t> n_callers(t->n_rules, 0);
  auto add_caller = [&](int32_t below_of, int32_t ret) {
    const int32_t r = t->node_rule[below_of];
    if (r < 0 || r >= t->n_rules) return;
    int32_t* c = callers.data() + (size_t)r * kMaxCallers;
    for (int j = 0; j < n_callers[r]; ++j)
      if (c[j] == ret) return;
    if (n_callers[r] < kRootCaller) c[n_callers[r]++] = ret;
  };
  for (int32_t i = 0; i < t->n_trans; ++i) {
    const int32_t d = t->trans[2 * i];
    const uint32_t pk = (uint32_t)t->trans[2 * i + 1];
    const uint32_t poff = pk & 0xFFFFFF, plen = pk >> 24;
    for (uint32_t k = 0; k < plen; ++k)
      add_caller(k + 1 < plen ? t->push_pool[poff + k + 1] : d, t->push_pool[poff + k]);
  }
  const size_t o_callers = put(callers.data(), callers.size() * 4);
  if (blob.size() > (size_t)INT32_MAX) return fail(GM_ERR_INVALID, "automaton tables too large");
  BlobHdr bh{};
  bh.bytes = (int32_t)blob.size();
  bh.n_classes = t->n_classes;
  bh.n_nodes = t->n_nodes;
  bh.o_bc = (int32_t)o_bc;
  bh.o_flags = (int32_t)o_flags;
  bh.o_toff = (int32_t)o_toff;
  bh.o_trans = (int32_t)o_trans;
  bh.o_pool = (int32_t)o_pool;
  bh.o_kon = (int32_t)o_kon;
  bh.o_rule = (int32_t)o_rule;
  bh.o_ninfo = 0;
  bh.o_fast = (int32_t)o_fast;
  bh.o_callers = (int32_t)o_callers;
  bh.start_node = t->start_node;
  std::memcpy(blob.data(), &bh, sizeof(bh));
  gm_grammar* g = new gm_grammar();
  gm_status st;
  uint8_t* d_blob;
  int32_t *keys, *fstart, *fnext;
  if ((st = g->mem.upload(&d_blob, blob.data(), blob.size())) ||
      (st = g->mem.upload(&keys, t->cache_keys, (size_t)t->n_keys)) ||
      (st = g->mem.upload(&fstart, t->follow_start, (size_t)t->n_rules)) ||
      (st = g->mem.upload(&fnext, t->follow_next, (size_t)t->n_fstates * t->n_classes))) {
    g->mem.release();
    delete g;
    return st;
  }
  DevGrammar& G = g->dev;
  G.n_nodes = t->n_nodes;
  G.n_rules = t->n_rules;
  G.n_classes = t->n_classes;
  G.start_node = t->start_node;
  G.n_keys = t->n_keys;
  G.n_fstates = t->n_fstates;
  G.byte_class = d_blob + o_bc;
  G.node_flags = d_blob + o_flags;
  G.trans_off = reinterpret_cast<const int32_t*>(d_blob + o_toff);
  G.trans = reinterpret_cast<const int2*>(d_blob + o_trans);
  G.push_pool = reinterpret_cast<const int32_t*>(d_blob + o_pool);
  G.key_of_node = reinterpret_cast<const int32_t*>(d_blob + o_kon);
  G.node_rule = reinterpret_cast<const int32_t*>(d_blob + o_rule);
  G.cache_keys = keys;
  G.follow_start = fstart;
  G.follow_next = fnext;
  G.node_info = nullptr;
  G.fast = reinterpret_cast<const int32_t*>(d_blob + o_fast);
  G.callers = reinterpret_cast<const int32_t*>(d_blob + o_callers);
  G.blob = d_blob;
  G.blob_bytes = (int32_t)blob.size();
  g->keys.assign(t->cache_keys, t->cache_keys + t->n_keys);
  g->blob_host = std::move(blob);
  g->key_of_node = std::move(key_of_node);
  g->node_rule.assign(t->node_rule, t->node_rule + t->n_nodes);
  *out = g;
  return GM_OK;
}

void gm_grammar_release(gm_grammar* g) {
  if (!g) return;
  g->mem.release();
  delete g;
}

// ---------------------------------------------------------------------------
// Rows of cache keys [key_begin, key_begin + n), or of the keys listed in
// host array key_list[0..n) (position sharding: any subset in any order).
static gm_status cache_build(const gm_grammar* g, const gm_vocab* v, int32_t key_begin, const int32_t* key_list,
                             int32_t n, int32_t* acc_rows, int32_t* dep_rows, void* stream) {
  if (!g || !v) return fail(GM_ERR_INVALID, "null grammar/vocab");
  if (n < 0) return fail(GM_ERR_INVALID, "negative key count");
  if (key_list) {
    for (int32_t k = 0; k < n; ++k)
      if (key_list[k] < 0 || key_list[k] >= g->dev.n_keys) return fail(GM_ERR_INVALID, "key index out of bounds");
  } else if (key_begin < 0 || key_begin + n > g->dev.n_keys) {
    return fail(GM_ERR_INVALID, "key range out of bounds");
  }
  if (n == 0) return GM_OK;
  cudaStream_t s = as_stream(stream);
  const size_t bytes = (size_t)n * v->dev.W * 4;
  GM_CUDA_TRY(cudaMemsetAsync(acc_rows, 0, bytes, s));
  GM_CUDA_TRY(cudaMemsetAsync(dep_rows, 0, bytes, s));
  BuildScratch* B;
  gm_status st = build_scratch(&B, s);
  if (st) return st;
  int32_t* d_keys = nullptr;
  if (key_list) {
    GM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d_keys), (size_t)n * 4, s));
    GM_CUDA_TRY(cudaMemcpyAsync(d_keys, key_list, (size_t)n * 4, cudaMemcpyHostToDevice, s));
  }
  st = launch_cache_build(g->dev, v->dev, B->arena, B->ovf, key_begin, d_keys, n,
                          reinterpret_cast<uint32_t*>(acc_rows), reinterpret_cast<uint32_t*>(dep_rows),
                          B->arena.err, s);
  if (d_keys) cudaFreeAsync(d_keys, s);
  if (st) return st;
  uint32_t bits = 0;
  GM_CUDA_TRY(cudaMemcpyAsync(&bits, B->arena.err, 4, cudaMemcpyDeviceToHost, s));
  GM_CUDA_TRY(cudaStreamSynchronize(s));
  return err_bits_to_status(bits, "cache build");
}

gm_status gm_cache_build_rows(const gm_grammar* g, const gm_vocab* v, int32_t key_begin, int32_t n,
                              int32_t* acc_rows, int32_t* dep_rows, void* stream) {
  return cache_build(g, v, key_begin, nullptr, n, acc_rows, dep_rows, stream);
}

gm_status gm_cache_build_keys(const gm_grammar* g, const gm_vocab* v, const int32_t* key_list, int32_t n,
                              int32_t* acc_rows, int32_t* dep_rows, void* stream) {
  if (n > 0 && !key_list) return fail(GM_ERR_INVALID, "null key list");
  return cache_build(g, v, 0, key_list, n, acc_rows, dep_rows, stream);
}

int32_t gm_grammar_num_keys(const gm_grammar* g) { return g ? g->dev.n_keys : 0; }

gm_status gm_cache_create(const gm_grammar* g, const gm_vocab* v, const int32_t* acc_rows,
                          const int32_t* dep_rows, gm_cache** out, gm_cache_stats* stats, void* stream) {
  if (!g || !v || !out) return fail(GM_ERR_INVALID, "null argument");
  cudaStream_t s = as_stream(stream);
  const int32_t n = g->dev.n_keys, W = v->dev.W;
  gm_cache* c = new gm_cache();
  gm_status st;
  auto bail = [&](gm_status e) {
    c->mem.release();
    delete c;
    return e;
  };
  // phase 1 (one allocation): the cache's own accepted rows + row counts
  const size_t rows_bytes = (size_t)n * W * 4;
  const size_t off_counts = (rows_bytes + 15) & ~size_t(15);
  uint8_t* buf1;
  if ((st = c->mem.alloc(&buf1, off_counts + (size_t)(3 * n + 1) * 8))) return bail(st);
  uint32_t* acc = reinterpret_cast<uint32_t*>(buf1);
  int64_t* counts = reinterpret_cast<int64_t*>(buf1 + off_counts);
  std::vector<int64_t> cnt(3 * (size_t)n);
  if (n) {
    GM_CUDA_TRY(cudaMemcpyAsync(acc, acc_rows, rows_bytes, cudaMemcpyDeviceToDevice, s));
    if ((st = launch_row_popcount(reinterpret_cast<const uint32_t*>(dep_rows), W, n, counts, s))) return bail(st);
    if ((st = launch_row_popcount(acc, W, n, counts + n, s))) return bail(st);
    if ((st = launch_row_mixstats(acc, W, n, counts + 2 * n, s))) return bail(st);
    GM_CUDA_TRY(cudaMemcpyAsync(cnt.data(), counts, (size_t)3 * n * 8, cudaMemcpyDeviceToHost, s));
    GM_CUDA_TRY(cudaStreamSynchronize(s));
  }
  std::vector<int32_t> off(n + 1, 0);
  int64_t dep_total = 0, acc_total = 0;
  for (int32_t k = 0; k < n; ++k) {
    dep_total += cnt[k];
    acc_total += cnt[(size_t)n + k];
    if (dep_total > INT32_MAX) return bail(fail(GM_ERR_INVALID, "too many dependent tokens"));
    off[k + 1] = (int32_t)dep_total;
  }
  // Fused-apply policy per key (2-byte logits): a row whose 16-byte chunks
  // are densely mixed and heavily masked (SQL identifier classes) is applied
  // with loaded + blended full-chunk stores instead of element stores.  The
  // thresholds are K0's (gm_apply_set_blend at build time) scaled from its
  // 1,024-token tile to the row; decided here from the accepted row so the
  // step kernels pay nothing per step (per-step statistics measured +0.3 us
  // on JSON).  A step blends when a top's key has the flag (header flag 4)
  // and the runtime policy is non-zero.
  const int32_t policy = apply_blend_policy();
  std::vector<uint8_t> blend_key(n, 0);
  for (int32_t k = 0; k < n && policy > 0; ++k) {
    const int64_t mix = (int64_t)((uint64_t)cnt[2 * (size_t)n + k] >> 32);
    const int64_t nel = (int64_t)((uint64_t)cnt[2 * (size_t)n + k] & 0xFFFFFFFFu);
    blend_key[k] = mix > 0 && 128 * mix >= (int64_t)(policy & 0xFF) * (int64_t)W * 4 &&
                   nel >= (int64_t)((policy >> 8) & 0xFF) * mix;
  }
  c->n_blend_keys = 0;
  for (int32_t k = 0; k < n; ++k) c->n_blend_keys += blend_key[k];
  // binding blob: grammar blob + node_info (key, dep_lo, dep_hi, rule | blend << 30) per node
  std::vector<uint8_t> bblob = g->blob_host;
  const size_t o_ninfo = (bblob.size() + 15) & ~size_t(15);
  bblob.resize(o_ninfo + (size_t)g->dev.n_nodes * 16, 0);
  for (int32_t nd = 0; nd < g->dev.n_nodes; ++nd) {
    const int32_t k = g->key_of_node[nd];
    int32_t ni[4] = {k, k >= 0 ? off[k] : 0, k >= 0 ? off[k + 1] : 0,
                     g->node_rule[nd] | ((k >= 0 && blend_key[k]) ? (1 << 30) : 0)};
    std::memcpy(bblob.data() + o_ninfo + (size_t)nd * 16, ni, 16);
  }
  BlobHdr bh;
  std::memcpy(&bh, bblob.data(), sizeof(bh));
  bh.o_ninfo = (int32_t)o_ninfo;
  bh.bytes = (int32_t)bblob.size();
  std::memcpy(bblob.data(), &bh, sizeof(bh));
  // phase 2 (one allocation): dep_off | dep_ids | dependent records | blob |
  // binding; host-side pieces go up in one copy
  auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t o_off = 0, o_ids = align((size_t)(n + 1) * 4), o_rec = o_ids + align((size_t)dep_total * 4 + 4);
  const size_t o_blob = o_rec + align((size_t)dep_total * 32 + 32), o_bind = o_blob + align(bblob.size());
  const size_t o_ctx2 = align(o_bind + sizeof(DevBinding));
  const size_t total = o_ctx2 + (size_t)dep_total * kMaxCallers * 4 + 4;
  uint8_t* buf2;
  if ((st = c->mem.alloc(&buf2, total))) return bail(st);
  // two-level context classes: opt-in (GMASK_TWO_LEVEL=1).  The median
  // request walks ~4x fewer dependents on JSON (0.1 us/step faster), but
  // XML-like keys with 10^4 dependents pay an extra load each (+4.6 us/step)
  // and the precompute costs up to 100 ms per schema (config 5)
  const char* tl = getenv("GMASK_TWO_LEVEL");
  const bool two_level = tl && tl[0] == '1';
  uint32_t* ctx2 = two_level ? reinterpret_cast<uint32_t*>(buf2 + o_ctx2) : nullptr;
  {  // the binding blob carries the two-level context table's address (0: off)
    const unsigned long long a = reinterpret_cast<unsigned long long>(ctx2);
    bh.ctx2_lo = (uint32_t)a;
    bh.ctx2_hi = (uint32_t)(a >> 32);
    std::memcpy(bblob.data(), &bh, sizeof(bh));
  }
  int32_t* dep_off = reinterpret_cast<int32_t*>(buf2 + o_off);
  int32_t* dep_ids = reinterpret_cast<int32_t*>(buf2 + o_ids);
  int4* rec = reinterpret_cast<int4*>(buf2 + o_rec);
  uint8_t* d_bblob = buf2 + o_blob;
  DevBinding* db = reinterpret_cast<DevBinding*>(buf2 + o_bind);
  c->host_binding.g = g->dev;
  c->host_binding.v = v->dev;
  c->host_binding.c = DevCache{acc, dep_off, dep_ids, rec, nullptr, d_bblob, (int32_t)bblob.size()};
  std::vector<uint8_t> host(total, 0);
  std::memcpy(host.data() + o_off, off.data(), (size_t)(n + 1) * 4);
  std::memcpy(host.data() + o_blob, bblob.data(), bblob.size());
  std::memcpy(host.data() + o_bind, &c->host_binding, sizeof(DevBinding));
  // dep_off first (the compaction needs it), blob + binding after the records
  GM_CUDA_TRY(cudaMemcpyAsync(buf2, host.data(), o_ids, cudaMemcpyHostToDevice, s));
  GM_CUDA_TRY(cudaMemcpyAsync(buf2 + o_blob, host.data() + o_blob, o_ctx2 - o_blob, cudaMemcpyHostToDevice, s));
  if (n && (st = launch_dep_compact(reinterpret_cast<const uint32_t*>(dep_rows), W, n, dep_off, dep_ids, s)))
    return bail(st);
  // records gathered from the vocabulary's token records (their byte offsets
  // point into the vocabulary buffer), then the one-level context classes
  // GMASK_CTX_CLASSES=0 (diagnostics): no context classes, the fill walks
  // every dependent (with an uncached compile: every token, REF
  // matcher.py:446-460 brute force)
  const char* cc = getenv("GMASK_CTX_CLASSES");
  const bool ctx_classes = !(cc && cc[0] == '0');
  if ((st = launch_dep_records(dep_ids, dep_total, v->dev.tokrec, rec, s)) ||
      (ctx_classes &&
       (st = launch_dep_context(g->dev, dep_off, n, dep_total, rec, reinterpret_cast<const uint8_t*>(v->dev.tokrec),
                                s))) ||
      (two_level &&
       (st = launch_dep_context2(g->dev, dep_off, n, dep_total, rec, reinterpret_cast<const uint8_t*>(v->dev.tokrec),
                                 ctx2, s))))
    return bail(st);
  GM_CUDA_TRY(cudaStreamSynchronize(s));  // host buffer + every consumer on other streams
  c->binding = db;
  c->n_keys = n;
  if (stats) {
    int64_t n_univ = v->dev.n_sorted;
    stats->n_keys = n;
    stats->accepted_total = acc_total;
    stats->dependent_total = dep_total;
    stats->rejected_total = (int64_t)n * n_univ - acc_total - dep_total;
    stats->row_bytes = (int64_t)n * W * 4;
    stats->blend_keys = c->n_blend_keys;
  }
  *out = c;
  return GM_OK;
}

void gm_cache_release(gm_cache* c) {
  if (!c) return;
  {
    std::lock_guard<std::mutex> lk(g_pools_mu);
    for (gm_pool* p : g_pools) {
      if (!p->bound.erase(c)) continue;
      for (auto& sc : p->slot_cache)
        if (sc == c) sc = nullptr;
      refresh_hint(p);
    }
  }
  c->mem.release();
  delete c;
}
gm_status gm_cache_export(const gm_cache* c, int32_t* acc_rows_out, int32_t* dep_off_out, int32_t* dep_ids_out,
                          int64_t* n_dep_out) {
  if (!c) return fail(GM_ERR_INVALID, "null cache");
  const int32_t n = c->n_keys, W = c->host_binding.v.W;
  int32_t total = 0;
  GM_CUDA_TRY(cudaMemcpy(&total, c->host_binding.c.dep_off + n, 4, cudaMemcpyDeviceToHost));
  if (n_dep_out) *n_dep_out = total;
  if (acc_rows_out && n)
    GM_CUDA_TRY(cudaMemcpy(acc_rows_out, c->host_binding.c.acc_rows, (size_t)n * W * 4, cudaMemcpyDeviceToDevice));
  if (dep_off_out)
    GM_CUDA_TRY(cudaMemcpy(dep_off_out, c->host_binding.c.dep_off, (size_t)(n + 1) * 4, cudaMemcpyDeviceToDevice));
  if (dep_ids_out && total)
    GM_CUDA_TRY(cudaMemcpy(dep_ids_out, c->host_binding.c.dep_ids, (size_t)total * 4, cudaMemcpyDeviceToDevice));
  return GM_OK;
}

// ---------------------------------------------------------------------------
gm_status gm_pool_create(int32_t capacity, int32_t max_stacks, int32_t max_window, int64_t arena_log2,
                         gm_pool** out) {
  if (capacity <= 0 || max_stacks <= 0 || max_stacks > 32 || max_window < 0 || arena_log2 < 10 ||
      arena_log2 > 30 || !out)
    return fail(GM_ERR_INVALID, "bad pool arguments (max_stacks <= 32, 10 <= arena_log2 <= 30)");
  gm_pool* p = new gm_pool();
  const int32_t H = max_window + 1;
  const uint32_t acap = 1u << arena_log2;
  // wide top sets (> max_stacks stacks, up to kWideCap): blocks of kWideCap
  // stacks shared by the pool; overflow-walker lanes
  const int32_t n_wide = std::max(0, env_i32("GMASK_WIDE_BLOCKS", 64));
  const int32_t lanes = std::max(1, env_i32("GMASK_OVF_LANES", 32));
  gm_status st;
  int2 *tops, *wide_pool;
  int32_t *meta, *head, *hist, *win, *scr, *wide;
  const DevBinding** bind;
  unsigned long long* keys;
  uint32_t *err, *arena_err, *wide_bits;
  uint8_t* sb;
  SlotHdr* hdr;
  DevOverflow ovf;
  auto bail = [&](gm_status e) {
    p->mem.release();
    delete p;
    return e;
  };
  if ((st = p->mem.alloc(&hdr, (size_t)capacity)) || (st = p->mem.alloc(&tops, (size_t)capacity * H * max_stacks)) ||
      (st = p->mem.alloc(&meta, (size_t)capacity * H)) || (st = p->mem.alloc(&head, (size_t)capacity)) ||
      (st = p->mem.alloc(&hist, (size_t)capacity)) || (st = p->mem.alloc(&win, (size_t)capacity)) ||
      (st = p->mem.alloc(&bind, (size_t)capacity)) || (st = p->mem.alloc(&keys, (size_t)acap)) ||
      (st = p->mem.alloc(&err, (size_t)capacity)) || (st = p->mem.alloc(&arena_err, 1)) ||
      (st = p->mem.alloc(&sb, 1 << 16)) || (st = p->mem.alloc(&scr, 1024)) ||
      (st = p->mem.alloc(&wide_pool, (size_t)std::max(n_wide, 1) * kWideCap)) ||
      (st = p->mem.alloc(&wide, (size_t)capacity * H)) ||
      (st = p->mem.alloc(&wide_bits, (size_t)(n_wide + 31) / 32 + 1)) ||
      (st = alloc_overflow(lanes, &ovf, &p->mem.ptrs)))
    return bail(st);
  GM_CUDA_TRY(cudaMemset(keys, 0xFF, sizeof(unsigned long long) * acap));
  GM_CUDA_TRY(cudaMemset(err, 0, 4 * (size_t)capacity));
  GM_CUDA_TRY(cudaMemset(arena_err, 0, 4));
  GM_CUDA_TRY(cudaMemset(meta, 0, sizeof(int32_t) * (size_t)capacity * H));
  GM_CUDA_TRY(cudaMemset(wide, 0xFF, sizeof(int32_t) * (size_t)capacity * H));
  GM_CUDA_TRY(cudaMemset(wide_bits, 0, 4 * ((size_t)(n_wide + 31) / 32 + 1)));
  GM_CUDA_TRY(cudaMemset(head, 0, sizeof(int32_t) * (size_t)capacity));
  GM_CUDA_TRY(cudaMemset(hist, 0, sizeof(int32_t) * (size_t)capacity));
  GM_CUDA_TRY(cudaMemset(bind, 0, sizeof(void*) * (size_t)capacity));
  GM_CUDA_TRY(cudaMemset(hdr, 0, sizeof(SlotHdr) * (size_t)capacity));
  unsigned long long* trace = nullptr;
  const char* tr = getenv("GMASK_TRACE");
  const int32_t trace_ring = (tr && tr[0] == '2') ? 16 : 0;
  if (tr && (tr[0] == '1' || tr[0] == '2')) {
    const size_t n = 64 + 16 * (size_t)capacity * (1 + trace_ring) + (size_t)capacity;
    if ((st = p->mem.alloc(&trace, n))) return bail(st);
    GM_CUDA_TRY(cudaMemset(trace, 0, n * 8));
  }
  p->dev = DevPool{};
  p->dev.capacity = capacity;
  p->dev.max_stacks = max_stacks;
  p->dev.H = H;
  p->dev.tops = tops;
  p->dev.meta = meta;
  p->dev.head = head;
  p->dev.hist_len = hist;
  p->dev.window = win;
  p->dev.binding = bind;
  p->dev.arena = DevArena{keys, acap - 1, arena_err};
  p->dev.err = err;
  p->dev.wide_pool = wide_pool;
  p->dev.wide = wide;
  p->dev.wide_bits = wide_bits;
  p->dev.n_wide = n_wide;
  p->dev.ovf = ovf;
  p->dev.hdr = hdr;
  p->dev.trace = trace;
  p->dev.trace_ring = trace_ring;
  // opt-in L2 persistence for the arena (GMASK_L2_PERSIST=1): a device-wide
  // persisting carve-out + a persisting access-policy window on the step
  // launches; measured no gain on the JSON bench (the contended arena lines
  // are L2-resident anyway)
  const char* pe = getenv("GMASK_L2_PERSIST");
  if (pe && pe[0] == '1') {
    int dev = 0, max_persist = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
    const size_t abytes = sizeof(unsigned long long) * acap;
    if (max_persist > 0) {
      size_t cur = 0;
      cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
      const size_t want = std::min<size_t>((size_t)max_persist, std::max(cur, abytes));
      if (want > cur) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
      cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
      if (cur > 0) {
        p->dev.l2_base = keys;
        p->dev.l2_bytes = abytes;
        p->dev.l2_hit = abytes <= cur ? 1.0f : (float)cur / (float)abytes;
        launch_l2_touch(keys, abytes, L2Window{keys, abytes, p->dev.l2_hit});
      }
      cudaGetLastError();  // the limit is advisory: ignore a refusal
    }
  }
  {
    std::lock_guard<std::mutex> lk(g_pools_mu);
    g_pools.insert(p);
  }
  p->scratch_bytes = sb;
  p->scratch_cap = 1 << 16;
  p->scratch_i32 = scr;
  p->max_w = 0;
  *out = p;
  return GM_OK;
}

void gm_pool_release(gm_pool* p) {
  if (!p) return;
  {
    std::lock_guard<std::mutex> lk(g_pools_mu);
    g_pools.erase(p);
  }
  cudaDeviceSynchronize();
  p->mem.release();
  delete p;
}

// Host bookkeeping of slot bindings -> the pool's launch hint (DevPool
// hint_*): set while every bound slot shares one binding.
static void refresh_hint(gm_pool* p) {
  const gm_cache* h = p->bound.size() == 1 ? p->bound.begin()->first : nullptr;
  const bool fits = h && h->host_binding.c.blob_bytes <= kStageBytes;
  p->dev.hint_blob = fits ? h->host_binding.c.blob : nullptr;
  p->dev.hint_blob_bytes = fits ? h->host_binding.c.blob_bytes : 0;
  p->dev.hint_tokrec = fits ? h->host_binding.v.tokrec : nullptr;
  p->dev.hint_V = fits ? h->host_binding.v.V : 0;
}

static void bind_slot(gm_pool* p, int32_t slot, const gm_cache* c) {
  std::lock_guard<std::mutex> lk(g_pools_mu);
  if ((int32_t)p->slot_cache.size() < p->dev.capacity) p->slot_cache.resize(p->dev.capacity, nullptr);
  const gm_cache* old = p->slot_cache[slot];
  if (old && --p->bound[old] == 0) p->bound.erase(old);
  p->slot_cache[slot] = c;
  if (c) ++p->bound[c];
  refresh_hint(p);
}

gm_status gm_pool_reset(gm_pool* p, int32_t slot, const gm_grammar* g, const gm_cache* c, const gm_vocab* v,
                        int32_t window, void* stream) {
  if (!p || !g || !c || !v) return fail(GM_ERR_INVALID, "null argument");
  if (slot < 0 || slot >= p->dev.capacity) return fail(GM_ERR_INVALID, "slot out of range");
  if (window < 0 || window > p->dev.H - 1) return fail(GM_ERR_INVALID, "history window exceeds pool maximum");
  if (v->dev.W > p->max_w) p->max_w = v->dev.W;
  bind_slot(p, slot, c);
  return launch_reset(p->dev, slot, c->binding, g->dev.start_node, window, as_stream(stream));
}

gm_status gm_pool_fork(gm_pool* p, int32_t src, int32_t dst, void* stream) {
  if (!p || src < 0 || dst < 0 || src >= p->dev.capacity || dst >= p->dev.capacity)
    return fail(GM_ERR_INVALID, "slot out of range");
  bind_slot(p, dst, (int32_t)p->slot_cache.size() > src ? p->slot_cache[src] : nullptr);
  return launch_fork(p->dev, src, dst, as_stream(stream));
}

gm_status gm_accept_tokens(gm_pool* p, const int32_t* slots, const int32_t* token_ids, int32_t n,
                           uint8_t* accepted_out, void* stream) {
  if (!p) return fail(GM_ERR_INVALID, "null pool");
  return launch_accept_tokens(p->dev, slots, token_ids, n, accepted_out, as_stream(stream));
}

gm_status gm_accept_bytes(gm_pool* p, int32_t slot, const uint8_t* data, int64_t len, uint8_t* accepted_out,
                          void* stream) {
  if (!p || slot < 0 || slot >= p->dev.capacity) return fail(GM_ERR_INVALID, "slot out of range");
  cudaStream_t s = as_stream(stream);
  if (len > p->scratch_cap) {
    uint8_t* nb;
    GM_CUDA_TRY(cudaStreamSynchronize(s));
    GM_CUDA_TRY(cudaMalloc(&nb, (size_t)len));
    p->mem.ptrs.push_back(nb);
    p->scratch_bytes = nb;
    p->scratch_cap = len;
  }
  if (len) GM_CUDA_TRY(cudaMemcpyAsync(p->scratch_bytes, data, (size_t)len, cudaMemcpyHostToDevice, s));
  return launch_accept_bytes(p->dev, slot, p->scratch_bytes, len, accepted_out, s);
}

gm_status gm_fill_tokens(gm_pool* p, const int32_t* slots, int32_t n, int32_t* bitmask, int64_t bitmask_stride,
                         const int32_t* rows, uint8_t* need_apply_out, void* stream) {
  if (!p) return fail(GM_ERR_INVALID, "null pool");
  return launch_fill(p->dev, slots, n, bitmask, bitmask_stride, rows, need_apply_out, p->max_w,
                     as_stream(stream));
}

gm_status gm_fill_apply_tokens(gm_pool* p, const int32_t* slots, int32_t n, int32_t* bitmask, int64_t bitmask_stride,
                               const int32_t* rows, void* logits, int32_t dtype, int64_t vocab_size,
                               int64_t logits_stride, void* stream) {
  if (!p || !logits) return fail(GM_ERR_INVALID, "null pool/logits");
  int32_t eb;
  uint32_t neg;
  switch (dtype) {
    case GM_DTYPE_F32: eb = 4; neg = 0xFF800000u; break;
    case GM_DTYPE_F16: eb = 2; neg = 0xFC00FC00u; break;
    case GM_DTYPE_BF16: eb = 2; neg = 0xFF80FF80u; break;
    default: return fail(GM_ERR_INVALID, "unknown dtype");
  }
  if (reinterpret_cast<uintptr_t>(logits) % 16 || (logits_stride * eb) % 16)
    return fail(GM_ERR_INVALID, "fused fill+apply needs 16-byte aligned logits rows");
  return launch_fill_apply(p->dev, slots, n, bitmask, bitmask_stride, rows, p->max_w, logits, eb, neg, vocab_size,
                           logits_stride * eb, as_stream(stream));
}

gm_status gm_step_tokens(gm_pool* p, const int32_t* slots, int32_t n, const int32_t* token_ids, uint8_t* accepted_out,
                         int32_t recycle_terminated, int32_t* bitmask, int64_t bitmask_stride, const int32_t* rows,
                         void* logits, int32_t dtype, int64_t vocab_size, int64_t logits_stride, void* stream) {
  if (!p) return fail(GM_ERR_INVALID, "null pool");
  if (token_ids && !accepted_out) return fail(GM_ERR_INVALID, "accepted_out is required with token_ids");
  if (!bitmask && !logits) return fail(GM_ERR_INVALID, "need a bitmask and/or logits");
  int32_t eb = 2;
  uint32_t neg = 0;
  if (logits) {
    switch (dtype) {
      case GM_DTYPE_F32: eb = 4; neg = 0xFF800000u; break;
      case GM_DTYPE_F16: eb = 2; neg = 0xFC00FC00u; break;
      case GM_DTYPE_BF16: eb = 2; neg = 0xFF80FF80u; break;
      default: return fail(GM_ERR_INVALID, "unknown dtype");
    }
    if (reinterpret_cast<uintptr_t>(logits) % 16 || (logits_stride * eb) % 16)
      return fail(GM_ERR_INVALID, "fused step+apply needs 16-byte aligned logits rows");
  }
  return launch_step(p->dev, slots, n, token_ids, accepted_out, recycle_terminated, bitmask, bitmask_stride, rows,
                     p->max_w, logits, eb, neg, vocab_size, logits_stride * eb, as_stream(stream));
}

gm_status gm_step_tokens_host_slots(gm_pool* p, const int32_t* host_slots, int32_t n, const int32_t* token_ids,
                                    uint8_t* accepted_out, int32_t recycle_terminated, int32_t* bitmask,
                                    int64_t bitmask_stride, void* logits, int32_t dtype, int64_t vocab_size,
                                    int64_t logits_stride, void* stream) {
  if (!p || (n > 0 && !host_slots)) return fail(GM_ERR_INVALID, "null pool / slots");
  if (token_ids && !accepted_out) return fail(GM_ERR_INVALID, "accepted_out is required with token_ids");
  if (!bitmask && !logits) return fail(GM_ERR_INVALID, "need a bitmask and/or logits");
  for (int32_t i = 0; i < n; ++i)
    if (host_slots[i] < 0 || host_slots[i] >= p->dev.capacity) return fail(GM_ERR_INVALID, "slot out of range");
  int32_t eb = 2;
  uint32_t neg = 0;
  if (logits) {
    switch (dtype) {
      case GM_DTYPE_F32: eb = 4; neg = 0xFF800000u; break;
      case GM_DTYPE_F16: eb = 2; neg = 0xFC00FC00u; break;
      case GM_DTYPE_BF16: eb = 2; neg = 0xFF80FF80u; break;
      default: return fail(GM_ERR_INVALID, "unknown dtype");
    }
    if (reinterpret_cast<uintptr_t>(logits) % 16 || (logits_stride * eb) % 16)
      return fail(GM_ERR_INVALID, "fused step+apply needs 16-byte aligned logits rows");
  }
  return launch_step_ptok(p->dev, host_slots, n, nullptr, token_ids, accepted_out, recycle_terminated, bitmask,
                          bitmask_stride, p->max_w, logits, eb, neg, vocab_size, logits_stride * eb,
                          as_stream(stream));
}

// ---------------------------------------------------------------------------
// Native decode loop (gm_decoder_*): per step one host memcpy into pinned
// staging, H2D on an input copy stream, K5 on the caller's stream, D2H of
// the accepted flags on an output copy stream — all ordered by events (so
// step s+1's H2D overlaps step s's kernel), no host sync except the reuse
// guard of a step slot.
struct gm_decoder {
  gm_pool* pool = nullptr;
  const int32_t* slots = nullptr;
  int32_t n = 0, n_buf = 0, recycle = 1, dtype = GM_DTYPE_BF16;
  int64_t bstride = 0, vocab = 0, lstride = 0;
  std::vector<int32_t*> bitmask;
  std::vector<void*> logits;
  std::vector<int32_t*> tok_host, tok_dev;
  std::vector<uint8_t*> acc_host, acc_dev;
  std::vector<cudaEvent_t> h2d, k5, done;
  std::vector<int> issued;
  std::vector<int32_t> host_slots;  // the slot ids, passed by value to K5
  bool no_ptok = false;             // GMASK_DECODER_COPY=1: token ids via the H2D copy path
  cudaStream_t copy = nullptr;      // H2D of token ids
  cudaStream_t copy_out = nullptr;  // D2H of accepted flags (separate: the next H2D must not queue behind it)
};

static void decoder_free(gm_decoder* d) {
  if (!d) return;
  if (d->copy) cudaStreamSynchronize(d->copy);
  if (d->copy_out) cudaStreamSynchronize(d->copy_out);
  for (auto e : d->h2d) if (e) cudaEventDestroy(e);
  for (auto e : d->k5) if (e) cudaEventDestroy(e);
  for (auto e : d->done) if (e) cudaEventDestroy(e);
  for (auto q : d->tok_host) if (q) cudaFreeHost(q);
  for (auto q : d->acc_host) if (q) cudaFreeHost(q);
  for (auto q : d->tok_dev) if (q) cudaFree(q);
  for (auto q : d->acc_dev) if (q) cudaFree(q);
  if (d->copy) cudaStreamDestroy(d->copy);
  if (d->copy_out) cudaStreamDestroy(d->copy_out);
  delete d;
}

gm_status gm_decoder_create(gm_pool* p, const int32_t* slots, int32_t n, int32_t n_buf, int32_t* const* bitmasks,
                            int64_t bitmask_stride, void* const* logits, int32_t dtype, int64_t vocab_size,
                            int64_t logits_stride, int32_t recycle, gm_decoder** out) {
  if (!p || !slots || n <= 0 || n_buf <= 0 || !out || !logits) return fail(GM_ERR_INVALID, "bad decoder arguments");
  auto* d = new gm_decoder();
  d->pool = p;
  d->slots = slots;
  d->n = n;
  d->n_buf = n_buf;
  d->recycle = recycle;
  d->dtype = dtype;
  d->bstride = bitmask_stride;
  d->vocab = vocab_size;
  d->lstride = logits_stride;
  d->issued.assign(n_buf, 0);
  {
    const char* e = getenv("GMASK_DECODER_COPY");
    d->no_ptok = e && e[0] == '1';
  }
  auto bail = [&](cudaError_t e) {
    decoder_free(d);
    return fail(GM_ERR_CUDA, std::string("gm_decoder_create: ") + cudaGetErrorString(e));
  };
  d->host_slots.resize(n);
  {
    const cudaError_t e0 = cudaMemcpy(d->host_slots.data(), slots, (size_t)n * 4, cudaMemcpyDeviceToHost);
    if (e0 != cudaSuccess) return bail(e0);
  }
  cudaError_t e = cudaStreamCreateWithFlags(&d->copy, cudaStreamNonBlocking);
  if (e != cudaSuccess) return bail(e);
  if ((e = cudaStreamCreateWithFlags(&d->copy_out, cudaStreamNonBlocking)) != cudaSuccess) return bail(e);
  for (int32_t b = 0; b < n_buf; ++b) {
    d->bitmask.push_back(bitmasks ? bitmasks[b] : nullptr);
    d->logits.push_back(logits[b]);
    int32_t *th = nullptr, *td = nullptr;
    uint8_t *ah = nullptr, *ad = nullptr;
    cudaEvent_t e1 = nullptr, e2 = nullptr, e3 = nullptr;
    if ((e = cudaHostAlloc(&th, (size_t)n * 4, cudaHostAllocDefault)) != cudaSuccess) return bail(e);
    d->tok_host.push_back(th);
    if ((e = cudaHostAlloc(&ah, (size_t)n, cudaHostAllocDefault)) != cudaSuccess) return bail(e);
    d->acc_host.push_back(ah);
    if ((e = cudaMalloc(&td, (size_t)n * 4)) != cudaSuccess) return bail(e);
    d->tok_dev.push_back(td);
    if ((e = cudaMalloc(&ad, (size_t)n)) != cudaSuccess) return bail(e);
    d->acc_dev.push_back(ad);
    if ((e = cudaEventCreateWithFlags(&e1, cudaEventDisableTiming)) != cudaSuccess) return bail(e);
    d->h2d.push_back(e1);
    if ((e = cudaEventCreateWithFlags(&e2, cudaEventDisableTiming)) != cudaSuccess) return bail(e);
    d->k5.push_back(e2);
    if ((e = cudaEventCreateWithFlags(&e3, cudaEventDisableTiming)) != cudaSuccess) return bail(e);
    d->done.push_back(e3);
    std::memset(ah, 0, (size_t)n);
  }
  *out = d;
  return GM_OK;
}

gm_status gm_decoder_step(gm_decoder* d, int32_t buf, const int32_t* host_tokens, void* stream) {
  if (!d || buf < 0 || buf >= d->n_buf) return fail(GM_ERR_INVALID, "bad decoder slot");
  cudaStream_t s = as_stream(stream);
  if (d->issued[buf]) GM_CUDA_TRY(cudaEventSynchronize(d->done[buf]));  // staging reuse guard
  const int32_t n = d->n;
  if (host_tokens && n <= 512 && !d->no_ptok) {
    // token ids by value in the K5 launch parameters: no staging, no H2D copy
    int32_t eb = 2;
    uint32_t neg = 0;
    switch (d->dtype) {
      case GM_DTYPE_F32: eb = 4; neg = 0xFF800000u; break;
      case GM_DTYPE_F16: eb = 2; neg = 0xFC00FC00u; break;
      default: eb = 2; neg = 0xFF80FF80u; break;
    }
    gm_status st = launch_step_ptok(d->pool->dev, d->host_slots.data(), n, host_tokens, nullptr, d->acc_dev[buf],
                                    d->recycle, d->bitmask[buf], d->bstride, d->pool->max_w, d->logits[buf], eb, neg,
                                    d->vocab, d->lstride * eb, s);
    if (st) return st;
    GM_CUDA_TRY(cudaEventRecord(d->k5[buf], s));
    GM_CUDA_TRY(cudaStreamWaitEvent(d->copy_out, d->k5[buf], 0));
    GM_CUDA_TRY(cudaMemcpyAsync(d->acc_host[buf], d->acc_dev[buf], (size_t)n, cudaMemcpyDeviceToHost, d->copy_out));
    GM_CUDA_TRY(cudaEventRecord(d->done[buf], d->copy_out));
    d->issued[buf] = 1;
    return GM_OK;
  }
  if (host_tokens) {
    std::memcpy(d->tok_host[buf], host_tokens, (size_t)n * 4);
    GM_CUDA_TRY(cudaMemcpyAsync(d->tok_dev[buf], d->tok_host[buf], (size_t)n * 4, cudaMemcpyHostToDevice, d->copy));
    GM_CUDA_TRY(cudaEventRecord(d->h2d[buf], d->copy));
    GM_CUDA_TRY(cudaStreamWaitEvent(s, d->h2d[buf], 0));
  }
  gm_status st = gm_step_tokens(d->pool, d->slots, n, host_tokens ? d->tok_dev[buf] : nullptr,
                                host_tokens ? d->acc_dev[buf] : nullptr, d->recycle, d->bitmask[buf], d->bstride,
                                nullptr, d->logits[buf], d->dtype, d->vocab, d->lstride, stream);
  if (st) return st;
  GM_CUDA_TRY(cudaEventRecord(d->k5[buf], s));
  GM_CUDA_TRY(cudaStreamWaitEvent(d->copy_out, d->k5[buf], 0));
  if (host_tokens)
    GM_CUDA_TRY(cudaMemcpyAsync(d->acc_host[buf], d->acc_dev[buf], (size_t)n, cudaMemcpyDeviceToHost, d->copy_out));
  else
    std::memset(d->acc_host[buf], 0, (size_t)n);
  GM_CUDA_TRY(cudaEventRecord(d->done[buf], d->copy_out));
  d->issued[buf] = 1;
  return GM_OK;
}

gm_status gm_decoder_flags(gm_decoder* d, int32_t buf, uint8_t* out, int32_t wait) {
  if (!d || buf < 0 || buf >= d->n_buf || !out) return fail(GM_ERR_INVALID, "bad decoder slot");
  if (d->issued[buf]) {
    if (wait) {
      GM_CUDA_TRY(cudaEventSynchronize(d->done[buf]));
    } else {
      const cudaError_t q = cudaEventQuery(d->done[buf]);
      if (q == cudaErrorNotReady) return fail(GM_ERR_INVALID, "decoder step not complete");
      GM_CUDA_TRY(q);
    }
  }
  std::memcpy(out, d->acc_host[buf], (size_t)d->n);
  return GM_OK;
}

void gm_decoder_release(gm_decoder* d) { decoder_free(d); }

gm_status gm_rollback(gm_pool* p, const int32_t* slots, const int32_t* steps, int32_t n, void* stream) {
  if (!p) return fail(GM_ERR_INVALID, "null pool");
  return launch_rollback(p->dev, slots, steps, n, as_stream(stream));
}

gm_status gm_pool_recycle(gm_pool* p, const int32_t* slots, int32_t n, void* stream) {
  if (!p) return fail(GM_ERR_INVALID, "null pool");
  return launch_recycle(p->dev, slots, n, as_stream(stream));
}

gm_status gm_pool_check(gm_pool* p, int32_t* flags_out) {
  if (!p) return fail(GM_ERR_INVALID, "null pool");
  GM_CUDA_TRY(cudaDeviceSynchronize());
  std::vector<uint32_t> words((size_t)p->dev.capacity);
  GM_CUDA_TRY(cudaMemcpy(words.data(), p->dev.err, words.size() * 4, cudaMemcpyDeviceToHost));
  GM_CUDA_TRY(cudaMemset(p->dev.err, 0, words.size() * 4));
  uint32_t bits = 0;
  for (uint32_t w : words) bits |= w;
  if (flags_out) *flags_out = (int32_t)bits;
  return err_bits_to_status(bits, "matcher");
}

gm_status gm_pool_errors(gm_pool* p, const int32_t* slots, int32_t n, uint32_t* out, int32_t clear, void* stream) {
  if (!p) return fail(GM_ERR_INVALID, "null pool");
  return launch_pool_errors(p->dev, slots, n, out, clear, as_stream(stream));
}

gm_status gm_status_of_error_bits(uint32_t bits) { return err_bits_to_status(bits, "matcher"); }

gm_status gm_pool_slot_info(gm_pool* p, int32_t slot, int32_t* info5, int32_t* stacks_out, int32_t max_out) {
  if (!p || slot < 0 || slot >= p->dev.capacity) return fail(GM_ERR_INVALID, "slot out of range");
  if (max_out > 32) max_out = 32;
  int32_t* d = p->scratch_i32;  // [0..8) info, [16..24) bytes, [64..) stacks
  gm_status st = launch_probe(p->dev, slot, d, reinterpret_cast<int2*>(d + 64), max_out,
                              reinterpret_cast<uint32_t*>(d + 16), 0);
  if (st) return st;
  int32_t host[128];
  GM_CUDA_TRY(cudaMemcpy(host, d, sizeof(host), cudaMemcpyDeviceToHost));
  std::memcpy(info5, host, 5 * 4);
  if (stacks_out && max_out > 0) std::memcpy(stacks_out, host + 64, (size_t)std::min(max_out, host[0]) * 8);
  return GM_OK;
}

gm_status gm_pool_first_bytes(gm_pool* p, int32_t slot, uint32_t* bytes8, int32_t* terminable) {
  if (!p || slot < 0 || slot >= p->dev.capacity) return fail(GM_ERR_INVALID, "slot out of range");
  int32_t* d = p->scratch_i32;
  gm_status st = launch_probe(p->dev, slot, d, reinterpret_cast<int2*>(d + 64), 0,
                              reinterpret_cast<uint32_t*>(d + 16), 0);
  if (st) return st;
  int32_t host[32];
  GM_CUDA_TRY(cudaMemcpy(host, d, sizeof(host), cudaMemcpyDeviceToHost));
  std::memcpy(bytes8, host + 16, 32);
  if (terminable) *terminable = host[3];
  return GM_OK;
}

gm_status gm_pool_materialize(gm_pool* p, int32_t handle, int32_t* out, int32_t max_out, int32_t* depth) {
  if (!p) return fail(GM_ERR_INVALID, "null pool");
  std::vector<int32_t> chain;
  int32_t h = handle;
  while (h >= 0) {
    unsigned long long k;
    GM_CUDA_TRY(cudaMemcpy(&k, p->dev.arena.keys + h, 8, cudaMemcpyDeviceToHost));
    chain.push_back((int32_t)((uint32_t)k >> 1));
    h = (int32_t)(uint32_t)(k >> 32) - 1;
    if ((int64_t)chain.size() > (int64_t)p->dev.arena.mask + 1) return fail(GM_ERR_INVALID, "corrupt chain");
  }
  std::reverse(chain.begin(), chain.end());
  *depth = (int32_t)chain.size();
  for (int32_t i = 0; i < (int32_t)chain.size() && i < max_out; ++i) out[i] = chain[i];
  return GM_OK;
}

gm_status gm_pool_trace(gm_pool* p, uint64_t* out, int64_t n) {
  if (!p || !p->dev.trace) return fail(GM_ERR_INVALID, "pool created without GMASK_TRACE=1");
  const int64_t cap = 64 + 16 * (int64_t)p->dev.capacity * (1 + p->dev.trace_ring) + (int64_t)p->dev.capacity;
  if (n > cap) n = cap;
  GM_CUDA_TRY(cudaDeviceSynchronize());
  GM_CUDA_TRY(cudaMemcpy(out, p->dev.trace, n * 8, cudaMemcpyDeviceToHost));
  return GM_OK;
}

gm_status gm_pool_arena_stats(gm_pool* p, int64_t* live, int64_t* tombstones, int64_t* capacity) {
  if (!p) return fail(GM_ERR_INVALID, "null pool");
  gm_status st;
  if (!p->counts && (st = p->mem.alloc(&p->counts, 2))) return st;
  if ((st = launch_arena_count(p->dev.arena, p->counts, 0))) return st;
  unsigned long long c[2];
  GM_CUDA_TRY(cudaMemcpy(c, p->counts, 16, cudaMemcpyDeviceToHost));
  if (live) *live = (int64_t)c[0];
  if (tombstones) *tombstones = (int64_t)c[1];
  if (capacity) *capacity = (int64_t)p->dev.arena.mask + 1;
  return GM_OK;
}

int64_t gm_pool_arena_used(gm_pool* p) {
  int64_t live = -1;
  if (gm_pool_arena_stats(p, &live, nullptr, nullptr)) return -1;
  return live;
}

gm_status gm_pool_collect(gm_pool* p, const int32_t* live_slots, int32_t n, void* stream) {
  if (!p || n < 0 || (n > 0 && !live_slots)) return fail(GM_ERR_INVALID, "bad collect arguments");
  for (int32_t i = 0; i < n; ++i)
    if (live_slots[i] < 0 || live_slots[i] >= p->dev.capacity) return fail(GM_ERR_INVALID, "slot out of range");
  gm_status st;
  const size_t words = ((size_t)p->dev.arena.mask + 1) / 32;
  if (!p->gc_mark && ((st = p->mem.alloc(&p->gc_mark, words)) || (st = p->mem.alloc(&p->gc_need, words)))) return st;
  cudaStream_t s = as_stream(stream);
  int32_t* d_live = nullptr;
  if (n > 0) {
    GM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d_live), (size_t)n * 4, s));
    GM_CUDA_TRY(cudaMemcpyAsync(d_live, live_slots, (size_t)n * 4, cudaMemcpyHostToDevice, s));
  }
  st = launch_collect(p->dev, d_live, n, p->gc_mark, p->gc_need, s);
  if (d_live) cudaFreeAsync(d_live, s);
  return st;
}

}  // extern "C"
