// Device-side data model shared by the cache builder (K1), fill (K2) and
// accept (K4) kernels: grammar tables, vocabulary, the hash-consed stack
// arena, the slot header and the byte-level stack-set walker.
//
// Stack model (restates the reference's matching stacks, REF pda.py:539-545,
// pstack.py:1-16): a stack is (chain, node) where `node` is the resting
// automaton node and `chain` is the stack of pending return nodes.  Chains are
// referenced by an int32 "ref":
//     ref == -1            empty chain (REF pstack.py EMPTY)
//     ref >=  0            walker-local frame (fast, per-thread)
//     ref <= -2            arena handle h = -2 - ref (global, hash-consed)
// The reference's closure over eps / rule push / final pop (REF matcher.py:
// 162-190, cache.py:110-143) is pre-closed on the host into per-(node, byte
// class) transitions, so one byte step here is:
//     for each stack (r, m): take every transition (push run P, target d) of
//     (m, class(b)); if m can silently complete its rule (GM_NODE_POP), pop
//     one frame and repeat from the caller's return node.
// Spent finals (dead ends) are popped through after the step (REF matcher.py
// 192-206) so resting nodes are always cache keys.
//
// Latency design: between decode steps the model's forward pass evicts L2, so
// the per-step kernels are bounded by dependent HBM round trips, not bytes.
// Everything a step needs is therefore reachable in few hops: a 256-byte slot
// header (pointers + current tops + cache keys + dependent ranges + EOS fact),
// one "binding blob" per (grammar, vocabulary) holding the walker tables and
// per-node cache info (staged into shared memory with one coalesced copy), and
// 32-byte token records with the token bytes inline.
#pragma once
#include <stdint.h>

#include "common.cuh"

namespace gm {

// sticky device error bits (pool / build scratch word)
enum : uint32_t {
  kErrCap = 1u << GM_ERR_STATE_CAP,
  kErrArena = 1u << GM_ERR_ARENA_FULL,
  kErrTerminated = 1u << GM_ERR_TERMINATED,
  kErrInvalid = 1u << GM_ERR_INVALID,
};

// ---------------------------------------------------------------------------
// Table blob: [BlobHdr | byte_class[256] | node_flags[n] | trans_off[n*C+1] |
// trans int2[] | push_pool[] | key_of_node[n] | node_rule[n] | node_info int4[n]]
// all sections 16-byte aligned; offsets in bytes from the blob start.
// node_info[n] = (cache key, first dependent, end dependent, rule) and is only
// present in binding blobs (grammar blobs have o_ninfo = 0).
constexpr int32_t kFastPopDies = INT32_MIN;

struct BlobHdr {
  int32_t bytes, n_classes, n_nodes, o_bc;
  int32_t o_flags, o_toff, o_trans, o_pool;
  int32_t o_kon, o_rule, o_ninfo, o_fast, o_callers, start_node;
  uint32_t ctx2_lo, ctx2_hi;  // binding blobs: device address of the two-level context classes (or 0)
};
static_assert(sizeof(BlobHdr) == 64, "BlobHdr layout");

struct DevGrammar {
  int32_t n_nodes, n_rules, n_classes, start_node, n_keys, n_fstates;
  const uint8_t* byte_class;   // [256]
  const int32_t* trans_off;    // [n_nodes*n_classes+1]
  const int2* trans;           // (target, push_off | push_len << 24)
  const int32_t* push_pool;
  const uint8_t* node_flags;
  const int32_t* node_rule;
  const int32_t* cache_keys;   // [n_keys]
  const int32_t* key_of_node;  // [n_nodes] -> key index or -1
  const int32_t* follow_start; // [n_rules]
  const int32_t* follow_next;  // [n_fstates*n_classes]
  const int4* node_info;       // binding views only
  const int32_t* fast;         // [n_nodes*n_classes] single-stack DFA move, -1 dies, -2 general;
                               // above the bottom frame also -3 - target / kFastPopDies (gm_grammar_create)
  const int32_t* callers;      // [n_rules*kMaxCallers] return nodes that can sit below a frame of the rule, -1 pad
  const uint32_t* ctx2;        // binding views: [n_dep*kMaxCallers] two-level context classes, or null
  const uint8_t* blob;
  int32_t blob_bytes;
};

// Walker view of a blob located at `base` (global or shared memory).
__device__ __forceinline__ DevGrammar blob_view(const uint8_t* base) {
  const BlobHdr* h = reinterpret_cast<const BlobHdr*>(base);
  DevGrammar g{};
  g.n_classes = h->n_classes;
  g.n_nodes = h->n_nodes;
  g.start_node = h->start_node;
  g.byte_class = base + h->o_bc;
  g.node_flags = base + h->o_flags;
  g.trans_off = reinterpret_cast<const int32_t*>(base + h->o_toff);
  g.trans = reinterpret_cast<const int2*>(base + h->o_trans);
  g.push_pool = reinterpret_cast<const int32_t*>(base + h->o_pool);
  g.key_of_node = reinterpret_cast<const int32_t*>(base + h->o_kon);
  g.node_rule = reinterpret_cast<const int32_t*>(base + h->o_rule);
  g.node_info = h->o_ninfo ? reinterpret_cast<const int4*>(base + h->o_ninfo) : nullptr;
  g.fast = reinterpret_cast<const int32_t*>(base + h->o_fast);
  g.callers = reinterpret_cast<const int32_t*>(base + h->o_callers);
  g.ctx2 = reinterpret_cast<const uint32_t*>(((unsigned long long)h->ctx2_hi << 32) | h->ctx2_lo);
  g.blob = base;
  g.blob_bytes = h->bytes;
  return g;
}

constexpr int kStageBytes = 32 * 1024;
// One-level context classes of a dependent token, packed 2 bits per caller
// (caller j of the key's rule) into the dependent record's 4th word.
// Index kRootCaller is the bottom of the stack (a top on the root frame).
constexpr int kMaxCallers = 16;
constexpr int kRootCaller = kMaxCallers - 1;
constexpr uint32_t kCtxUnknown = 0, kCtxAccept = 1, kCtxReject = 2, kCtxDeeper = 3;  // shared-memory budget for staged tables

// Stage a blob (`bytes` long, 16-byte multiple) into shared memory with one
// TMA bulk copy (cp.async.bulk, completion tracked by an mbarrier): a single
// HBM round trip however large the blob, instead of a loop of per-thread
// loads.  Returns a view of the shared copy — or of the global blob when it
// does not fit.  Must be called by every thread of the CTA (barrier inside).
// TMA bulk-copy helpers (cp.async.bulk global -> shared, mbarrier-tracked).
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* mbar, uint32_t tx_bytes) {
  const uint32_t m = smem_u32(mbar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(m));
  // CTA-local barrier used by this thread's own TMA copies: a proxy fence
  // suffices (a cluster-scope release fence would also wait for every prior
  // global store of the thread — e.g. the accept's state writes in K5)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(m), "r"(tx_bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(mbar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* mbar, uint32_t parity) {
  const uint32_t m = smem_u32(mbar);
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(m), "r"(parity) : "memory");
  }
}

__device__ __forceinline__ DevGrammar stage_blob(const uint8_t* blob, int32_t bytes, uint8_t* smem) {
  __shared__ __align__(8) unsigned long long mbar;
  const bool fits = bytes <= kStageBytes;
  if (fits && threadIdx.x == 0) {
    mbar_init(&mbar, (uint32_t)bytes);
    bulk_g2s(smem, blob, (uint32_t)bytes, &mbar);
  }
  __syncthreads();
  if (fits) mbar_wait(&mbar, 0);
  return blob_view(fits ? smem : blob);
}

struct DevVocab {
  int32_t V, W, n_sorted, eos;
  const uint8_t* bytes;
  const int32_t* off;          // [V+1]
  const int32_t* sorted_ids;   // non-special non-empty ids, lexicographic
  const uint32_t* universe;    // [W]
  const uint8_t* reject;       // [V] 1 = special or empty (never accepted)
  const int4* tokrec;          // [2V]: (reject, len, byte offset, 0), 16 inline bytes
};

// 32-byte token record: first int4 (id or flags, len, offset, 0), second int4
// the first 16 bytes inline.  Used for vocabulary tokens (accept) and
// dependent entries (fill).
constexpr int kInlineBytes = 16;
__device__ __forceinline__ uint8_t rec_byte(const int4& inl, const uint8_t* far, int i) {
  if (i < kInlineBytes) {
    const int w = (i < 4) ? inl.x : (i < 8) ? inl.y : (i < 12) ? inl.z : inl.w;
    return (uint8_t)((uint32_t)w >> ((i & 3) * 8));
  }
  return __ldg(far + i);
}

struct DevCache {
  const uint32_t* acc_rows;    // [n_keys*W]
  const int32_t* dep_off;      // [n_keys+1]
  const int32_t* dep_ids;
  const int4* dep_ent;         // [2*n_dep] records (tid, len, byte offset into the vocabulary's
                               // token-record buffer, context classes) + 16 inline bytes
  const uint8_t* dep_bytes;    // unused (null)
  const uint8_t* blob;         // binding blob (tables + node_info)
  int32_t blob_bytes;
};

// Everything a matcher slot needs, resident in device memory.
struct DevBinding {
  DevGrammar g;
  DevVocab v;
  DevCache c;
};

// ---------------------------------------------------------------------------
// Hash-consed frame arena: slot i of an open-addressing table holds the key
// (parent+1)<<32 | node<<1 | term; the handle of a frame IS its slot, so equal
// (parent, node) => equal handle (REF pstack.py:41-52 interning mode, made
// lock-free).  term = "every frame of the chain can silently complete", the
// running AND used for the O(1) EOS test.

constexpr unsigned long long kEmptyKey = ~0ull;

struct DevArena {
  unsigned long long* keys;
  uint32_t mask;
  uint32_t* err;
};

__device__ __forceinline__ unsigned long long arena_key(int32_t parent, int32_t node, uint32_t term) {
  return ((unsigned long long)(uint32_t)(parent + 1) << 32) | ((unsigned long long)(uint32_t)node << 1) | term;
}
__device__ __forceinline__ uint32_t mix64(unsigned long long k) {
  k ^= k >> 33; k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return (uint32_t)k;
}
// GPU-scope relaxed load (L2): an arena slot only ever changes from empty to
// its key, so no system-scope ordering is needed — a volatile (.sys) load of
// a hot slot (frames are hash-consed: every request shares its stack prefix,
// so 100+ CTAs read the same few slots each step) measured 1.5-3.5 us.
__device__ __forceinline__ unsigned long long arena_load(const DevArena& A, int32_t h) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(A.keys + h) : "memory");
  return v;
}
__device__ __forceinline__ int32_t key_parent(unsigned long long k) { return (int32_t)(uint32_t)(k >> 32) - 1; }
__device__ __forceinline__ int32_t key_node(unsigned long long k) { return (int32_t)((uint32_t)k >> 1); }
__device__ __forceinline__ uint32_t key_term(unsigned long long k) { return (uint32_t)k & 1u; }

// Tombstone: a slot whose frame was reclaimed by the pool's collector
// (gm_pool_collect) while a live key further along the same probe chain
// still needs the chain unbroken.  Never a valid key (parent+1 < 2^31).
constexpr unsigned long long kTombKey = ~1ull;

// Handle of `key`, inserting it if absent, probing linearly from `start`;
// -1 + error bit when the table is full.  Keys are only ever inserted at
// the first empty-or-tombstone slot of their probe chain, and the collector
// keeps every slot between a live key's home and its position non-empty, so
// reaching an EMPTY slot proves the key absent.  A tombstone is reused only
// after the scan has proved the key absent; a lost race rescans (slots only
// fill while kernels run, so two racing inserts of one key claim the same
// first free slot).
__device__ inline int32_t arena_probe(const DevArena& A, unsigned long long key, uint32_t start) {
  for (int attempt = 0; attempt < 64; ++attempt) {
    uint32_t i = start & A.mask;
    int64_t tomb = -1;
    int probe = 0;
    for (; probe < 8192; ++probe) {
      const unsigned long long cur = arena_load(A, (int32_t)i);
      if (cur == key) return (int32_t)i;
      if (cur == kEmptyKey) break;
      if (cur == kTombKey && tomb < 0) tomb = i;
      i = (i + 1) & A.mask;
    }
    if (probe == 8192 && tomb < 0) break;  // full
    const uint32_t at = tomb >= 0 ? (uint32_t)tomb : i;
    const unsigned long long expect = tomb >= 0 ? kTombKey : kEmptyKey;
    const unsigned long long old = atomicCAS(A.keys + at, expect, key);
    if (old == expect || old == key) return (int32_t)at;
  }
  if (A.err) atomicOr(A.err, kErrArena);
  return -1;
}
__device__ inline int32_t arena_intern(const DevArena& A, int32_t parent, int32_t node, uint32_t term) {
  const unsigned long long key = arena_key(parent, node, term);
  return arena_probe(A, key, mix64(key));
}

// ---------------------------------------------------------------------------
// Walker: a set of at most S stacks plus a pool of F walker-local frames and a
// small cache of arena keys already known to the caller (slot header), so the
// first pop below a top costs no HBM round trip.

constexpr int kChain = 16;  // ancestor frames cached in the slot header

template <int S, int F, int K = 24>
struct Walker {
  int32_t ref[S];
  int32_t node[S];
  int n;
  int32_t fpar[F];
  int32_t fnode[F];
  uint8_t fterm[F];
  int nf;
  uint32_t err;
  // arena keys this walk already knows: its own cache (frames it loaded or
  // interned) plus an optional read-only external one (the slot header's
  // ancestor chain in shared memory)
  int32_t kh[K];
  unsigned long long kk[K];
  int nk;
  const int32_t* xh;
  const unsigned long long* xk;
  int nx;

  __device__ __forceinline__ void reset() { n = 0; nf = 0; err = 0; nk = 0; nx = 0; }

  __device__ __forceinline__ void external(const int32_t* h, const unsigned long long* k, int cnt) {
    xh = h; xk = k; nx = cnt;
  }

  __device__ __forceinline__ bool lookup(int32_t h, unsigned long long& key) const {
    for (int i = 0; i < nk; ++i)
      if (kh[i] == h) { key = kk[i]; return true; }
    for (int i = 0; i < nx; ++i)
      if (xh[i] == h) { key = xk[i]; return true; }
    return false;
  }

  __device__ __forceinline__ void know(int32_t h, unsigned long long key) {
    if (h < 0 || key >= kTombKey || nk == K) return;
    for (int i = 0; i < nk; ++i)
      if (kh[i] == h) return;
    kh[nk] = h; kk[nk] = key; ++nk;
  }

  __device__ __forceinline__ unsigned long long key_of(const DevArena& A, int32_t h) {
    unsigned long long k;
    if (lookup(h, k)) {
#ifdef GM_VERIFY_KNOWN
      if (arena_load(A, h) != k) err |= 1u << 30;
#endif
      return k;
    }
    k = arena_load(A, h);
    if (k >= kTombKey) err |= kErrInvalid;  // dangling handle: report, never walk garbage
    else know(h, k);
    return k;
  }

  __device__ __forceinline__ bool add(int32_t r, int32_t d) {
    for (int q = 0; q < n; ++q)
      if (ref[q] == r && node[q] == d) return true;
    if (n == S) { err |= kErrCap; return false; }
    ref[n] = r; node[n] = d; ++n;
    return true;
  }

  __device__ __forceinline__ uint32_t term_of(const DevArena& A, int32_t r) {
    if (r == -1) return 1u;
    if (r >= 0) return fterm[r];
    return key_term(key_of(A, -2 - r));
  }

  __device__ __forceinline__ void pop(const DevArena& A, int32_t r, int32_t& pr, int32_t& pn) {
    if (r >= 0) { pr = fpar[r]; pn = fnode[r]; return; }
    const unsigned long long k = key_of(A, -2 - r);
    if (k >= kTombKey) { pr = -1; pn = 0; return; }  // reported by key_of
    const int32_t p = key_parent(k);
    pr = p < 0 ? -1 : -2 - p;
    pn = key_node(k);
  }

  __device__ __forceinline__ int32_t push(const DevGrammar& G, const DevArena& A, int32_t r, int32_t ret) {
    for (int q = nf - 1; q >= 0; --q)
      if (fpar[q] == r && fnode[q] == ret) return q;
    if (nf == F) { err |= kErrCap; return r; }
    fpar[nf] = r; fnode[nf] = ret;
    fterm[nf] = (uint8_t)(((G.node_flags[ret] & GM_NODE_POP) ? 1u : 0u) & term_of(A, r));
    return nf++;
  }

  // Can stack (r, m) silently reach an empty chain at a root final?
  // (REF matcher.py:219-237 _closed_facts.term)
  __device__ __forceinline__ bool terminable(const DevGrammar& G, const DevArena& A, int32_t r, int32_t m) {
    return (G.node_flags[m] & GM_NODE_POP) && term_of(A, r);
  }

  // One byte step of the whole set.  Sets *pop_bottom when some stack would
  // pop past an empty chain (REF cache.py:128-131 "popped" in synthetic
  // mode; at a real root this is the completed root and simply dies).
  // Table reads are plain (generic) loads: the tables may live in shared
  // memory.
  template <int SN>
  __device__ int step(const DevGrammar& G, const DevArena& A, uint32_t b, bool* pop_bottom) {
    const int c = G.byte_class[b];
    if (n == 1) {  // single stack: plain DFA moves need one table read
      const int32_t f = G.fast[node[0] * G.n_classes + c];
      if (f >= 0) { node[0] = f; return 1; }
      if (f == -1) { n = 0; return 0; }
    }
    int32_t nr[SN], nn[SN];
    int cnt = 0;
    for (int s = 0; s < n; ++s) {
      int32_t r = ref[s], m = node[s];
      while (true) {
        const int32_t idx = m * G.n_classes + c;
        const int32_t t0 = G.trans_off[idx], t1 = G.trans_off[idx + 1];
        for (int32_t t = t0; t < t1; ++t) {
          const int2 tr = G.trans[t];
          int32_t d = tr.x;
          const int plen = (int)((uint32_t)tr.y >> 24);
          const int poff = tr.y & 0xFFFFFF;
          int32_t rr = r;
          for (int k = 0; k < plen; ++k) rr = push(G, A, rr, G.push_pool[poff + k]);
          if (plen == 0) {
            while ((G.node_flags[d] & GM_NODE_DEAD_END) && rr != -1) {
              int32_t pr, pn;
              pop(A, rr, pr, pn);
              rr = pr; d = pn;
              if ((uint32_t)d >= (uint32_t)G.n_nodes) { err |= 1u << 29; d = 0; rr = -1; }
            }
          }
          bool dup = false;
          for (int q = 0; q < cnt; ++q)
            if (nr[q] == rr && nn[q] == d) { dup = true; break; }
          if (!dup) {
            if (cnt == SN) err |= kErrCap;
            else { nr[cnt] = rr; nn[cnt] = d; ++cnt; }
          }
        }
        if (!(G.node_flags[m] & GM_NODE_POP)) break;
        if (r == -1) { *pop_bottom = true; break; }
        pop(A, r, r, m);
        if ((uint32_t)m >= (uint32_t)G.n_nodes) { err |= 1u << 28; break; }
      }
    }
    for (int q = 0; q < cnt; ++q) { ref[q] = nr[q]; node[q] = nn[q]; }
    n = cnt;
    return cnt;
  }

  // Move every live stack's local frames into the arena and re-dedupe;
  // afterwards all refs are -1 or arena refs.  Speculative parallel
  // interning: each frame's handle is first assumed to be its key's home slot
  // (which also fixes its children's keys), so all CASes are independent and
  // in flight together (one HBM round trip instead of one per frame); a frame
  // whose home slot holds another key — and every frame after it — is redone
  // with sequential probing.  Entries written under a wrong speculative
  // parent are still valid frames (content-addressed), just unreferenced.
  // The arena keys of the live tops are remembered (know()).  Returns false
  // on arena exhaustion.
  __device__ bool intern_all(const DevArena& A) {
    if (nf == 0) return true;
    int32_t gmap[F];
    for (int q = 0; q < nf; ++q) gmap[q] = 0;  // 0 = unneeded, 1 = needed
    for (int s = 0; s < n; ++s) {
      int32_t r = ref[s];
      while (r >= 0 && gmap[r] == 0) { gmap[r] = 1; r = fpar[r]; }
    }
    unsigned long long keyq[F];
    unsigned long long old[F];
    for (int q = 0; q < nf; ++q) {  // frames are allocated parent-first
      if (!gmap[q]) { gmap[q] = -1; continue; }
      const int32_t p = fpar[q];
      const int32_t ph = p == -1 ? -1 : (p >= 0 ? gmap[p] : -2 - p);
      keyq[q] = arena_key(ph, fnode[q], fterm[q]);
      gmap[q] = (int32_t)(mix64(keyq[q]) & A.mask);
      old[q] = atomicCAS(A.keys + gmap[q], kEmptyKey, keyq[q]);
    }
    bool redo = false;
    for (int q = 0; q < nf; ++q) {
      if (gmap[q] < 0) continue;
      if (!redo && (old[q] == kEmptyKey || old[q] == keyq[q])) continue;
      redo = true;  // this frame and everything after: sequential probing
      const int32_t p = fpar[q];
      const int32_t ph = p == -1 ? -1 : (p >= 0 ? gmap[p] : -2 - p);
      keyq[q] = arena_key(ph, fnode[q], fterm[q]);
      const int32_t h = arena_probe(A, keyq[q], mix64(keyq[q]));
      if (h < 0) { err |= kErrArena; return false; }
      gmap[q] = h;
    }
    // known-key cache := the first stack's new frames in chain order (its own
    // frame first, then its interned ancestors); older entries are dropped —
    // the header's ancestor chain stays reachable through external()
    nk = 0;
    if (n > 0)
      for (int32_t r = ref[0]; r >= 0 && nk < K; r = fpar[r]) {
        kh[nk] = gmap[r];
        kk[nk] = keyq[r];
        ++nk;
      }
    int m = n;
    n = 0;
    int32_t or_[S], on_[S];
    for (int s = 0; s < m; ++s) { or_[s] = ref[s]; on_[s] = node[s]; }
    for (int s = 0; s < m; ++s) {
      int32_t r = or_[s];
      if (r >= 0) r = -2 - gmap[r];
      add(r, on_[s]);
    }
    nf = 0;
    return true;
  }
};

// ---------------------------------------------------------------------------
// RWalker: the common-case walker.  At most R stacks, held in registers (every
// array index below is a compile-time constant after unrolling), so a byte
// step is a handful of shared-memory table reads instead of a chain of
// local-memory round trips.  Chain references add a fourth kind,
//     ref >= kChainRef     position i = ref - kChainRef of the slot header's
//                          ancestor chain (xh/xk, shared memory),
// so popping through the cached chain is an index increment.  Pushes use
// walker-local frames (local memory, touched only when a rule is entered).
// Any overflow (more than R stacks, more than F frames) sets `spill`; the
// caller then redoes the walk with the general Walker.
constexpr int32_t kChainRef = 1 << 30;

template <int R, int F>
struct RWalker {
  int32_t ref[R];
  int32_t node[R];
  int n;
  int32_t fpar[F];
  int32_t fnode[F];
  uint8_t fterm[F];
  int nf;
  bool spill;
  uint32_t err;
  const int32_t* xh;
  const unsigned long long* xk;
  int nx;
  int nload;  // arena loads issued (diagnostics)

  __device__ __forceinline__ void init(const int32_t* ch, const unsigned long long* ck, int nc) {
    n = 0; nf = 0; spill = false; err = 0; nload = 0;
    xh = ch; xk = ck; nx = nc;
  }

  // Reference for arena handle h (-1 = empty chain), as a chain position when
  // h heads the cached chain.
  __device__ __forceinline__ int32_t ref_of_handle(int32_t h) const {
    if (h < 0) return -1;
    if (nx > 0 && xh[0] == h) return kChainRef;
    return -2 - h;
  }

  __device__ __forceinline__ unsigned long long global_key(const DevArena& A, int32_t r) {
    if (r >= kChainRef) return xk[r - kChainRef];
    ++nload;
    return arena_load(A, -2 - r);
  }

  __device__ __forceinline__ void pop(const DevArena& A, int32_t r, int32_t& pr, int32_t& pn) {
    if (r >= 0 && r < kChainRef) { pr = fpar[r]; pn = fnode[r]; return; }
    const unsigned long long k = global_key(A, r);
    if (k >= kTombKey) { err |= kErrInvalid; pr = -1; pn = 0; return; }
    pn = key_node(k);
    if (r >= kChainRef && r - kChainRef + 1 < nx) { pr = r + 1; return; }
    const int32_t p = key_parent(k);
    pr = p < 0 ? -1 : -2 - p;
  }

  __device__ __forceinline__ uint32_t term_of(const DevArena& A, int32_t r) {
    if (r == -1) return 1u;
    if (r >= 0 && r < kChainRef) return fterm[r];
    return key_term(global_key(A, r));
  }

  __device__ __forceinline__ int32_t push(const DevGrammar& G, const DevArena& A, int32_t r, int32_t ret) {
    for (int q = nf - 1; q >= 0; --q)
      if (fpar[q] == r && fnode[q] == ret) return q;
    if (nf == F) { spill = true; return r; }
    fpar[nf] = r; fnode[nf] = ret;
    fterm[nf] = (uint8_t)(((G.node_flags[ret] & GM_NODE_POP) ? 1u : 0u) & term_of(A, r));
    return nf++;
  }

  __device__ __forceinline__ void add(int32_t r, int32_t d) {
    bool dup = false;
#pragma unroll
    for (int q = 0; q < R; ++q) dup |= (q < n && ref[q] == r && node[q] == d);
    if (dup) return;
    if (n == R) { spill = true; return; }
#pragma unroll
    for (int q = 0; q < R; ++q)
      if (q == n) { ref[q] = r; node[q] = d; }
    ++n;
  }

  // One byte step; same semantics as Walker::step.
  // kPopFilter (accept and fill walks, which ignore *pop_bottom): also take
  // the pop-filtered moves of the fast table; the cache build's walks keep
  // the general step there, so a pop chain that would reach their synthetic
  // bottom still reports it (ref[0] == -1 is the bottom frame itself).
  template <bool kPopFilter = false>
  __device__ __forceinline__ int step(const DevGrammar& G, const DevArena& A, uint32_t b, bool* pop_bottom) {
    const int c = G.byte_class[b];
    if (n == 1) {  // plain DFA move
      const int32_t f = G.fast[node[0] * G.n_classes + c];
      if (f >= 0) { node[0] = f; return 1; }
      if (f == -1) { n = 0; return 0; }
      if (kPopFilter && f < -2 && ref[0] != -1) {  // pops cannot consume c: move (or die) inside the frame
        if (f == kFastPopDies) { n = 0; return 0; }
        node[0] = -3 - f;
        return 1;
      }
    }
    int32_t nr[R], nn[R];
    int cnt = 0;
#pragma unroll
    for (int s = 0; s < R; ++s) {
      if (s >= n) break;
      int32_t r = ref[s], m = node[s];
      while (true) {
        const int32_t idx = m * G.n_classes + c;
        const int32_t t0 = G.trans_off[idx], t1 = G.trans_off[idx + 1];
        for (int32_t t = t0; t < t1; ++t) {
          const int2 tr = G.trans[t];
          int32_t d = tr.x;
          const int plen = (int)((uint32_t)tr.y >> 24);
          const int poff = tr.y & 0xFFFFFF;
          int32_t rr = r;
          for (int k = 0; k < plen; ++k) rr = push(G, A, rr, G.push_pool[poff + k]);
          if (plen == 0) {
            while ((G.node_flags[d] & GM_NODE_DEAD_END) && rr != -1) {
              int32_t pr, pn;
              pop(A, rr, pr, pn);
              rr = pr; d = pn;
              if ((uint32_t)d >= (uint32_t)G.n_nodes) { err |= 1u << 29; d = 0; rr = -1; }
            }
          }
          bool dup = false;
#pragma unroll
          for (int q = 0; q < R; ++q) dup |= (q < cnt && nr[q] == rr && nn[q] == d);
          if (!dup) {
            if (cnt == R) {
              spill = true;
            } else {
#pragma unroll
              for (int q = 0; q < R; ++q)
                if (q == cnt) { nr[q] = rr; nn[q] = d; }
              ++cnt;
            }
          }
        }
        if (!(G.node_flags[m] & GM_NODE_POP)) break;
        if (r == -1) { *pop_bottom = true; break; }
        pop(A, r, r, m);
        if ((uint32_t)m >= (uint32_t)G.n_nodes) { err |= 1u << 28; break; }
      }
    }
#pragma unroll
    for (int q = 0; q < R; ++q) { ref[q] = nr[q]; node[q] = nn[q]; }
    n = cnt;
    return cnt;
  }

  // Arena handle of a chain / global reference (not for local frames).
  __device__ __forceinline__ int32_t handle_of(int32_t r) const {
    if (r == -1) return -1;
    if (r >= kChainRef) return xh[r - kChainRef];
    return -2 - r;
  }
};

// Ancestor chain of the first top, ordered from its own frame upward.
struct Chain {
  int32_t h[kChain];
  unsigned long long k[kChain];
  int n;
};

// Intern an RWalker's surviving stacks (speculative parallel CAS as in
// Walker::intern_all), write them as (handle, node) to out[] (deduplicated),
// and build the first top's ancestor chain: its new frames, then the cached
// chain of the previous header from the first frame they share.  Returns the
// number of tops, or -1 on arena exhaustion.
template <int R, int F>
__device__ inline int rwalker_commit(RWalker<R, F>& w, const DevArena& A, int2* out, Chain& ch) {
  int32_t gmap[F];
  unsigned long long keyq[F], old[F];
  for (int q = 0; q < w.nf; ++q) gmap[q] = 0;
#pragma unroll
  for (int s = 0; s < R; ++s) {
    if (s >= w.n) break;
    int32_t r = w.ref[s];
    while (r >= 0 && r < kChainRef && gmap[r] == 0) { gmap[r] = 1; r = w.fpar[r]; }
  }
  auto parent_handle = [&](int32_t p) -> int32_t {
    if (p == -1) return -1;
    if (p >= kChainRef) return w.xh[p - kChainRef];
    if (p >= 0) return gmap[p];
    return -2 - p;
  };
  for (int q = 0; q < w.nf; ++q) {
    if (!gmap[q]) { gmap[q] = -1; continue; }
    keyq[q] = arena_key(parent_handle(w.fpar[q]), w.fnode[q], w.fterm[q]);
    gmap[q] = (int32_t)(mix64(keyq[q]) & A.mask);
    old[q] = atomicCAS(A.keys + gmap[q], kEmptyKey, keyq[q]);
  }
  bool redo = false;
  for (int q = 0; q < w.nf; ++q) {
    if (gmap[q] < 0) continue;
    if (!redo && (old[q] == kEmptyKey || old[q] == keyq[q])) continue;
    redo = true;
    keyq[q] = arena_key(parent_handle(w.fpar[q]), w.fnode[q], w.fterm[q]);
    const int32_t h = arena_probe(A, keyq[q], mix64(keyq[q]));
    if (h < 0) return -1;
    gmap[q] = h;
  }
  int n = 0;
#pragma unroll
  for (int s = 0; s < R; ++s) {
    if (s >= w.n) break;
    const int32_t r = w.ref[s];
    const int32_t h = (r >= 0 && r < kChainRef) ? gmap[r] : w.handle_of(r);
    bool dup = false;
    for (int q = 0; q < n; ++q) dup |= (out[q].x == h && out[q].y == w.node[s]);
    if (!dup) out[n++] = make_int2(h, w.node[s]);
  }
  // chain of the first top
  ch.n = 0;
  if (w.n > 0) {
    int32_t r = w.ref[0];
    while (r >= 0 && r < kChainRef && ch.n < kChain) {
      ch.h[ch.n] = gmap[r];
      ch.k[ch.n] = keyq[r];
      ++ch.n;
      r = w.fpar[r];
    }
    int i = -1;
    if (r >= kChainRef) {
      i = r - kChainRef;
    } else if (r <= -2) {
      const int32_t h = -2 - r;
      for (int j = 0; j < w.nx; ++j)
        if (w.xh[j] == h) { i = j; break; }
    }
    if (i >= 0)
      for (; i < w.nx && ch.n < kChain; ++i) {
        ch.h[ch.n] = w.xh[i];
        ch.k[ch.n] = w.xk[i];
        ++ch.n;
      }
  }
  return n;
}

// ---------------------------------------------------------------------------
// Overflow walker.  The register and local-memory walkers above hold at most
// 2-32 stacks; a walk that exceeds them (ambiguous grammars keep one stack
// per live alternative) is redone here with its stack sets in global-memory
// scratch, every pushed frame interned into the arena at once, and dedupe
// through a generation-tagged hash set — up to kWideCap stacks, the
// reference's branch cap (REF matcher.py:116 DEFAULT_BRANCH_CAP = 4096,
// cache.py:58, pda.py:53; exceeding it raises there and here).  Scratch comes
// in "lanes" (pool- or build-level), taken by one thread for the duration of
// one walk (spin lock: holders never wait on anything, so it cannot
// deadlock).
constexpr int kWideCap = 4096;
constexpr int kHashCap = 2 * kWideCap;  // power of two

struct DevOverflow {
  int2* bufs;                  // [lanes][2][kWideCap]
  unsigned long long* hkeys;   // [lanes][kHashCap]
  uint32_t* hgen;              // [lanes][kHashCap]
  uint32_t* gen;               // [lanes]
  int32_t* lock;               // [lanes]
  int32_t lanes;
};

struct BigWalk {
  DevOverflow O;
  int lane;
  int2* cur;
  int2* nxt;
  int n;
  uint32_t err;

  __device__ void acquire(const DevOverflow& ov, uint32_t hint) {
    O = ov;
    n = 0;
    err = 0;
    lane = -1;
    for (uint32_t i = hint;; ++i) {
      const int l = (int)(i % (uint32_t)O.lanes);
      if (atomicCAS(O.lock + l, 0, 1) == 0) { lane = l; break; }
      if ((i - hint) % (uint32_t)O.lanes == (uint32_t)O.lanes - 1) __nanosleep(256);
    }
    __threadfence();
    cur = O.bufs + (size_t)lane * 2 * kWideCap;
    nxt = cur + kWideCap;
  }
  __device__ void release() {
    __threadfence();
    atomicExch(O.lock + lane, 0);
  }
  // fresh dedupe set for the next generation of stacks
  __device__ void new_set() {
    uint32_t g = O.gen[lane] + 1;
    if (g == 0) {  // wrapped: clear the tags
      uint32_t* t = O.hgen + (size_t)lane * kHashCap;
      for (int i = 0; i < kHashCap; ++i) t[i] = 0;
      g = 1;
    }
    O.gen[lane] = g;
  }
  // append (h, node) to `out` (count *cnt) unless already present
  __device__ void add_to(int2* out, int* cnt, int32_t h, int32_t node) {
    const unsigned long long key = ((unsigned long long)(uint32_t)(h + 1) << 32) | (uint32_t)node;
    const uint32_t g = O.gen[lane];
    unsigned long long* hk = O.hkeys + (size_t)lane * kHashCap;
    uint32_t* hg = O.hgen + (size_t)lane * kHashCap;
    for (uint32_t i = mix64(key) & (kHashCap - 1);; i = (i + 1) & (kHashCap - 1)) {
      if (hg[i] != g) {
        if (*cnt >= kWideCap) { err |= kErrCap; return; }
        hg[i] = g;
        hk[i] = key;
        out[(*cnt)++] = make_int2(h, node);
        return;
      }
      if (hk[i] == key) return;
    }
  }
  __device__ void start() { new_set(); n = 0; }
  __device__ void add(int32_t h, int32_t node) { add_to(cur, &n, h, node); }

  __device__ uint32_t term_of(const DevArena& A, int32_t h) {
    if (h < 0) return 1u;
    const unsigned long long k = arena_load(A, h);
    if (k >= kTombKey) { err |= kErrInvalid; return 0u; }
    return key_term(k);
  }
  __device__ void pop(const DevArena& A, int32_t h, int32_t& ph, int32_t& pn) {
    const unsigned long long k = arena_load(A, h);
    if (k >= kTombKey) { err |= kErrInvalid; ph = -1; pn = 0; return; }
    ph = key_parent(k);
    pn = key_node(k);
  }

  // One byte step of the whole set, Walker::step semantics, all frames
  // interned.  Returns the number of live stacks.
  __device__ int step(const DevGrammar& G, const DevArena& A, uint32_t b, bool* pop_bottom) {
    const int c = G.byte_class[b];
    new_set();
    int cnt = 0;
    for (int s = 0; s < n && !err; ++s) {
      int32_t h = cur[s].x, m = cur[s].y;
      while (true) {
        const int32_t idx = m * G.n_classes + c;
        const int32_t t0 = G.trans_off[idx], t1 = G.trans_off[idx + 1];
        for (int32_t t = t0; t < t1; ++t) {
          const int2 tr = G.trans[t];
          int32_t d = tr.x;
          const int plen = (int)((uint32_t)tr.y >> 24);
          const int poff = tr.y & 0xFFFFFF;
          int32_t hh = h;
          for (int k = 0; k < plen; ++k) {
            const int32_t ret = G.push_pool[poff + k];
            const uint32_t term = ((G.node_flags[ret] & GM_NODE_POP) ? 1u : 0u) & term_of(A, hh);
            hh = arena_intern(A, hh, ret, term);
            if (hh < 0) { err |= kErrArena; return 0; }
          }
          if (plen == 0)
            while ((G.node_flags[d] & GM_NODE_DEAD_END) && hh >= 0) pop(A, hh, hh, d);
          add_to(nxt, &cnt, hh, d);
        }
        if (!(G.node_flags[m] & GM_NODE_POP)) break;
        if (h < 0) { *pop_bottom = true; break; }
        pop(A, h, h, m);
        if ((uint32_t)m >= (uint32_t)G.n_nodes) { err |= kErrInvalid; break; }
      }
    }
    int2* t = cur; cur = nxt; nxt = t;
    n = err ? 0 : cnt;
    return n;
  }
};

// ---------------------------------------------------------------------------
// Allowed-continuation check of the context-expansion DFA (REF cache.py:
// 303-333 FollowFsa.allows): may some legal continuation of rule `rid` start
// with (or extend) data[0:len)?
__device__ __forceinline__ bool follow_allows(const DevGrammar& G, int32_t rid, const uint8_t* data, int len) {
  int32_t s = __ldg(G.follow_start + rid);
  for (int i = 0; i < len; ++i) {
    if (s == GM_FOLLOW_ANY) return true;
    if (s == GM_FOLLOW_DEAD) return false;
    s = __ldg(G.follow_next + s * G.n_classes + G.byte_class[data[i]]);
  }
  return s != GM_FOLLOW_DEAD;
}

// ---------------------------------------------------------------------------
// Matcher pool: ring of (window+1) top sets per slot (REF matcher.py:239-244
// history, 310-326 rollback) plus the slot header.

// Current-state summary of a slot, one 256-byte record written by every state
// change (reset / accept / rollback / recycle / fork): all a fill or accept
// needs to start, in one coalesced load.
constexpr int kHdrTops = 8;
struct __align__(16) SlotHdr {
  const uint8_t* blob;         // binding blob (walker tables + node_info)
  const uint32_t* acc_rows;
  const uint32_t* universe;
  const int4* dep_ent;
  const int4* tokrec;
  int32_t blob_bytes, V, W, eos;
  int32_t ntops;               // -1: more than kHdrTops stacks (read the ring)
  int32_t flags;               // bit0 terminated, bit1 terminable
  int32_t key[kHdrTops];
  int32_t dep_lo[kHdrTops];
  int32_t dep_hi[kHdrTops];
  int2 top[kHdrTops];
  // ancestor-chain cache: arena keys of the tops' chain frames (top 0's chain
  // first), so walks pop through the first kChain frames without touching
  // the arena
  int32_t nchain;
  int32_t wide_owned;          // 1: some ring entry of the slot holds a wide block (release on restart)
  int32_t chain_h[kChain];
  int32_t pad1[2];
  unsigned long long chain_k[kChain];
  int32_t pad2[20];
};
static_assert(sizeof(SlotHdr) == 512, "SlotHdr layout");
constexpr int kHdrVec = sizeof(SlotHdr) / 16;  // int4 per header

struct DevPool {
  int32_t capacity, max_stacks, H;
  int2* tops;                 // [capacity][H][max_stacks] (handle, node)
  int32_t* meta;              // [capacity][H]: n_stacks | terminated << 16
  int32_t* head;              // [capacity]
  int32_t* hist_len;          // [capacity]
  int32_t* window;            // [capacity]
  const DevBinding** binding; // [capacity]
  DevArena arena;
  uint32_t* err;              // [capacity] per-slot sticky error bits (GM_ERR_* as 1 << code)
  // wide top sets (more than max_stacks stacks, up to kWideCap): a ring
  // entry's stacks then live in a block of wide_pool, owned by that (slot,
  // ring position) until the slot is reset / recycled
  int2* wide_pool;            // [n_wide][kWideCap]
  int32_t* wide;              // [capacity][H] block index or -1
  uint32_t* wide_bits;        // allocation bitmap [ceil(n_wide/32)]
  int32_t n_wide;
  DevOverflow ovf;            // overflow-walker scratch lanes
  SlotHdr* hdr;               // [capacity]
  unsigned long long* trace;  // optional phase timestamps (GMASK_TRACE=1), else null
  int32_t trace_ring;         // GMASK_TRACE=2: launches kept per CTA (back-to-back timelines), else 0
  // launch hint: the binding every bound slot shares (host bookkeeping,
  // gm_pool_reset / fork), or null.  Grammar blobs and token records are
  // immutable, so a step kernel may start staging them before its
  // griddepcontrol.wait and before its slot header arrives; it still checks
  // the header's binding and restages on a mismatch.
  const uint8_t* hint_blob;
  const int4* hint_tokrec;
  int32_t hint_blob_bytes, hint_V;
  // host-side launch setting: the pool's hot block (arena + slot headers +
  // ring positions) as an L2 persisting access-policy window, or null
  void* l2_base;
  size_t l2_bytes;
  float l2_hit;
};

// Phase timestamps of CTA 0 (diagnostics only): trace[kernel*16 + phase].
// Compiled in only with -DGM_TRACE_MARKS: even untaken, the calls sit in
// every thread's path and ncu attributed ~13 % of K5's warp samples
// (branch resolution) to them; the per-CTA timeline (GMASK_TRACE=1)
// supersedes them.
__device__ __forceinline__ void trace_mark(const DevPool& P, int kernel, int phase) {
#ifdef GM_TRACE_MARKS
  if (P.trace && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    P.trace[kernel * 16 + phase] = t;
  }
#else
  (void)P; (void)kernel; (void)phase;
#endif
}

__device__ __forceinline__ int2* slot_tops(const DevPool& P, int32_t slot, int32_t h) {
  return P.tops + ((size_t)slot * P.H + h) * P.max_stacks;
}

// Per-slot error reporting: the request whose operation failed gets the bit
// (REF raises MatcherError on that matcher, matcher.py:188-189, 379-381).
__device__ __forceinline__ void slot_error(const DevPool& P, int32_t slot, uint32_t bits) {
  if (bits) atomicOr(P.err + slot, bits);
}

// Stacks of ring entry h holding n stacks (inline or in its wide block).
__device__ __forceinline__ const int2* ring_tops(const DevPool& P, int32_t slot, int32_t h, int n) {
  if (n <= P.max_stacks) return slot_tops(P, slot, h);
  const int32_t b = P.wide[(size_t)slot * P.H + h];
  return b >= 0 ? P.wide_pool + (size_t)b * kWideCap : slot_tops(P, slot, h);
}

// Destination for n stacks in ring entry h: inline, or the entry's wide
// block (allocated on first use); null when n exceeds the cap or no block is
// free.
__device__ inline int2* ring_tops_w(const DevPool& P, int32_t slot, int32_t h, int n) {
  if (n <= P.max_stacks) return slot_tops(P, slot, h);
  if (n > kWideCap || P.n_wide <= 0) return nullptr;
  int32_t* wb = P.wide + (size_t)slot * P.H + h;
  if (*wb >= 0) return P.wide_pool + (size_t)*wb * kWideCap;
  const int nw = (P.n_wide + 31) >> 5;
  for (int w0 = 0; w0 < nw; ++w0) {
    const int w = (w0 + slot) % nw;
    for (;;) {
      const uint32_t cur = ((volatile uint32_t*)P.wide_bits)[w];
      const uint32_t avail = ~cur & (w == nw - 1 && (P.n_wide & 31) ? ((1u << (P.n_wide & 31)) - 1u) : ~0u);
      if (!avail) break;
      const int bit = __ffs(avail) - 1;
      if (!(atomicOr(P.wide_bits + w, 1u << bit) & (1u << bit))) {
        *wb = w * 32 + bit;
        return P.wide_pool + (size_t)*wb * kWideCap;
      }
    }
  }
  return nullptr;
}

// Return every wide block of a slot (reset / recycle / fork target).
__device__ inline void release_wide(const DevPool& P, int32_t slot, int lane = 0, int nlanes = 1) {
  if (P.n_wide <= 0) return;
  for (int h = lane; h < P.H; h += nlanes) {
    int32_t* wb = P.wide + (size_t)slot * P.H + h;
    const int32_t b = *wb;
    if (b >= 0) {
      atomicAnd(P.wide_bits + (b >> 5), ~(1u << (b & 31)));
      *wb = -1;
    }
  }
}

__device__ __forceinline__ void load_header(const DevPool& P, int32_t slot, SlotHdr* s_hdr) {
  if (threadIdx.x < kHdrVec)
    reinterpret_cast<int4*>(s_hdr)[threadIdx.x] = reinterpret_cast<const int4*>(P.hdr + slot)[threadIdx.x];
}

__device__ __forceinline__ void header_pointers(SlotHdr& h, const DevBinding* B) {
  h.blob = B->c.blob;
  h.acc_rows = B->c.acc_rows;
  h.universe = B->v.universe;
  h.dep_ent = B->c.dep_ent;
  h.tokrec = B->v.tokrec;
  h.blob_bytes = B->c.blob_bytes;
  h.V = B->v.V;
  h.W = B->v.W;
  h.eos = B->v.eos;
}

// Chain of handle `cur`: first from `fresh` (frames just interned, already in
// chain order), then by splicing the previous header's chain at the first
// frame they share — no arena traffic, no quadratic scans.
__device__ inline void build_chain(Chain& c, int32_t cur, const int32_t* fh, const unsigned long long* fk, int nfresh,
                                   const SlotHdr& old) {
  c.n = 0;
  for (int i = 0; i < nfresh && cur >= 0 && c.n < kChain; ++i) {
    if (fh[i] != cur) break;
    c.h[c.n] = cur;
    c.k[c.n] = fk[i];
    ++c.n;
    cur = key_parent(fk[i]);
  }
  if (cur < 0) return;
  int j = 0;
  while (j < old.nchain && old.chain_h[j] != cur) ++j;
  for (; j < old.nchain && c.n < kChain; ++j) {
    c.h[c.n] = old.chain_h[j];
    c.k[c.n] = old.chain_k[j];
    ++c.n;
  }
}

// Fill the state part of a header from (tops, n, terminated) and the first
// top's ancestor chain.  `G` must be a binding view (node_info present).
// Only the EOS fact may need an arena load (a top whose frame is unknown).
__device__ inline void header_state(const DevPool& P, SlotHdr& h, const DevGrammar& G, const int2* tops, int n,
                                    int terminated, const Chain* chain) {
  int term = 0, blend = 0;
  for (int s = 0; s < n; ++s) {
    const int2 t = tops[s];
    if (!terminated && !term && (G.node_flags[t.y] & GM_NODE_POP)) {
      if (t.x < 0) {
        term = 1;
      } else {
        const unsigned long long k = (s == 0 && chain && chain->n && chain->h[0] == t.x)
                                         ? chain->k[0] : arena_load(P.arena, t.x);
        term = (int)key_term(k);
      }
    }
    if (s < kHdrTops) {
      const int4 ni = G.node_info[t.y];
      h.key[s] = ni.x;
      h.dep_lo[s] = ni.y;
      h.dep_hi[s] = ni.z;
      h.top[s] = t;
      blend |= (ni.w >> 28) & 4;
    }
  }
  const int nc = (chain && n > 0) ? chain->n : 0;
  for (int i = 0; i < nc; ++i) {
    h.chain_h[i] = chain->h[i];
    h.chain_k[i] = chain->k[i];
  }
  h.nchain = nc;
  h.ntops = n <= kHdrTops ? n : -1;
  h.flags = (terminated ? 1 : 0) | (term ? 2 : 0) | blend;  // 4: a top's row is applied blended
}

// rwalker_commit for the fused step kernel: interns exactly like
// rwalker_commit, but writes the first top's ancestor chain straight into
// the shared-memory header `h` (whose chain the walker used as its external
// chain, w.xh/w.xk == h.chain_h/h.chain_k): the surviving part of the old
// chain is shifted in place and the fresh frames written in front — no
// walker-local Chain copy (16 local-memory round trips per accept).
// Deferred interning (fused step kernel, single surviving stack): a fresh
// frame's handle is its key's hash slot unless a different key sits there,
// so the commit uses the slots as handles at once and leaves the CASes to
// another warp, whose results are checked only at the end of the kernel
// (spec_fixup re-interns and rewrites the published state on the rare
// collision).  The step's mask never depends on fresh handle values: fresh
// frames sit in the header's ancestor chain and are walked by position.
constexpr int kSpecMax = 8;
struct SpecOut {
  int n;                             // fresh frames awaiting their CAS (0: committed synchronously)
  int32_t slot[kSpecMax];            // speculative handle = hash slot, push order (parents first)
  unsigned long long key[kSpecMax];  // keys, parents as speculative handles
};

template <int R, int F>
__device__ inline int rwalker_commit_inplace(RWalker<R, F>& w, const DevArena& A, int2* out, SlotHdr& h,
                                             SpecOut* spec = nullptr) {
  // scratch in shared memory: one committing thread per CTA (the accept
  // thread); local-memory arrays here cost an L2 round trip per access
  __shared__ int32_t gmap[F];
  __shared__ unsigned long long keyq[F];
  for (int q = 0; q < w.nf; ++q) gmap[q] = 0;
#pragma unroll
  for (int s = 0; s < R; ++s) {
    if (s >= w.n) break;
    int32_t r = w.ref[s];
    while (r >= 0 && r < kChainRef && gmap[r] == 0) { gmap[r] = 1; r = w.fpar[r]; }
  }
  auto parent_handle = [&](int32_t p) -> int32_t {
    if (p == -1) return -1;
    if (p >= kChainRef) return w.xh[p - kChainRef];
    if (p >= 0) return gmap[p];
    return -2 - p;
  };
  // speculative handles (a frame's slot = its key's hash), then the CASes
  // issued in batches of 8 with their results in registers, so the atomic
  // round trips overlap instead of serialising on a local-memory store
  for (int q = 0; q < w.nf; ++q) {
    if (!gmap[q]) { gmap[q] = -1; continue; }
    keyq[q] = arena_key(parent_handle(w.fpar[q]), w.fnode[q], w.fterm[q]);
    gmap[q] = (int32_t)(mix64(keyq[q]) & A.mask);
  }
  bool redo = false;
  bool deferred = false;
  if (spec) {  // single stack, <= kSpecMax fresh frames on pairwise distinct slots: defer the CASes
    spec->n = 0;
    if (w.n == 1) {
      int k = 0;
      deferred = true;
      for (int q = 0; q < w.nf && deferred; ++q) {
        if (gmap[q] < 0) continue;
        if (k == kSpecMax) { deferred = false; break; }
        for (int j = 0; j < k; ++j) deferred &= spec->slot[j] != gmap[q];
        spec->slot[k] = gmap[q];
        spec->key[k] = keyq[q];
        ++k;
      }
      if (deferred) spec->n = k;
    }
  }
  constexpr int kBatch = 8;
  for (int q0 = 0; q0 < w.nf && !deferred; q0 += kBatch) {
    unsigned long long res[kBatch];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const int q = q0 + j;
      res[j] = kEmptyKey;
#ifdef GM_EXPERIMENT_NO_CAS  // timing experiment only: assumes no collision
      if (q < w.nf && gmap[q] >= 0) { A.keys[gmap[q]] = keyq[q]; res[j] = kEmptyKey; }
#else
      if (q < w.nf && gmap[q] >= 0) res[j] = atomicCAS(A.keys + gmap[q], kEmptyKey, keyq[q]);
#endif
    }
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const int q = q0 + j;
      if (q >= w.nf || gmap[q] < 0) continue;
      if (!redo && (res[j] == kEmptyKey || res[j] == keyq[q])) continue;
      redo = true;  // collision: this frame and every later one probe serially
      keyq[q] = arena_key(parent_handle(w.fpar[q]), w.fnode[q], w.fterm[q]);
      const int32_t hh = arena_probe(A, keyq[q], mix64(keyq[q]));
      if (hh < 0) return -1;
      gmap[q] = hh;
    }
  }
  int n = 0;
#pragma unroll
  for (int s = 0; s < R; ++s) {
    if (s >= w.n) break;
    const int32_t r = w.ref[s];
    const int32_t hh = (r >= 0 && r < kChainRef) ? gmap[r] : w.handle_of(r);
    bool dup = false;
    for (int q = 0; q < n; ++q) dup |= (out[q].x == hh && out[q].y == w.node[s]);
    if (!dup) out[n++] = make_int2(hh, w.node[s]);
  }
  // chain of the first top = its fresh frames, then the old chain from the
  // first frame they share
  int nfresh = 0;
  int32_t r = w.n > 0 ? w.ref[0] : -1;
  const int32_t r0 = r;
  while (r >= 0 && r < kChainRef && nfresh < kChain) { ++nfresh; r = w.fpar[r]; }
  int from = -1;
  if (r >= 0 && r < kChainRef) {
    from = -1;  // more fresh frames than the chain holds: old part not reached
  } else if (r >= kChainRef) {
    from = r - kChainRef;
  } else if (r <= -2) {
    const int32_t hh = -2 - r;
    for (int j = 0; j < w.nx; ++j)
      if (w.xh[j] == hh) { from = j; break; }
  }
  const int on = h.nchain;
  const int nold = from >= 0 ? min(on - from, kChain - nfresh) : 0;
  if (nold > 0 && from != nfresh) {
    if (nfresh < from) {
      for (int j = 0; j < nold; ++j) { h.chain_h[nfresh + j] = h.chain_h[from + j]; h.chain_k[nfresh + j] = h.chain_k[from + j]; }
    } else {
      for (int j = nold - 1; j >= 0; --j) { h.chain_h[nfresh + j] = h.chain_h[from + j]; h.chain_k[nfresh + j] = h.chain_k[from + j]; }
    }
  }
  r = r0;
  for (int j = 0; j < nfresh; ++j) {
    h.chain_h[j] = gmap[r];
    h.chain_k[j] = keyq[r];
    r = w.fpar[r];
  }
  h.nchain = nfresh + max(nold, 0);
  return n;
}

constexpr int kHdrStateVec = 3;  // first int4 holding state (ntops at byte 56)
static_assert(offsetof(SlotHdr, ntops) >= kHdrStateVec * 16, "header state offset");
// header_state for a header whose ancestor chain (chain_h/chain_k/nchain)
// has already been rewritten in place (rwalker_commit_inplace): same state
// fields, no chain copy.
__device__ inline void header_state_inplace(const DevPool& P, SlotHdr& h, const DevGrammar& G, const int2* tops, int n,
                                            int terminated) {
  int term = 0, blend = 0;
  for (int s = 0; s < n; ++s) {
    const int2 t = tops[s];
    if (!terminated && !term && (G.node_flags[t.y] & GM_NODE_POP)) {
      if (t.x < 0) {
        term = 1;
      } else {
        const unsigned long long k = (s == 0 && h.nchain && h.chain_h[0] == t.x) ? h.chain_k[0] : arena_load(P.arena, t.x);
        term = (int)key_term(k);
      }
    }
    if (s < kHdrTops) {
      const int4 ni = G.node_info[t.y];
      h.key[s] = ni.x;
      h.dep_lo[s] = ni.y;
      h.dep_hi[s] = ni.z;
      h.top[s] = t;
      blend |= (ni.w >> 28) & 4;
    }
  }
  if (n == 0) h.nchain = 0;
  h.ntops = n <= kHdrTops ? n : -1;
  h.flags = (terminated ? 1 : 0) | (term ? 2 : 0) | blend;  // 4: a top's row is applied blended
}

// Publish the state part of a shared-memory header with the lanes of one
// warp (one 16-byte store each) — the deferred counterpart of
// store_header_state for the fused step kernel.
__device__ __forceinline__ void store_header_state_warp(const DevPool& P, int32_t slot, const SlotHdr& h, int lane) {
  const int i = kHdrStateVec + lane;
  if (i < kHdrVec) reinterpret_cast<int4*>(P.hdr + slot)[i] = reinterpret_cast<const int4*>(&h)[i];
}

__device__ inline void store_header(const DevPool& P, int32_t slot, const SlotHdr& h) {
  const int4* src = reinterpret_cast<const int4*>(&h);
  int4* dst = reinterpret_cast<int4*>(P.hdr + slot);
#pragma unroll
  for (int i = 0; i < kHdrVec; ++i) dst[i] = src[i];
}

// Publish the state part of a header (everything after the binding pointers
// and sizes, which never change for a slot) with 16-byte stores.
__device__ inline void store_header_state(const DevPool& P, int32_t slot, const SlotHdr& h) {
  const int4* src = reinterpret_cast<const int4*>(&h);
  int4* dst = reinterpret_cast<int4*>(P.hdr + slot);
#pragma unroll
  for (int i = kHdrStateVec; i < kHdrVec; ++i) dst[i] = src[i];
}

// Collision repair of a deferred commit (rare): re-intern the fresh frames in
// push order with their parents' real handles, then rewrite the shared
// header's chain and first top and republish it and the ring entry.
// Real handles of a deferred commit's fresh frames (push order, parents
// first): probe each with its parent's real handle.  Idempotent (hash-consed:
// every caller gets the same handles, whether or not the speculative CAS has
// landed yet).  False on arena exhaustion.
__device__ inline bool spec_real_handles(const DevArena& A, const SpecOut& sp, int32_t* real,
                                         unsigned long long* rkey) {
  for (int k = 0; k < sp.n; ++k) {
    int32_t ph = key_parent(sp.key[k]);
    for (int j = 0; j < k; ++j)
      if (sp.slot[j] == ph) { ph = real[j]; break; }
    rkey[k] = arena_key(ph, key_node(sp.key[k]), key_term(sp.key[k]));
    real[k] = arena_probe(A, rkey[k], mix64(rkey[k]));
    if (real[k] < 0) return false;
  }
  return true;
}

// A fresh frame is identified by (speculative slot, key): an older ancestor
// whose real handle happens to equal a fresh frame's slot (the very key that
// caused the collision may be that ancestor) has a different key and keeps
// its handle.  Fresh frames sit at the front of the chain.
__device__ __forceinline__ int spec_fresh_index(const SpecOut& sp, int32_t hh, unsigned long long kk) {
  for (int j = 0; j < sp.n; ++j)
    if (sp.slot[j] == hh && sp.key[j] == kk) return j;
  return -1;
}

// Rewrite a chain copy (and the top handle *th when it heads the chain) to
// real handles.  Used by walks that look frames up by handle (the general
// and overflow walkers) while a deferred commit's CASes may be in flight.
__device__ inline bool spec_realize(const DevArena& A, const SpecOut& sp, int32_t* ch_h, unsigned long long* ch_k,
                                    int nc, int32_t* th) {
  int32_t real[kSpecMax];
  unsigned long long rkey[kSpecMax];
  if (!spec_real_handles(A, sp, real, rkey)) return false;
  for (int i = 0; i < nc; ++i) {
    const int j = spec_fresh_index(sp, ch_h[i], ch_k[i]);
    if (j < 0) break;
    if (i == 0 && *th == ch_h[0]) *th = real[j];
    ch_h[i] = real[j];
    ch_k[i] = rkey[j];
  }
  return true;
}

__device__ inline bool spec_fixup(const DevPool& P, int32_t slot, const SpecOut& sp, SlotHdr& h) {
  int32_t real[kSpecMax];
  unsigned long long rkey[kSpecMax];
  if (!spec_real_handles(P.arena, sp, real, rkey)) {
    slot_error(P, slot, kErrArena);
    return false;
  }
  // the single surviving top is fresh iff chain position 0 is
  const int32_t top_old = h.ntops > 0 ? h.top[0].x : -1;
  const int top_j = (h.nchain > 0 && h.chain_h[0] == top_old) ? spec_fresh_index(sp, h.chain_h[0], h.chain_k[0]) : -1;
  for (int i = 0; i < h.nchain; ++i) {
    const int j = spec_fresh_index(sp, h.chain_h[i], h.chain_k[i]);
    if (j < 0) break;  // past the fresh frames: the rest of the chain is older
    h.chain_h[i] = real[j];
    h.chain_k[i] = rkey[j];
  }
  if (top_j >= 0) {
    h.top[0].x = real[top_j];
    const int32_t head = P.head[slot];
    int2* ring = slot_tops(P, slot, head);  // deferred commits keep one stack: ring entry 0 is the top
    if (ring[0].x == top_old) ring[0].x = real[top_j];
  }
  store_header_state(P, slot, h);
  return true;
}

// Rebuild a slot header from the binding (reset / recycle / rollback path).
__device__ inline void write_header(const DevPool& P, int32_t slot, const DevBinding* B, const int2* tops, int n,
                                    int terminated, int wide_owned) {
  SlotHdr h;
  header_pointers(h, B);
  h.wide_owned = wide_owned;
  const DevGrammar G = blob_view(B->c.blob);
  header_state(P, h, G, tops, n, terminated, nullptr);
  store_header(P, slot, h);
}


}  // namespace gm
