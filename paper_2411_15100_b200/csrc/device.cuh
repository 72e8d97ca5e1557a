// Device-side data model shared by the cache builder (K1), fill (K2) and
// accept (K4) kernels: grammar tables, vocabulary, the hash-consed stack
// arena, and the byte-level stack-set walker.
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
  // The walker tables (byte_class .. key_of_node) live in one contiguous
  // 16-byte-aligned blob so a CTA can stage them into shared memory with a
  // single coalesced copy.
  const uint8_t* blob;
  int32_t blob_bytes;
};

constexpr int kStageBytes = 32 * 1024;  // shared-memory budget for staged tables

// Cooperative copy of the grammar blob into shared memory; returns a view
// whose table pointers address the shared copy (or the global tables when
// the blob does not fit).  Must be called by every thread of the CTA.
__device__ __forceinline__ DevGrammar stage_grammar(const DevGrammar& G, uint8_t* smem) {
  DevGrammar g = G;
  if (G.blob_bytes > kStageBytes) return g;
  const int4* src = reinterpret_cast<const int4*>(G.blob);
  int4* dst = reinterpret_cast<int4*>(smem);
  for (int i = threadIdx.x; i < G.blob_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
  auto rb = [&](const void* p) { return smem + (reinterpret_cast<const uint8_t*>(p) - G.blob); };
  g.byte_class = rb(G.byte_class);
  g.node_flags = rb(G.node_flags);
  g.trans_off = reinterpret_cast<const int32_t*>(rb(G.trans_off));
  g.trans = reinterpret_cast<const int2*>(rb(G.trans));
  g.push_pool = reinterpret_cast<const int32_t*>(rb(G.push_pool));
  g.key_of_node = reinterpret_cast<const int32_t*>(rb(G.key_of_node));
  g.node_rule = reinterpret_cast<const int32_t*>(rb(G.node_rule));
  return g;
}

struct DevVocab {
  int32_t V, W, n_sorted, eos;
  const uint8_t* bytes;
  const int32_t* off;          // [V+1]
  const int32_t* sorted_ids;   // non-special non-empty ids, lexicographic
  const uint32_t* universe;    // [W]
  const uint8_t* reject;       // [V] 1 = special or empty (never accepted)
};

struct DevCache {
  const uint32_t* acc_rows;    // [n_keys*W]
  const int32_t* dep_off;      // [n_keys+1]
  const int32_t* dep_ids;
  const int4* dep_ent;         // [n_dep]: (token id, byte offset, length, 0)
  const uint8_t* dep_bytes;    // dependent tokens' bytes, contiguous
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
__device__ __forceinline__ unsigned long long arena_load(const DevArena& A, int32_t h) {
  return *reinterpret_cast<volatile const unsigned long long*>(A.keys + h);
}
__device__ __forceinline__ int32_t key_parent(unsigned long long k) { return (int32_t)(uint32_t)(k >> 32) - 1; }
__device__ __forceinline__ int32_t key_node(unsigned long long k) { return (int32_t)((uint32_t)k >> 1); }
__device__ __forceinline__ uint32_t key_term(unsigned long long k) { return (uint32_t)k & 1u; }

// Returns the handle of (parent, node), inserting it if absent; -1 + error
// bit when the table is full.
__device__ inline int32_t arena_intern(const DevArena& A, int32_t parent, int32_t node, uint32_t term) {
  const unsigned long long key = arena_key(parent, node, term);
  uint32_t i = mix64(key) & A.mask;
  for (int probe = 0; probe < 8192; ++probe) {
    unsigned long long cur = arena_load(A, (int32_t)i);
    if (cur == key) return (int32_t)i;
    if (cur == kEmptyKey) {
      cur = atomicCAS(A.keys + i, kEmptyKey, key);
      if (cur == kEmptyKey || cur == key) return (int32_t)i;
    }
    i = (i + 1) & A.mask;
  }
  atomicOr(A.err, kErrArena);
  return -1;
}

// ---------------------------------------------------------------------------
// Walker: a set of at most S stacks plus a pool of F walker-local frames.

template <int S, int F>
struct Walker {
  int32_t ref[S];
  int32_t node[S];
  int n;
  int32_t fpar[F];
  int32_t fnode[F];
  uint8_t fterm[F];
  int nf;
  uint32_t err;

  __device__ __forceinline__ void reset() { n = 0; nf = 0; err = 0; }

  __device__ __forceinline__ bool add(int32_t r, int32_t d) {
    for (int q = 0; q < n; ++q)
      if (ref[q] == r && node[q] == d) return true;
    if (n == S) { err |= kErrCap; return false; }
    ref[n] = r; node[n] = d; ++n;
    return true;
  }

  __device__ __forceinline__ uint32_t term_of(const DevArena& A, int32_t r) const {
    if (r == -1) return 1u;
    if (r >= 0) return fterm[r];
    return key_term(arena_load(A, -2 - r));
  }

  __device__ __forceinline__ void pop(const DevArena& A, int32_t r, int32_t& pr, int32_t& pn) const {
    if (r >= 0) { pr = fpar[r]; pn = fnode[r]; return; }
    const unsigned long long k = arena_load(A, -2 - r);
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
  __device__ __forceinline__ bool terminable(const DevGrammar& G, const DevArena& A, int32_t r, int32_t m) const {
    return (G.node_flags[m] & GM_NODE_POP) && term_of(A, r);
  }

  // One byte step of the whole set.  Sets *pop_bottom when some stack would
  // pop past an empty chain (REF cache.py:128-131 "popped" in synthetic
  // mode; at a real root this is the completed root and simply dies).
  template <int SN>
  __device__ int step(const DevGrammar& G, const DevArena& A, uint32_t b, bool* pop_bottom) {
    int32_t nr[SN], nn[SN];
    int cnt = 0;
    const int c = G.byte_class[b];
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
      }
    }
    for (int q = 0; q < cnt; ++q) { ref[q] = nr[q]; node[q] = nn[q]; }
    n = cnt;
    return cnt;
  }

  // Move every live stack's local frames into the arena (parents first) and
  // re-dedupe; afterwards all refs are -1 or arena refs.  Returns false on
  // arena exhaustion.
  __device__ bool intern_all(const DevArena& A) {
    if (nf == 0) return true;
    int32_t gmap[F];
    for (int q = 0; q < nf; ++q) gmap[q] = 0;  // 0 = unneeded, 1 = needed
    for (int s = 0; s < n; ++s) {
      int32_t r = ref[s];
      while (r >= 0 && gmap[r] == 0) { gmap[r] = 1; r = fpar[r]; }
    }
    for (int q = 0; q < nf; ++q) {  // frames are allocated parent-first
      if (!gmap[q]) { gmap[q] = -1; continue; }
      int32_t p = fpar[q];
      int32_t ph = p == -1 ? -1 : (p >= 0 ? gmap[p] : -2 - p);  // parent handle
      int32_t h = arena_intern(A, ph, fnode[q], fterm[q]);
      if (h < 0) { err |= kErrArena; return false; }
      gmap[q] = h;
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

// Matcher pool: ring of (window+1) top sets per slot (REF matcher.py:239-244
// history, 310-326 rollback).
struct DevPool {
  int32_t capacity, max_stacks, H;
  int2* tops;                 // [capacity][H][max_stacks] (handle, node)
  int32_t* meta;              // [capacity][H]: n_stacks | terminated << 16
  int32_t* head;              // [capacity]
  int32_t* hist_len;          // [capacity]
  int32_t* window;            // [capacity]
  const DevBinding** binding; // [capacity]
  DevArena arena;
  uint32_t* err;
  struct SlotHdr* hdr;        // [capacity] current-state summary
};

__device__ __forceinline__ int2* slot_tops(const DevPool& P, int32_t slot, int32_t h) {
  return P.tops + ((size_t)slot * P.H + h) * P.max_stacks;
}

// Current-state summary of a slot, one 256-byte record written by every
// state change (reset / accept / rollback / recycle / fork).  The fill kernel
// reads it with one coalesced load instead of chasing head -> ring entry ->
// key_of_node -> dep_off (each a cold HBM round trip once the model's forward
// pass has flushed L2).
constexpr int kHdrTops = 8;
struct __align__(16) SlotHdr {
  const DevBinding* binding;
  int32_t ntops;               // -1: more than kHdrTops stacks (fill uses the ring)
  int32_t flags;               // bit0 terminated, bit1 terminable
  int32_t key[kHdrTops];
  int32_t dep_lo[kHdrTops];
  int32_t dep_hi[kHdrTops];
  int2 top[kHdrTops];
  int32_t pad[20];
};
static_assert(sizeof(SlotHdr) == 256, "SlotHdr layout");

// Summarise (tops, terminated) of `slot` into its header.
__device__ inline void write_header(const DevPool& P, int32_t slot, const DevBinding* B, const int2* tops, int n,
                                    int terminated) {
  const DevGrammar& G = B->g;
  SlotHdr h;
  h.binding = B;
  int term = 0;
  for (int s = 0; s < n; ++s) {
    const int2 t = tops[s];
    if (!terminated && (G.node_flags[t.y] & GM_NODE_POP) &&
        (t.x < 0 || key_term(arena_load(P.arena, t.x))))
      term = 1;
    if (s < kHdrTops) {
      const int32_t k = G.key_of_node[t.y];
      h.key[s] = k;
      h.dep_lo[s] = k >= 0 ? B->c.dep_off[k] : 0;
      h.dep_hi[s] = k >= 0 ? B->c.dep_off[k + 1] : 0;
      h.top[s] = t;
    }
  }
  h.ntops = n <= kHdrTops ? n : -1;
  h.flags = (terminated ? 1 : 0) | (term ? 2 : 0);
  for (int i = 0; i < 20; ++i) h.pad[i] = 0;
  P.hdr[slot] = h;
}

}  // namespace gm
