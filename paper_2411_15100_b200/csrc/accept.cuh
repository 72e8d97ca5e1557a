// Device-side accept machinery shared by K4 (k_accept.cu) and the fused
// step kernel (k_fill.cu): advance one request's stack set by a token's
// bytes, intern the survivors, append the history ring entry and publish
// the new slot header.  REF matcher.py:192-217, 239-294.
//
// Walk tiers: RWalker (<= kAccR stacks in registers) -> Walker (<= kAccS
// stacks, local frames) -> BigWalk (<= kWideCap = 4096 stacks in global
// scratch, the reference's branch cap).  A walk is redone on the next tier
// whenever it exceeds a cap, so the result never depends on the tier; only
// exceeding 4096 stacks is an error (GM_ERR_STATE_CAP, REF matcher.py:
// 188-189).
#pragma once
#include "device.cuh"

namespace gm {

constexpr int kAccS = 32;
constexpr int kAccF = 160;
constexpr int kAccThreads = 32;
#ifndef GM_ACC_R
#define GM_ACC_R 2
#endif
constexpr int kAccR = GM_ACC_R;  // stacks held in registers by the fast walker
#ifndef GM_ACC_RF
#define GM_ACC_RF 48
#endif
constexpr int kAccRF = GM_ACC_RF;  // its walker-local frames

// accept_one results: bit 0 = accepted, bit 1 = error (the slot's error
// word says which; the state is unchanged)
constexpr int kAccOk = 1, kAccErr = 2;
#ifndef GM_ACC_MICRO
#define GM_ACC_MICRO 0  // measured: K5 b2b +0.8 us (code layout), cold -1.8 us
#endif

// Current (handle, node) set of a slot: from the header when it fits, else
// from the ring (inline entry or its wide block).  Returns the count; *out
// points at the stacks (shared header or global ring).
__device__ inline int view_tops(const DevPool& P, int32_t slot, const SlotHdr& hdr, const int2** out) {
  if (hdr.ntops >= 0) {
    *out = hdr.top;
    return hdr.ntops;
  }
  const int32_t h = P.head[slot];
  const int n = P.meta[(size_t)slot * P.H + h] & 0xFFFF;
  *out = ring_tops(P, slot, h, n);
  return n;
}

// Ancestor chain of handle h read from the arena (first kChain frames).
__device__ inline void chain_from_arena(const DevPool& P, int32_t h, Chain& c) {
  c.n = 0;
  while (h >= 0 && c.n < kChain) {
    const unsigned long long k = arena_load(P.arena, h);
    if (k >= kTombKey) break;
    c.h[c.n] = h;
    c.k[c.n] = k;
    ++c.n;
    h = key_parent(k);
  }
}

// Ring position of a slot (head, history length, window).
struct RingPos {
  int32_t head, hist_len, window;
};

// Slot header + ring position in ONE round trip: every load is issued before
// any shared-memory store (a store waiting on its load would otherwise hold
// back the loads behind it — measured: four serial trips).
__device__ __forceinline__ void load_header_ring(const DevPool& P, int32_t slot, SlotHdr* s_hdr, RingPos* rp) {
  const int t = threadIdx.x;
  int4 v = make_int4(0, 0, 0, 0);
  int32_t x = 0;
  if (t < kHdrVec) v = __ldcg(reinterpret_cast<const int4*>(P.hdr + slot) + t);
  if (t == 1) x = __ldcg(P.head + slot);
  else if (t == 2) x = __ldcg(P.hist_len + slot);
  else if (t == 3) x = __ldcg(P.window + slot);
  if (t < kHdrVec) reinterpret_cast<int4*>(s_hdr)[t] = v;
  if (t == 1) rp->head = x;
  else if (t == 2) rp->hist_len = x;
  else if (t == 3) rp->window = x;
}

// Append (handle, node) tops as the next ring entry and publish the new
// header state.  The binding pointers of the global header are unchanged, so
// only its state fields are rewritten in place.  False when the set cannot
// be stored (more than kWideCap stacks, or no wide block free).
__device__ inline bool push_tops(const DevPool& P, int32_t slot, const RingPos& rp, const DevGrammar& G,
                                 const int2* tops, int nt, int terminated, const Chain& c, SlotHdr* mirror) {
  const int32_t nh = (rp.head + 1) % P.H;
  int2* dst = ring_tops_w(P, slot, nh, nt);
  if (!dst) return false;
  if (nt > P.max_stacks) (mirror ? mirror : &P.hdr[slot])->wide_owned = 1;
  if (dst != tops)
    for (int s = 0; s < nt; ++s) dst[s] = tops[s];
  P.meta[(size_t)slot * P.H + nh] = nt | (terminated << 16);
  P.head[slot] = nh;
  const int32_t hl = rp.hist_len + 1;
  P.hist_len[slot] = hl < rp.window ? hl : rp.window;
  if (mirror) {  // new state into the caller's shared copy; the caller publishes it
    header_state(P, *mirror, G, dst, nt, terminated, &c);
  } else {
    header_state(P, P.hdr[slot], G, dst, nt, terminated, &c);
  }
  return true;
}

// Restart a slot at the grammar's start state (recycle_kernel semantics)
// from inside a step kernel: ring entry 0, empty history, header state.
__device__ inline void restart_slot(const DevPool& P, int32_t slot, const DevGrammar& G, SlotHdr* mirror) {
  if (mirror->wide_owned) {
    release_wide(P, slot);
    mirror->wide_owned = 0;
  }
  P.head[slot] = 0;
  P.hist_len[slot] = 0;
  const int2 t0 = make_int2(-1, G.start_node);
  *slot_tops(P, slot, 0) = t0;
  P.meta[(size_t)slot * P.H] = 1;
  header_state(P, *mirror, G, &t0, 1, 0, nullptr);  // the caller publishes it
}

__device__ inline bool push_history(const DevPool& P, int32_t slot, const RingPos& rp, const SlotHdr& hdr,
                                    const DevGrammar& G, int nt, const int32_t* refs, const int32_t* nodes,
                                    int terminated, const int32_t* fh, const unsigned long long* fk, int nfresh,
                                    SlotHdr* mirror = nullptr) {
  int2 loc[kAccS];
  for (int s = 0; s < nt; ++s) {
    const int32_t r = refs[s];
    loc[s] = make_int2(r == -1 ? -1 : -2 - r, nodes[s]);
  }
  Chain c;
  build_chain(c, nt > 0 ? loc[0].x : -1, fh, fk, nfresh, hdr);
  return push_tops(P, slot, rp, G, loc, nt, terminated, c, mirror);
}

// The overflow tier: walk `len` bytes from `tops` in global scratch.  The
// surviving set is written as the next ring entry.  Returns accept_one's
// result code.
template <class ByteFn>
#ifdef GM_ACC_WIDE_NOINLINE
__device__ __noinline__ int accept_wide(
#else
__device__ inline int accept_wide(
#endif
    const DevPool& P, int32_t slot, const RingPos& rp, const DevGrammar& G,
                                  const int2* tops, int ntops, int64_t len, ByteFn byte, SlotHdr* mirror) {
#ifdef GM_DIAG_NO_DEP_BIGWALK  // diagnostics: code-size experiment (wide sets then fail)
  slot_error(P, slot, kErrCap);
  return kAccErr;
#endif
  BigWalk bw;
  bw.acquire(P.ovf, (uint32_t)slot);
  bw.start();
  for (int s = 0; s < ntops; ++s) bw.add(tops[s].x, tops[s].y);
  for (int64_t i = 0; i < len && bw.n > 0 && !bw.err; ++i) {
    bool pb = false;
    bw.step(G, P.arena, byte(i), &pb);
  }
  int res = 0;
  if (bw.err) {
    slot_error(P, slot, bw.err);
    res = kAccErr;
  } else if (bw.n > 0) {
    Chain c;
    chain_from_arena(P, bw.cur[0].x, c);
    if (push_tops(P, slot, rp, G, bw.cur, bw.n, 0, c, mirror)) {
      res = kAccOk;
    } else {
      slot_error(P, slot, kErrCap);
      res = kAccErr;
    }
  }
  bw.release();
  return res;
}

// Shared by token and byte-string acceptance (one thread).  byte(i) gives
// the i-th input byte; is_eos = EOS token.  Returns kAccOk if accepted, 0 if
// rejected (state unchanged), kAccErr on an error (recorded in the slot's
// error word; state unchanged).  With `mirror` (== &hdr, the caller's shared
// header) the new state is written there and the ring updated, but the
// caller publishes the header (warp-parallel, store_header_state_warp) so a
// fused step kernel can fill from it.
struct NoWalkHook {
  template <class W>
  __device__ __forceinline__ void operator()(const W&) const {}
};

// `on_walk(rw)` runs after a successful register-walker walk, before the
// survivors are interned and published: the fused step kernel uses it to
// start fetching the new tops' cache rows while the commit runs.
template <class ByteFn, class OnWalk = NoWalkHook>
__device__ inline int accept_one(const DevPool& P, int32_t slot, const RingPos& rp, const SlotHdr& hdr,
                                 const DevGrammar& G, int64_t len, ByteFn byte, bool is_eos, bool reject_token,
                                 SlotHdr* mirror = nullptr, OnWalk on_walk = OnWalk(), unsigned long long* ts = nullptr,
                                 SpecOut* spec = nullptr) {
  if (hdr.flags & 1) {  // REF matcher.py:276-277 "matcher is terminated"
    slot_error(P, slot, kErrTerminated);
    return kAccErr;
  }
  const int2* tops;
  const int ntops = view_tops(P, slot, hdr, &tops);
  if (is_eos) {  // REF matcher.py:280-288
    if (!(hdr.flags & 2)) return 0;
    Chain c;
    build_chain(c, ntops > 0 ? tops[0].x : -1, nullptr, nullptr, 0, hdr);
    if (!push_tops(P, slot, rp, G, tops, ntops, 1, c, mirror)) {
      slot_error(P, slot, kErrCap);
      return kAccErr;
    }
    return kAccOk;
  }
  if (reject_token) return 0;  // special or empty token (REF matcher.py:289-293)
  if (__builtin_expect(ntops > kAccS, 0)) return accept_wide(P, slot, rp, G, tops, ntops, len, byte, mirror);
  // micro path: one stack, every byte a plain table move inside its frame
  // (no push, no pop, no dead end: the fast table's -1 / >= 0 entries and,
  // above the bottom frame, the pop-filtered ones) — the chain is
  // unchanged, so the commit is the new top node.  Same result as the
  // walkers (their n == 1 step takes exactly these entries first); a few
  // dozen instructions instead of the walker + commit code.
  if (GM_ACC_MICRO && ntops == 1 && mirror) {
    int32_t node = tops[0].y;
    const bool above = tops[0].x >= 0;
    int64_t i = 0;
    for (; i < len; ++i) {
      const int32_t f = G.fast[node * G.n_classes + G.byte_class[byte(i)]];
      if (f >= 0) {
        node = f;
      } else if (f == -1 || (above && f == kFastPopDies)) {
        return 0;  // the only stack dies: rejected, state unchanged
      } else if (above && f < -2) {
        node = -3 - f;
      } else {
        break;  // a push / pop / several targets: the walkers below
      }
    }
    if (i == len) {
      const int2 t = make_int2(tops[0].x, node);
      const int32_t nh = (rp.head + 1) % P.H;
      *slot_tops(P, slot, nh) = t;
      P.meta[(size_t)slot * P.H + nh] = 1;
      P.head[slot] = nh;
      const int32_t hl = rp.hist_len + 1;
      P.hist_len[slot] = hl < rp.window ? hl : rp.window;
      SlotHdr& h = *mirror;
      int term = 0;
      if (G.node_flags[node] & GM_NODE_POP)
        term = t.x < 0 ? 1 : (int)key_term((h.nchain && h.chain_h[0] == t.x) ? h.chain_k[0] : arena_load(P.arena, t.x));
      const int4 ni = G.node_info[node];
      h.key[0] = ni.x;
      h.dep_lo[0] = ni.y;
      h.dep_hi[0] = ni.z;
      h.top[0] = t;
      h.ntops = 1;
      h.flags = (term ? 2 : 0) | ((ni.w >> 28) & 4);  // 4: the fused apply blends this key's row
      if (spec) spec->n = 0;
      return kAccOk;
    }
  }
  // fast path: register walker (<= kAccR stacks)
  if (ntops <= kAccR) {
    RWalker<kAccR, kAccRF> rw;
    rw.init(hdr.chain_h, hdr.chain_k, hdr.nchain);
    for (int s = 0; s < ntops; ++s) rw.add(rw.ref_of_handle(tops[s].x), tops[s].y);
    for (int64_t i = 0; i < len && rw.n > 0 && !rw.spill; ++i) {
      bool pb = false;
      rw.template step<true>(G, P.arena, byte(i), &pb);
    }
    trace_mark(P, 0, 3);
    if (__builtin_expect(!rw.spill, 1)) {
      if (rw.err) {
        slot_error(P, slot, rw.err);
        return kAccErr;
      }
      if (rw.n == 0) return 0;
      on_walk(rw);
      int2 out[kAccR];
      if (mirror) {  // fused step kernel: chain rewritten in place in the shared header
        if (ts) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts[2]));
        const int nout = rwalker_commit_inplace(rw, P.arena, out, *mirror, spec);
        if (nout < 0) {
          slot_error(P, slot, kErrArena);
          return kAccErr;
        }
        if (ts) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts[0]));
        const int32_t nh = (rp.head + 1) % P.H;
        int2* dst = slot_tops(P, slot, nh);
        for (int s = 0; s < nout; ++s) dst[s] = out[s];
        P.meta[(size_t)slot * P.H + nh] = nout;
        P.head[slot] = nh;
        const int32_t hl = rp.hist_len + 1;
        P.hist_len[slot] = hl < rp.window ? hl : rp.window;
        if (ts) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts[3]));
        header_state_inplace(P, *mirror, G, out, nout, 0);
        if (ts) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts[1]));
        return kAccOk;
      }
      Chain c;
      const int nout = rwalker_commit(rw, P.arena, out, c);
      if (nout < 0) {
        slot_error(P, slot, kErrArena);
        return kAccErr;
      }
      trace_mark(P, 0, 4);
      if (ts) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts[0]));
      push_tops(P, slot, rp, G, out, nout, 0, c, mirror);  // <= kAccR stacks: always inline
      if (ts) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts[1]));
      trace_mark(P, 0, 5);
      return kAccOk;
    }
  }
#ifdef GM_DIAG_NO_GENERAL  // diagnostics: code-size experiment (multi-stack requests then fail)
  slot_error(P, slot, kErrCap);
  return kAccErr;
#endif
  // general path: up to kAccS stacks, local frames
  Walker<kAccS, kAccF> w;
  w.reset();
  w.external(hdr.chain_h, hdr.chain_k, hdr.nchain);
  for (int s = 0; s < ntops; ++s) w.add(tops[s].x < 0 ? -1 : -2 - tops[s].x, tops[s].y);
  for (int64_t i = 0; i < len; ++i) {
    if (w.nf > kAccF / 2) {
      if (!w.intern_all(P.arena)) break;
    }
    bool pb = false;
    if (!w.template step<kAccS>(G, P.arena, byte(i), &pb)) break;
  }
  trace_mark(P, 0, 3);
  if (__builtin_expect(w.err & kErrCap, 0)) return accept_wide(P, slot, rp, G, tops, ntops, len, byte, mirror);
  if (w.err) {
    slot_error(P, slot, w.err);
    return kAccErr;
  }
  if (w.n == 0) return 0;
  if (!w.intern_all(P.arena)) {
    slot_error(P, slot, w.err | kErrArena);
    return kAccErr;
  }
  trace_mark(P, 0, 4);
  if (!push_history(P, slot, rp, hdr, G, w.n, w.ref, w.node, 0, w.kh, w.kk, w.nk, mirror)) {
    slot_error(P, slot, kErrCap);
    return kAccErr;
  }
  trace_mark(P, 0, 5);
  return kAccOk;
}

}  // namespace gm
