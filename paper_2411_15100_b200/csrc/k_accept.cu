// K4 — batched accept_token / accept_bytes on device-resident stacks, plus
// the small state kernels (reset, recycle, rollback, probe, fork).
//
// Replaces Matcher.accept_token / accept_bytes / _sim_bytes / _rewrite_kernel
// / _push_history / rollback / branch (REF matcher.py:192-217, 239-355).
// One CTA (one warp) advances one request, with few dependent HBM round
// trips: slot header (1) -> token record with inline bytes, in parallel with
// staging the binding blob into shared memory (2) -> lane 0 walks the stack
// set byte by byte with walker-local frames (first pops served from the
// header's known arena keys) -> survivors are interned into the hash-consed
// arena with speculative parallel CAS (3) -> the next history-ring entry and
// the new header are written.  Dedupe by (handle, node) is dedupe by stack
// content because the arena is hash-consed (REF matcher.py:202-206).  A
// rejected token leaves the slot unchanged (REF matcher.py:267-268).
#include "accept.cuh"

namespace gm {

__global__ void __maxnreg__(128)
accept_tokens_kernel(DevPool P, const int32_t* __restrict__ slots, const int32_t* __restrict__ token_ids, int32_t n,
                     uint8_t* __restrict__ accepted) {
  extern __shared__ __align__(16) uint8_t tables[];
  __shared__ SlotHdr hd;
  __shared__ int4 s_rec[2];
  __shared__ RingPos rp;
  pdl_trigger();
  pdl_wait();
  const int32_t i = blockIdx.x;
  if (i >= n) return;
  trace_mark(P, 0, 0);
  const int32_t slot = __ldg(slots + i);
  const int32_t tid = __ldg(token_ids + i);
  load_header_ring(P, slot, &hd, &rp);
  __syncthreads();
  trace_mark(P, 0, 1);
  const bool in_range = tid >= 0 && tid < hd.V;
  if (threadIdx.x < 2 && in_range) s_rec[threadIdx.x] = __ldg(hd.tokrec + 2 * (size_t)tid + threadIdx.x);
  const DevGrammar G = stage_blob(hd.blob, hd.blob_bytes, tables);  // barrier inside
  trace_mark(P, 0, 2);
  if (threadIdx.x != 0) return;
  if (!in_range) {  // REF matcher.py:278-279
    slot_error(P, slot, kErrInvalid);
    accepted[i] = kAccErr;
    return;
  }
  const int4 e = s_rec[0], inl = s_rec[1];
  const uint8_t* far = reinterpret_cast<const uint8_t*>(hd.tokrec) + e.z;
  const int acc = accept_one(P, slot, rp, hd, G, e.y, [&](int64_t b) { return rec_byte(inl, far, (int)b); },
                             tid == hd.eos, e.x != 0, &hd);
  if (acc & kAccOk) store_header_state(P, slot, hd);  // accept_one leaves the mirror's publish to the caller
  accepted[i] = (uint8_t)acc;
}

__global__ void __maxnreg__(128)
accept_bytes_kernel(DevPool P, int32_t slot, const uint8_t* data, int64_t len, uint8_t* accepted) {
  extern __shared__ __align__(16) uint8_t tables[];
  __shared__ SlotHdr hd;
  __shared__ RingPos rp;
  load_header_ring(P, slot, &hd, &rp);
  __syncthreads();
  const DevGrammar G = stage_blob(hd.blob, hd.blob_bytes, tables);
  if (threadIdx.x != 0) return;
  if (hd.flags & 1) {
    slot_error(P, slot, kErrTerminated);
    *accepted = kAccErr;
    return;
  }
  if (len == 0) {  // REF matcher.py:253-258: empty input records a history entry
    const int2* tops;
    const int nt = view_tops(P, slot, hd, &tops);
    Chain c;
    build_chain(c, nt > 0 ? tops[0].x : -1, nullptr, nullptr, 0, hd);
    if (!push_tops(P, slot, rp, G, tops, nt, 0, c, nullptr)) {
      slot_error(P, slot, kErrCap);
      *accepted = kAccErr;
      return;
    }
    *accepted = kAccOk;
    return;
  }
  const int acc = accept_one(P, slot, rp, hd, G, len, [&](int64_t b) { return __ldg(data + b); }, false, false, &hd);
  if (acc & kAccOk) store_header_state(P, slot, hd);  // accept_one leaves the mirror's publish to the caller
  *accepted = (uint8_t)acc;
}

__global__ void reset_kernel(DevPool P, int32_t slot, const DevBinding* b, int32_t start, int32_t window) {
  if (threadIdx.x != 0) return;
  release_wide(P, slot);
  P.err[slot] = 0;
  P.binding[slot] = b;
  P.head[slot] = 0;
  P.hist_len[slot] = 0;
  P.window[slot] = window;
  int2* t = slot_tops(P, slot, 0);
  t[0] = make_int2(-1, start);
  P.meta[(size_t)slot * P.H] = 1;
  write_header(P, slot, b, t, 1, 0, 0);
}

// Request recycling for serving loops: a terminated slot restarts at the
// grammar's start state (fresh request, same grammar), others are untouched.
__global__ void recycle_kernel(DevPool P, const int32_t* __restrict__ slots, int32_t n) {
  pdl_trigger();
  pdl_wait();
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t slot = slots[i];
  if (!(P.hdr[slot].flags & 1)) return;
  const DevBinding* b = P.binding[slot];
  if (P.hdr[slot].wide_owned) release_wide(P, slot);
  P.head[slot] = 0;
  P.hist_len[slot] = 0;
  int2* t = slot_tops(P, slot, 0);
  t[0] = make_int2(-1, b->g.start_node);
  P.meta[(size_t)slot * P.H] = 1;
  write_header(P, slot, b, t, 1, 0, 0);
}

__global__ void rollback_kernel(DevPool P, const int32_t* __restrict__ slots, const int32_t* __restrict__ steps,
                                int32_t n) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t slot = slots[i], k = steps[i];
  const int32_t hl = P.hist_len[slot];
  if (k < 0 || k > hl) {  // REF matcher.py:313-314
    slot_error(P, slot, 1u << GM_ERR_ROLLBACK);
    return;
  }
  if (k == 0) return;
  const int32_t h = ((P.head[slot] - k) % P.H + P.H) % P.H;
  P.head[slot] = h;
  P.hist_len[slot] = hl - k;
  const int32_t meta = P.meta[(size_t)slot * P.H + h];
  write_header(P, slot, P.binding[slot], ring_tops(P, slot, h, meta & 0xFFFF), meta & 0xFFFF, (meta >> 16) & 1,
               P.hdr[slot].wide_owned);
}

// info: n_stacks, terminated, history_len, terminable, window; stacks copy;
// bytes8: union of acceptable first bytes over the closure (REF matcher.py:
// 219-237 _closed_facts).
__global__ void slot_probe_kernel(DevPool P, int32_t slot, int32_t* info, int2* stacks, int32_t max_out,
                                  uint32_t* bytes8) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const DevGrammar G = blob_view(P.binding[slot]->c.blob);
  const int32_t h = P.head[slot];
  const int32_t meta = P.meta[(size_t)slot * P.H + h];
  const int nt = meta & 0xFFFF;
  const int2* tops = ring_tops(P, slot, h, nt);
  int term = 0;
  uint32_t fb[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int s = 0; s < nt; ++s) {
    int32_t hh = tops[s].x, m = tops[s].y;
    if (s < max_out) stacks[s] = tops[s];
    while (true) {  // every node reachable by silent completion
      for (int b = 0; b < 256; ++b) {
        const int32_t idx = m * G.n_classes + G.byte_class[b];
        if (G.trans_off[idx + 1] > G.trans_off[idx]) fb[b >> 5] |= 1u << (b & 31);
      }
      if (!(G.node_flags[m] & GM_NODE_POP)) break;
      if (hh < 0) { term = 1; break; }
      const unsigned long long k = arena_load(P.arena, hh);
      hh = key_parent(k);
      m = key_node(k);
    }
  }
  info[0] = nt;
  info[1] = (meta >> 16) & 1;
  info[2] = P.hist_len[slot];
  info[3] = term && !((meta >> 16) & 1);
  info[4] = P.window[slot];
  for (int i = 0; i < 8; ++i) bytes8[i] = fb[i];
}

// branch / fork (REF matcher.py:328-355): copy the whole slot state (wide
// ring entries get blocks of their own).
__global__ void fork_kernel(DevPool P, int32_t src, int32_t dst) {
  __shared__ int2* s_dst;
  release_wide(P, dst, threadIdx.x, blockDim.x);
  if (threadIdx.x == 0) P.err[dst] = 0;
  __syncthreads();
  const size_t per = (size_t)P.H * P.max_stacks;
  for (size_t k = threadIdx.x; k < per; k += blockDim.x) P.tops[dst * per + k] = P.tops[src * per + k];
  for (int k = threadIdx.x; k < P.H; k += blockDim.x) P.meta[(size_t)dst * P.H + k] = P.meta[(size_t)src * P.H + k];
  for (int h = 0; h < P.H; ++h) {
    const int n = P.meta[(size_t)src * P.H + h] & 0xFFFF;
    if (n <= P.max_stacks) continue;
    if (threadIdx.x == 0) {
      s_dst = ring_tops_w(P, dst, h, n);
      if (!s_dst) {
        slot_error(P, dst, kErrCap);
        P.meta[(size_t)dst * P.H + h] = 0;
      }
    }
    __syncthreads();
    const int2* from = ring_tops(P, src, h, n);
    if (s_dst)
      for (int k = threadIdx.x; k < n; k += blockDim.x) s_dst[k] = from[k];
    __syncthreads();
  }
  if (threadIdx.x < kHdrVec)
    reinterpret_cast<int4*>(P.hdr + dst)[threadIdx.x] = reinterpret_cast<const int4*>(P.hdr + src)[threadIdx.x];
  if (threadIdx.x == 0) {
    P.head[dst] = P.head[src];
    P.hist_len[dst] = P.hist_len[src];
    P.window[dst] = P.window[src];
    P.binding[dst] = P.binding[src];
  }
}

// ---------------------------------------------------------------------------
// Arena collection (REF pstack.py:85-111 reclaims frames by refcount; here a
// mark / sweep over the live slots' histories, run between steps).
//   mark:    every frame reachable from a top of a live slot's history ring
//            entries (the rollback window, REF matcher.py:239-244, 310-326)
//   sweep:   unmarked frames -> tombstones
//   need:    every slot between a live key's home and its position
//   compact: tombstones no live key's probe chain crosses -> empty
// Handles are slots and never move, so nothing else is rewritten.
__global__ void gc_mark_kernel(DevPool P, const int32_t* __restrict__ live, int32_t n, uint32_t* __restrict__ mark) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)n * P.H) return;
  const int32_t slot = live[t / P.H];
  const int32_t k = (int32_t)(t % P.H);
  if (slot < 0 || slot >= P.capacity || k > P.hist_len[slot]) return;
  const int32_t h = ((P.head[slot] - k) % P.H + P.H) % P.H;
  const int nt = P.meta[(size_t)slot * P.H + h] & 0xFFFF;
  const int2* tops = ring_tops(P, slot, h, nt);
  for (int s = 0; s < nt; ++s) {
    int32_t hh = tops[s].x;
    while (hh >= 0 && (uint32_t)hh <= P.arena.mask) {
      const uint32_t bit = 1u << (hh & 31);
      if (atomicOr(mark + (hh >> 5), bit) & bit) break;  // this frame's ancestors are marked already
      const unsigned long long key = P.arena.keys[hh];
      if (key >= kTombKey) break;
      hh = key_parent(key);
    }
  }
}

__global__ void gc_sweep_kernel(DevArena A, const uint32_t* __restrict__ mark) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > A.mask) return;
  const unsigned long long key = A.keys[i];
  if (key < kTombKey && !(mark[i >> 5] & (1u << (i & 31)))) A.keys[i] = kTombKey;
}

__global__ void gc_need_kernel(DevArena A, uint32_t* __restrict__ need) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > A.mask) return;
  const unsigned long long key = A.keys[i];
  if (key >= kTombKey) return;
  for (uint32_t q = mix64(key) & A.mask; q != i; q = (q + 1) & A.mask) atomicOr(need + (q >> 5), 1u << (q & 31));
}

__global__ void gc_compact_kernel(DevArena A, const uint32_t* __restrict__ need) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > A.mask) return;
  if (A.keys[i] == kTombKey && !(need[i >> 5] & (1u << (i & 31)))) A.keys[i] = kEmptyKey;
}

// live frames / tombstones
__global__ void arena_count_kernel(DevArena A, unsigned long long* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long live = 0, tomb = 0;
  if (i <= A.mask) {
    const unsigned long long key = A.keys[i];
    live = key < kTombKey;
    tomb = key == kTombKey;
  }
  live = __reduce_add_sync(0xFFFFFFFFu, (unsigned)live);
  tomb = __reduce_add_sync(0xFFFFFFFFu, (unsigned)tomb);
  if ((threadIdx.x & 31) == 0) {
    if (live) atomicAdd(out, live);
    if (tomb) atomicAdd(out + 1, tomb);
  }
}

gm_status launch_collect(const DevPool& P, const int32_t* live, int32_t n, uint32_t* mark, uint32_t* need,
                         cudaStream_t s) {
  const size_t words = ((size_t)P.arena.mask + 1) / 32;
  const unsigned blocks = (unsigned)ceil_div((int64_t)P.arena.mask + 1, 256);
  GM_CUDA_TRY(cudaMemsetAsync(mark, 0, words * 4, s));
  GM_CUDA_TRY(cudaMemsetAsync(need, 0, words * 4, s));
  if (n > 0) {
    gc_mark_kernel<<<(unsigned)ceil_div((int64_t)n * P.H, 128), 128, 0, s>>>(P, live, n, mark);
    GM_LAUNCH_CHECK();
  }
  gc_sweep_kernel<<<blocks, 256, 0, s>>>(P.arena, mark);
  GM_LAUNCH_CHECK();
  gc_need_kernel<<<blocks, 256, 0, s>>>(P.arena, need);
  GM_LAUNCH_CHECK();
  gc_compact_kernel<<<blocks, 256, 0, s>>>(P.arena, need);
  GM_LAUNCH_CHECK();
  return GM_OK;
}

gm_status launch_arena_count(const DevArena& A, unsigned long long* out, cudaStream_t s) {
  GM_CUDA_TRY(cudaMemsetAsync(out, 0, 16, s));
  arena_count_kernel<<<(unsigned)ceil_div((int64_t)A.mask + 1, 256), 256, 0, s>>>(A, out);
  GM_LAUNCH_CHECK();
  return GM_OK;
}

// Per-slot error words of `slots` (gathered; cleared with `clear`).
__global__ void pool_errors_kernel(DevPool P, const int32_t* __restrict__ slots, int32_t n, uint32_t* __restrict__ out,
                                   int32_t clear) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t slot = slots[i];
  if (slot < 0 || slot >= P.capacity) {
    out[i] = kErrInvalid;
    return;
  }
  out[i] = clear ? atomicExch(P.err + slot, 0u) : P.err[slot];
}

static gm_status set_smem_attr(const void* fn) {
  GM_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kStageBytes));
  // keep most of the unified L1/shared array as L1: the walker's per-thread
  // state lives in local memory and must hit L1, not L2
  GM_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 25));
  return GM_OK;
}

gm_status launch_accept_tokens(const DevPool& P, const int32_t* slots, const int32_t* toks, int32_t n, uint8_t* acc,
                               cudaStream_t s) {
  if (n <= 0) return GM_OK;
  static gm_status once = set_smem_attr(reinterpret_cast<const void*>(accept_tokens_kernel));
  if (once) return once;
  const L2Window win{P.l2_base, P.l2_bytes, P.l2_hit};
  GM_CUDA_TRY(launch_pdl_w(&win, accept_tokens_kernel, dim3(n), dim3(kAccThreads), kStageBytes, s, P, slots, toks, n,
                           acc));
  return GM_OK;
}
gm_status launch_accept_bytes(const DevPool& P, int32_t slot, const uint8_t* data, int64_t len, uint8_t* acc,
                              cudaStream_t s) {
  static gm_status once = set_smem_attr(reinterpret_cast<const void*>(accept_bytes_kernel));
  if (once) return once;
  accept_bytes_kernel<<<1, kAccThreads, kStageBytes, s>>>(P, slot, data, len, acc);
  GM_LAUNCH_CHECK();
  return GM_OK;
}
gm_status launch_reset(const DevPool& P, int32_t slot, const DevBinding* b, int32_t start, int32_t window,
                       cudaStream_t s) {
  reset_kernel<<<1, 32, 0, s>>>(P, slot, b, start, window);
  GM_LAUNCH_CHECK();
  return GM_OK;
}
gm_status launch_recycle(const DevPool& P, const int32_t* slots, int32_t n, cudaStream_t s) {
  if (n <= 0) return GM_OK;
  GM_CUDA_TRY(launch_pdl(recycle_kernel, dim3((unsigned)ceil_div(n, 128)), dim3(128), 0, s, P, slots, n));
  return GM_OK;
}
gm_status launch_rollback(const DevPool& P, const int32_t* slots, const int32_t* steps, int32_t n, cudaStream_t s) {
  if (n <= 0) return GM_OK;
  rollback_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, s>>>(P, slots, steps, n);
  GM_LAUNCH_CHECK();
  return GM_OK;
}
gm_status launch_probe(const DevPool& P, int32_t slot, int32_t* info, int2* stacks, int32_t max_out,
                       uint32_t* bytes8, cudaStream_t s) {
  slot_probe_kernel<<<1, 32, 0, s>>>(P, slot, info, stacks, max_out, bytes8);
  GM_LAUNCH_CHECK();
  return GM_OK;
}
gm_status launch_pool_errors(const DevPool& P, const int32_t* slots, int32_t n, uint32_t* out, int32_t clear,
                             cudaStream_t s) {
  if (n <= 0) return GM_OK;
  pool_errors_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, s>>>(P, slots, n, out, clear);
  GM_LAUNCH_CHECK();
  return GM_OK;
}
gm_status launch_fork(const DevPool& P, int32_t src, int32_t dst, cudaStream_t s) {
  fork_kernel<<<1, 256, 0, s>>>(P, src, dst);
  GM_LAUNCH_CHECK();
  return GM_OK;
}

}  // namespace gm
