"""CUDA-graph capture of the per-decode-step grammar work.

A serving loop advances a fixed batch of matchers once per generated token:
hand the sampled token ids to the device, accept them, restart finished
requests, fill the next masks and apply them to the logits buffer, and hand
the accepted flags back.  With static buffers every one of those operations
has fixed arguments, so the whole step is captured once into a CUDA graph
and replayed with a single launch — the host cost per step drops from the
Python/ctypes path (~20 µs) to one graph launch, and the device sees one
dependency chain with no gaps.

    step = DecodeStepGraph(matchers, bitmask, logits_buffers)
    accepted = step.run(host_token_ids, buffer_index)   # pinned uint8 [B]

With one buffer per in-flight step (``len(logits_buffers)``), steps queue
back to back (``wait=False``) without host syncs.
"""

from __future__ import annotations

from typing import Optional, Sequence

import numpy as np
import torch

from .matcher import GrammarMatcher, batch_step
from .engine import get_pool


class DecodeStepGraph:
    """One captured graph per logits buffer: H2D token ids -> K5 step
    (accept + recycle + fill + apply) -> D2H accepted flags.

    ``logits`` is a list of static [B, V] buffers (e.g. the engine's
    double-buffered LM-head outputs); ``run(tokens, i)`` replays the graph of
    buffer i.  ``first(i)`` fills + applies without an accept (first step).
    Bit-identical to the eager calls (same kernels, same arguments)."""

    def __init__(self, matchers: Sequence[GrammarMatcher], bitmask: Optional[torch.Tensor],
                 logits: Sequence[torch.Tensor], recycle: bool = True, stream: Optional[torch.cuda.Stream] = None,
                 zero_copy: bool = False):
        pool = get_pool()
        dev = pool.device
        B = len(matchers)
        self.B = B
        # the graph replays raw slot ids: keep the matchers (and so their
        # slots) alive for the graph's lifetime
        self._matchers = list(matchers)
        self.slots = torch.tensor([m.slot for m in matchers], dtype=torch.int32, device=dev)
        n = len(logits)
        # per logits buffer: its own pinned staging (token ids in, accepted
        # flags out) and device buffers, so step s+1 can be queued while step
        # s is still in flight; an event per buffer guards the reuse of its
        # staging n steps later
        self.tokens_host = [torch.zeros(B, dtype=torch.int32).pin_memory() for _ in range(n)]
        self.accepted_host = [torch.zeros(B, dtype=torch.uint8).pin_memory() for _ in range(n)]
        self.tokens = [torch.zeros(B, dtype=torch.int32, device=dev) for _ in range(n)]
        self.accepted = [torch.zeros(B, dtype=torch.uint8, device=dev) for _ in range(n)]
        self.done = [torch.cuda.Event() for _ in range(n)]
        self._tok_np = [t.numpy() for t in self.tokens_host]  # host writes without a torch op
        # one bitmask for all steps, or one per logits buffer
        self.bitmasks = list(bitmask) if isinstance(bitmask, (list, tuple)) else [bitmask] * n
        self.bitmask = self.bitmasks[0]
        self.logits = list(logits)
        self.recycle = recycle
        self.stream = stream or torch.cuda.Stream(device=dev)
        # warm up outside capture (one-time kernel attribute setup): a
        # fill-only step into scratch buffers leaves the matchers unchanged
        with torch.cuda.stream(self.stream):
            scratch_mask = torch.empty_like(self.bitmask) if self.bitmask is not None else None
            scratch_logits = torch.empty((B, 8), dtype=self.logits[0].dtype, device=dev)
            batch_step(pool, self.slots, None, None, scratch_mask, scratch_logits, stream=self.stream)
        self.stream.synchronize()
        # default: H2D copy -> K5 -> D2H copy.  zero_copy: the step kernel
        # reads the token ids straight from the pinned host buffer (volatile
        # loads over PCIe, unified addressing) and writes the accepted flags
        # straight into pinned host memory — one launch, no copy engine, but
        # measured ~10x slower per step on the B200 box (356 vs 38 us: each
        # CTA's host access is a serialized PCIe round trip), so off.
        self.zero_copy = zero_copy
        self.graphs = []
        for i, buf in enumerate(self.logits):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.stream):
                if zero_copy:
                    batch_step(pool, self.slots, self.tokens_host[i], self.accepted_host[i], self.bitmasks[i], buf,
                               recycle=recycle, stream=self.stream)
                else:
                    self.tokens[i].copy_(self.tokens_host[i], non_blocking=True)
                    batch_step(pool, self.slots, self.tokens[i], self.accepted[i], self.bitmasks[i], buf,
                               recycle=recycle, stream=self.stream)
                    self.accepted_host[i].copy_(self.accepted[i], non_blocking=True)
            self.graphs.append(g)

    def first(self, i: int = 0) -> None:
        """First step of a batch: fill + apply only (no token to accept)."""
        with torch.cuda.stream(self.stream):
            batch_step(get_pool(), self.slots, None, None, self.bitmasks[i], self.logits[i], stream=self.stream)

    def run(self, tokens, i: int = 0, wait: bool = True) -> torch.Tensor:
        """Accept ``tokens`` (host ints), fill + apply into logits buffer i.
        Returns buffer i's pinned accepted flags (valid once the stream has
        passed this step: ``wait`` syncs before returning, else
        ``self.done[i]``).  Steps may be queued back to back: buffer i's
        staging is reused only after its previous replay has completed."""
        self.done[i].synchronize()
        if isinstance(tokens, torch.Tensor):
            tokens = tokens.numpy() if tokens.device.type == "cpu" else tokens.cpu().numpy()
        np.copyto(self._tok_np[i], np.asarray(tokens), casting="unsafe")
        with torch.cuda.stream(self.stream):  # replay() launches on the current stream
            self.graphs[i].replay()
            self.done[i].record(self.stream)
        if wait:
            self.stream.synchronize()
            flags = self.accepted_host[i].numpy()
            if (flags & 2).any():  # bit 1: that request's step failed
                get_pool().raise_slot_errors(self.slots, flags)
        return self.accepted_host[i]


class DecodeLoop:
    """Native decode loop (C-ABI gm_decoder_*): per step the library copies
    the host token ids into pinned staging, issues the H2D copy on its own
    copy stream, K5 (accept + recycle + fill + apply) on ``stream`` and the
    D2H copy of the accepted flags, ordered by events — no Python on the
    per-step path beyond one ctypes call, and the copies of neighbouring
    steps overlap the kernels.  ``len(logits)`` steps may be in flight.

        loop = DecodeLoop(matchers, bitmasks, logits_buffers)
        loop.step(None, 0)                 # first step: fill + apply
        loop.step(host_token_ids, i)       # later steps (int32 numpy / list)
        flags = loop.flags(i)              # uint8 [B], waits for step i
    """

    def __init__(self, matchers: Sequence[GrammarMatcher], bitmask, logits: Sequence[torch.Tensor],
                 recycle: bool = True, stream: Optional[torch.cuda.Stream] = None, collect_every: int = 0,
                 collect_threshold: float = 0.5):
        """``collect_every`` > 0: every that many steps, reclaim arena frames
        no live matcher references once the arena is more than
        ``collect_threshold`` full (MatcherPool.maybe_collect; syncs)."""
        import ctypes as C

        from . import _lib
        from .bitmask import _DTYPES

        pool = get_pool()
        dev = pool.device
        n_buf = len(logits)
        self.B = len(matchers)
        # the native decoder steps raw slot ids: keep the matchers (and so
        # their slots) alive until close()
        self._matchers = list(matchers)
        self._pool = pool
        self.slots = torch.tensor([m.slot for m in matchers], dtype=torch.int32, device=dev)
        self.bitmasks = list(bitmask) if isinstance(bitmask, (list, tuple)) else [bitmask] * n_buf
        self.logits = list(logits)
        lg0 = self.logits[0]
        for lg in self.logits:
            if lg.dtype not in _DTYPES or lg.dim() != 2 or lg.stride(-1) != 1 or lg.shape != lg0.shape:
                raise ValueError("logits buffers must be equal-shape 2-D fp32/fp16/bf16 CUDA tensors")
        self.stream = stream or torch.cuda.current_stream(dev)
        bm_ptrs = (C.c_void_p * n_buf)(*[b.data_ptr() if b is not None else None for b in self.bitmasks])
        lg_ptrs = (C.c_void_p * n_buf)(*[lg.data_ptr() for lg in self.logits])
        bstride = self.bitmasks[0].stride(0) if self.bitmasks[0] is not None else 0
        h = C.c_void_p()
        lib = _lib.load()
        _lib.check(lib.gm_decoder_create(pool.handle, self.slots.data_ptr(), self.B, n_buf,
                                         bm_ptrs if self.bitmasks[0] is not None else None, bstride, lg_ptrs,
                                         _DTYPES[lg0.dtype], lg0.shape[1], lg0.stride(0), 1 if recycle else 0,
                                         C.byref(h)), "gm_decoder_create")
        self._h = h
        self._lib = lib
        self._check = _lib.check
        self._sptr = int(self.stream.cuda_stream)
        self._tok = np.zeros(self.B, dtype=np.int32)
        self._flags = np.zeros(self.B, dtype=np.uint8)
        self.collect_every = collect_every
        self.collect_threshold = collect_threshold
        self._steps = 0
        self.collections = 0

    def step(self, tokens, i: int = 0) -> None:
        """Issue one decode step on buffer i (tokens: host ints, or None for
        the first step).  Blocks only if buffer i's previous step is still
        in flight."""
        if tokens is None:
            ptr = None
        else:
            t = tokens if isinstance(tokens, np.ndarray) and tokens.dtype == np.int32 else np.asarray(tokens, np.int32)
            ptr = t.ctypes.data
        st = self._lib.gm_decoder_step(self._h, i, ptr, self._sptr)
        if st:
            self._check(st, "gm_decoder_step")
        self._steps += 1
        if self.collect_every and self._steps % self.collect_every == 0:
            with torch.cuda.stream(self.stream):  # stream-ordered after this step's K5
                self.collections += self._pool.maybe_collect(self.collect_threshold, self.stream)

    def flags(self, i: int = 0, out: Optional[np.ndarray] = None, wait: bool = True,
              raise_errors: bool = True) -> np.ndarray:
        """Accepted flags (uint8 [B]) of buffer i's latest step: bit 0 =
        token accepted, bit 1 = the request's step failed (cap, terminated,
        arena...).  With ``raise_errors`` a failed request raises its
        MatcherError (RequestErrors for several, each keyed by its index in
        the batch); an error-free step costs nothing extra."""
        o = self._flags if out is None else out
        st = self._lib.gm_decoder_flags(self._h, i, o.ctypes.data, 1 if wait else 0)
        if st:
            self._check(st, "gm_decoder_flags")
        if raise_errors and (o & 2).any():
            self._pool.raise_slot_errors(self.slots, o)
        return o

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.gm_decoder_release(self._h)
            self._h = None
        self._matchers = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
