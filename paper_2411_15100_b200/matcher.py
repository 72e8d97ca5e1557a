"""Matchers over device-resident stacks (K2 fill, K4 accept).

``SlotMatcher`` is the shared core: one slot of the per-device MatcherPool
(engine.py), i.e. a ring of stack-top sets in HBM plus handles into the
hash-consed frame arena.  ``GrammarMatcher`` / ``BatchGrammarMatcher`` expose
XGrammar 0.2.0's names (xgrammar/matcher.py:191-534); the grammask adapter in
compat.py exposes the reference's (REF matcher.py:103-495).

Single-matcher calls that must return a host value (accept_token -> bool,
fill -> need_apply) synchronise; the batched calls are stream-ordered and
sync-free, so a decode loop runs accept -> fill -> apply entirely on the GPU.
"""

from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence, Union

import numpy as np
import torch

from . import _lib
from .bitmask import apply_token_bitmask_inplace  # noqa: F401  (re-export)
from .engine import MatcherError, MatcherPool, RequestErrors, get_pool

__all__ = ["SlotMatcher", "GrammarMatcher", "BatchGrammarMatcher", "MatcherError", "RequestErrors"]


class SlotMatcher:
    """One matcher slot; holds (compiled grammar, pool slot, device scratch)."""

    def __init__(self, compiled, window: int, pool: Optional[MatcherPool] = None, _slot: Optional[int] = None):
        self.compiled = compiled  # CompiledGrammar (keeps device tables alive)
        self._dev = compiled._dev
        self.pool = pool or get_pool()
        if window > self.pool.max_window:
            raise MatcherError(f"history window {window} exceeds the pool maximum {self.pool.max_window}")
        self.window = window
        self.vocab = self._dev.dvocab.vocab
        self.slot = self.pool.alloc() if _slot is None else _slot
        dev = self.pool.device
        self._slot_t = torch.tensor([self.slot], dtype=torch.int32, device=dev)
        self._tok_t = torch.zeros(1, dtype=torch.int32, device=dev)
        self._out_t = torch.zeros(1, dtype=torch.uint8, device=dev)
        self._closed = False
        if _slot is None:
            self.reset()

    # -- lifecycle --------------------------------------------------------------
    def reset(self):
        lib = _lib.load()
        _lib.check(lib.gm_pool_reset(self.pool.handle, self.slot, self._dev.grammar.handle, self._dev.cache.handle,
                                     self._dev.dvocab.handle, self.window, _lib.stream_ptr()), "gm_pool_reset")

    def fork(self) -> "SlotMatcher":
        other = SlotMatcher(self.compiled, self.window, self.pool, _slot=self.pool.alloc())
        _lib.check(_lib.load().gm_pool_fork(self.pool.handle, self.slot, other.slot, _lib.stream_ptr()), "gm_pool_fork")
        return other

    def release(self):
        if not self._closed:
            self._closed = True
            self.pool.free(self.slot)

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass

    # -- state ------------------------------------------------------------------
    def info(self) -> dict:
        buf = (C.c_int32 * 5)()
        stacks = (C.c_int32 * 64)()
        _lib.check(_lib.load().gm_pool_slot_info(self.pool.handle, self.slot, buf, stacks, 32), "slot_info")
        n = buf[0]
        return {
            "n_stacks": n,
            "terminated": bool(buf[1]),
            "history_len": buf[2],
            "terminable": bool(buf[3]),
            "window": buf[4],
            "stacks": [(stacks[2 * i], stacks[2 * i + 1]) for i in range(min(n, 32))],
        }

    def materialize(self, handle: int) -> tuple:
        out = (C.c_int32 * 4096)()
        depth = C.c_int32()
        _lib.check(_lib.load().gm_pool_materialize(self.pool.handle, handle, out, 4096, C.byref(depth)), "materialize")
        return tuple(out[i] for i in range(min(depth.value, 4096)))

    def first_bytes(self):
        words = (C.c_uint32 * 8)()
        term = C.c_int32()
        _lib.check(_lib.load().gm_pool_first_bytes(self.pool.handle, self.slot, words, C.byref(term)), "first_bytes")
        mask = 0
        for i in range(8):
            mask |= int(words[i]) << (32 * i)
        return mask, bool(term.value)

    def check(self):
        """Raise this matcher's own device error, if any (syncs; clears it)."""
        self.pool.raise_slot_errors(self._slot_t)

    # -- stepping -----------------------------------------------------------------
    def accept_token(self, tid: int) -> bool:
        """Device accept; False = rejected (state unchanged); raises this
        matcher's MatcherError on a device error (terminated / cap / range)."""
        self._tok_t.fill_(int(tid))
        _lib.check(_lib.load().gm_accept_tokens(self.pool.handle, self._slot_t.data_ptr(), self._tok_t.data_ptr(), 1,
                                                 self._out_t.data_ptr(), _lib.stream_ptr()), "gm_accept_tokens")
        flag = int(self._out_t.item())
        if flag & 2:
            self.check()
        return bool(flag & 1)

    def accept_bytes(self, data: bytes) -> bool:
        buf = np.frombuffer(bytes(data), dtype=np.uint8) if data else np.zeros(1, np.uint8)
        _lib.check(_lib.load().gm_accept_bytes(self.pool.handle, self.slot, buf.ctypes.data, len(data),
                                                self._out_t.data_ptr(), _lib.stream_ptr()), "gm_accept_bytes")
        flag = int(self._out_t.item())
        if flag & 2:
            self.check()
        return bool(flag & 1)

    def fill_row(self, bitmask: torch.Tensor, index: int = 0, need_apply: bool = True) -> Optional[bool]:
        """K2 for this slot into bitmask[index] (CUDA int32 2-D)."""
        row_ptr = bitmask.data_ptr() + index * bitmask.stride(0) * 4
        _lib.check(_lib.load().gm_fill_tokens(self.pool.handle, self._slot_t.data_ptr(), 1, row_ptr, bitmask.stride(0),
                                               None, self._out_t.data_ptr() if need_apply else None,
                                               _lib.stream_ptr()), "gm_fill_tokens")
        if need_apply:
            return bool(self._out_t.item())
        return None

    def rollback(self, steps: int):
        steps_t = torch.tensor([int(steps)], dtype=torch.int32, device=self.pool.device)
        _lib.check(_lib.load().gm_rollback(self.pool.handle, self._slot_t.data_ptr(), steps_t.data_ptr(), 1,
                                            _lib.stream_ptr()), "gm_rollback")
        self.check()

    def jump_forward(self, max_len: int = 4096) -> bytes:
        """Longest forced byte string (REF matcher.py:464-486); state unchanged."""
        scratch = self.fork()
        forced = bytearray()
        try:
            while len(forced) < max_len:
                allowed, term = scratch.first_bytes()
                if term or bin(allowed).count("1") != 1:
                    break
                b = allowed.bit_length() - 1
                if not scratch.accept_bytes(bytes([b])):
                    break
                forced.append(b)
        finally:
            scratch.release()
        return bytes(forced)


def _rollback_window(max_rollback_tokens: int, pool: MatcherPool) -> int:
    if max_rollback_tokens is None or max_rollback_tokens < 0:
        return pool.max_window
    return min(int(max_rollback_tokens), pool.max_window)


class GrammarMatcher:
    """XGrammar-compatible matcher (xgrammar/matcher.py:191-468)."""

    def __init__(self, compiled_grammar, *, override_stop_tokens: Optional[Union[int, List[int]]] = None,
                 terminate_without_stop_token: bool = False, max_rollback_tokens: int = -1) -> None:
        from .compiler import CompiledGrammar

        if not isinstance(compiled_grammar, CompiledGrammar):
            raise ValueError("The grammar should be compiled before passing it to GrammarMatcher.")
        if override_stop_tokens is not None:
            stops = [override_stop_tokens] if isinstance(override_stop_tokens, int) else list(override_stop_tokens)
            if stops != [compiled_grammar.tokenizer_info.vocab.eos_id]:
                raise ValueError("override_stop_tokens must equal the tokenizer's single EOS id")
        if terminate_without_stop_token:
            raise ValueError("terminate_without_stop_token is not supported (grammask EOS semantics)")
        pool = get_pool()
        self._core = SlotMatcher(compiled_grammar, _rollback_window(max_rollback_tokens, pool), pool)
        self._compiled = compiled_grammar

    @property
    def slot(self) -> int:
        return self._core.slot

    def accept_token(self, token_id: int, *, debug_print: bool = False) -> bool:
        if not 0 <= token_id < self._core.vocab.size:
            return False
        try:
            return self._core.accept_token(token_id)
        except MatcherError as exc:
            if "terminated" in str(exc):
                return False
            raise

    def accept_string(self, input_str: Union[str, bytes], *, debug_print: bool = False) -> bool:
        data = input_str.encode("utf-8") if isinstance(input_str, str) else bytes(input_str)
        try:
            return self._core.accept_bytes(data)
        except MatcherError as exc:
            if "terminated" in str(exc):
                return False
            raise

    def fill_next_token_bitmask(self, bitmask: torch.Tensor, index: int = 0, *, debug_print: bool = False) -> bool:
        """Fill bitmask[index] on the GPU; returns need_apply.  A CPU bitmask is
        accepted for drop-in use: the row is produced in HBM and copied out."""
        if bitmask.dtype != torch.int32 or bitmask.dim() != 2:
            raise RuntimeError("bitmask must be a 2-D int32 tensor")
        if bitmask.shape[1] * 32 < self._core.vocab.size:
            raise RuntimeError("bitmask is narrower than the vocabulary")
        if bitmask.device.type == "cuda":
            need = self._core.fill_row(bitmask, index)
        else:
            tmp = torch.empty((1, bitmask.shape[1]), dtype=torch.int32, device=self._core.pool.device)
            need = self._core.fill_row(tmp, 0)
            bitmask[index].copy_(tmp[0])
        self._core.check()  # this matcher's error: terminated -> MatcherError (REF matcher.py:379-381)
        return bool(need)

    def find_jump_forward_string(self) -> str:
        return self._core.jump_forward().decode("utf-8", errors="replace")

    def rollback(self, num_tokens: int = 1) -> None:
        self._core.rollback(num_tokens)

    def is_terminated(self) -> bool:
        return self._core.info()["terminated"]

    def is_completed(self) -> bool:
        return self._core.info()["terminable"]

    def reset(self) -> None:
        self._core.reset()

    def fork(self) -> "GrammarMatcher":
        m = GrammarMatcher.__new__(GrammarMatcher)
        m._core = self._core.fork()
        m._compiled = self._compiled
        return m

    @property
    def max_rollback_tokens(self) -> int:
        return self._core.window

    @property
    def stop_token_ids(self) -> List[int]:
        return [self._core.vocab.eos_id]

    def _debug_print_internal_state(self) -> str:
        return repr(self._core.info())


class BatchGrammarMatcher:
    """Batched fill / accept (xgrammar/matcher.py:482-534) — one kernel each,
    stream-ordered, no host synchronisation inside."""

    def __init__(self, max_threads: Union[int, str] = "auto") -> None:
        del max_threads
        self._slot_cache = {}

    def _slots(self, matchers: Sequence[GrammarMatcher]) -> torch.Tensor:
        key = tuple(m.slot for m in matchers)
        t = self._slot_cache.get(key)
        if t is None:
            if len(self._slot_cache) > 64:
                self._slot_cache.clear()
            t = torch.tensor(key, dtype=torch.int32, device=get_pool().device)
            self._slot_cache[key] = t
        return t

    def batch_fill_next_token_bitmask(self, matchers: Sequence[GrammarMatcher], bitmask: torch.Tensor,
                                      indices: Optional[Sequence[int]] = None, debug_print: bool = False,
                                      check_errors: bool = True) -> None:
        """K2 over the batch.  With ``check_errors`` (default, the reference's
        behaviour) a request whose fill failed raises its MatcherError
        (RequestErrors for several; syncs); ``check_errors=False`` keeps the
        call sync-free and leaves the errors in the slots' error words
        (``check_errors(matchers)``)."""
        if not matchers:
            return
        if bitmask.device.type != "cuda" or bitmask.dtype != torch.int32 or bitmask.dim() != 2:
            raise RuntimeError("bitmask must be a 2-D int32 CUDA tensor")
        rows = None
        if indices is not None:
            rows = torch.as_tensor(list(indices), dtype=torch.int32).to(bitmask.device, non_blocking=True)
        slots = self._slots(matchers)
        batch_fill(get_pool(), slots, bitmask, rows)
        if check_errors:
            get_pool().raise_slot_errors(slots)

    def check_errors(self, matchers: Sequence[GrammarMatcher], flags=None) -> None:
        """Raise the device errors of ``matchers`` (per request; syncs).
        ``flags``: the accepted flags of a batch_step (bit 1 = error), so an
        error-free batch costs nothing beyond reading them."""
        if matchers:
            get_pool().raise_slot_errors(self._slots(matchers), flags)

    def batch_fill_and_apply(self, matchers: Sequence[GrammarMatcher], logits: torch.Tensor,
                             bitmask: Optional[torch.Tensor] = None, vocab_size: Optional[int] = None) -> None:
        """Fused fill_next_token_bitmask + apply_token_bitmask_inplace for
        logits[i] <- matchers[i] (one kernel; bitmask optional output)."""
        if not matchers:
            return
        batch_fill_apply(get_pool(), self._slots(matchers), logits, bitmask, vocab_size=vocab_size)

    def batch_step(self, matchers: Sequence[GrammarMatcher], tokens=None, *, bitmask: Optional[torch.Tensor] = None,
                   logits: Optional[torch.Tensor] = None, recycle: bool = False,
                   accepted: Optional[torch.Tensor] = None) -> Optional[torch.Tensor]:
        """One decode step in one kernel (K5): accept ``tokens`` (int32 CUDA
        tensor or list; None on the first step), optionally restart finished
        requests, then fill the next masks into ``bitmask`` and/or apply
        them to ``logits`` in place.  Equivalent to batch_accept_token +
        (recycle) + batch_fill_next_token_bitmask [+ apply].  Returns the
        uint8 accepted flags on the device (or None without tokens)."""
        if not matchers:
            return None
        slots = self._slots(matchers)
        if tokens is not None and not isinstance(tokens, torch.Tensor):
            tokens = torch.tensor(list(tokens), dtype=torch.int32).to(slots.device, non_blocking=True)
        if tokens is not None and accepted is None:
            accepted = torch.empty(len(matchers), dtype=torch.uint8, device=slots.device)
        batch_step(get_pool(), slots, tokens, accepted if tokens is not None else None, bitmask, logits,
                   recycle=recycle, host_slots=[m.slot for m in matchers])
        return accepted if tokens is not None else None

    @staticmethod
    def batch_accept_token(matchers: Sequence[GrammarMatcher], tokens: Sequence[int],
                           debug_print: bool = False) -> List[bool]:
        pool = get_pool()
        slots = torch.tensor([m.slot for m in matchers], dtype=torch.int32, device=pool.device)
        toks = torch.tensor(list(tokens), dtype=torch.int32, device=pool.device)
        flags = batch_accept(pool, slots, toks).cpu().numpy()
        pool.raise_slot_errors(slots, flags)  # per-request MatcherError (bit 1 = error)
        return [bool(x & 1) for x in flags.tolist()]


def batch_fill(pool: MatcherPool, slots: torch.Tensor, bitmask: torch.Tensor, rows: Optional[torch.Tensor] = None,
               need_apply: Optional[torch.Tensor] = None, stream=None) -> None:
    """K2 over device slot ids (int32 CUDA tensor) — the zero-copy entry."""
    _lib.check(_lib.load().gm_fill_tokens(pool.handle, slots.data_ptr(), slots.numel(), bitmask.data_ptr(),
                                           bitmask.stride(0), rows.data_ptr() if rows is not None else None,
                                           need_apply.data_ptr() if need_apply is not None else None,
                                           _lib.stream_ptr(stream)), "gm_fill_tokens")


def batch_fill_apply(pool: MatcherPool, slots: torch.Tensor, logits: torch.Tensor,
                     bitmask: Optional[torch.Tensor] = None, rows: Optional[torch.Tensor] = None,
                     vocab_size: Optional[int] = None, stream=None) -> None:
    """K3: fill the masks of ``slots`` and apply them to ``logits`` in one
    kernel (optionally also storing the bitmask).  Same results as
    batch_fill followed by apply_token_bitmask_inplace."""
    from .bitmask import _DTYPES

    if logits.dtype not in _DTYPES or logits.dim() != 2 or logits.stride(-1) != 1:
        raise ValueError("logits must be a 2-D fp32/fp16/bf16 CUDA tensor, contiguous per row")
    v = logits.shape[1] if vocab_size is None else vocab_size
    _lib.check(_lib.load().gm_fill_apply_tokens(
        pool.handle, slots.data_ptr(), slots.numel(),
        bitmask.data_ptr() if bitmask is not None else None, bitmask.stride(0) if bitmask is not None else 0,
        rows.data_ptr() if rows is not None else None, logits.data_ptr(), _DTYPES[logits.dtype], v,
        logits.stride(0), _lib.stream_ptr(stream)), "gm_fill_apply_tokens")


def batch_step(pool: MatcherPool, slots: torch.Tensor, tokens: Optional[torch.Tensor], accepted: Optional[torch.Tensor],
               bitmask: Optional[torch.Tensor] = None, logits: Optional[torch.Tensor] = None,
               rows: Optional[torch.Tensor] = None, recycle: bool = False, vocab_size: Optional[int] = None,
               stream=None, host_slots: Optional[Sequence[int]] = None) -> None:
    """K5, one launch per decode step: accept ``tokens`` (int32 CUDA or pinned
    host, or None for the first step) into ``accepted`` (uint8 CUDA or pinned
    host; host buffers are read/written by the kernel directly), optionally restart
    requests that terminated, then fill the next masks into ``bitmask``
    and/or apply them to ``logits`` in place."""
    from .bitmask import _DTYPES

    if logits is not None and (logits.dtype not in _DTYPES or logits.dim() != 2 or logits.stride(-1) != 1):
        raise ValueError("logits must be a 2-D fp32/fp16/bf16 CUDA tensor, contiguous per row")
    if tokens is not None and accepted is None:
        raise ValueError("accepted output is required with tokens")
    for t in (tokens, accepted):  # device tensors, or pinned host memory read/written by the kernel (zero-copy)
        if t is not None and t.device.type == "cpu" and not t.is_pinned():
            raise ValueError("tokens / accepted must be CUDA tensors or pinned host tensors")
    v = (logits.shape[1] if vocab_size is None else vocab_size) if logits is not None else 0
    if host_slots is not None and rows is None and len(host_slots) <= 512 and (tokens is None or tokens.is_cuda):
        # slot ids by value in the launch parameters (host copy of ``slots``)
        hs = np.ascontiguousarray(np.asarray(host_slots, dtype=np.int32))
        _lib.check(_lib.load().gm_step_tokens_host_slots(
            pool.handle, hs.ctypes.data, len(hs), tokens.data_ptr() if tokens is not None else None,
            accepted.data_ptr() if accepted is not None else None, 1 if recycle else 0,
            bitmask.data_ptr() if bitmask is not None else None, bitmask.stride(0) if bitmask is not None else 0,
            logits.data_ptr() if logits is not None else None, _DTYPES[logits.dtype] if logits is not None else 0, v,
            logits.stride(0) if logits is not None else 0, _lib.stream_ptr(stream)), "gm_step_tokens_host_slots")
        return
    _lib.check(_lib.load().gm_step_tokens(
        pool.handle, slots.data_ptr(), slots.numel(), tokens.data_ptr() if tokens is not None else None,
        accepted.data_ptr() if accepted is not None else None, 1 if recycle else 0,
        bitmask.data_ptr() if bitmask is not None else None, bitmask.stride(0) if bitmask is not None else 0,
        rows.data_ptr() if rows is not None else None, logits.data_ptr() if logits is not None else None,
        _DTYPES[logits.dtype] if logits is not None else 0, v, logits.stride(0) if logits is not None else 0,
        _lib.stream_ptr(stream)), "gm_step_tokens")


def batch_recycle(pool: MatcherPool, slots: torch.Tensor, stream=None) -> None:
    """Restart every terminated slot among ``slots`` (serving loops)."""
    _lib.check(_lib.load().gm_pool_recycle(pool.handle, slots.data_ptr(), slots.numel(), _lib.stream_ptr(stream)),
               "gm_pool_recycle")


def batch_accept(pool: MatcherPool, slots: torch.Tensor, tokens: torch.Tensor, out: Optional[torch.Tensor] = None,
                 stream=None) -> torch.Tensor:
    """K4 over device slot ids / token ids; returns uint8 accepted flags (device)."""
    if out is None:
        out = torch.empty(slots.numel(), dtype=torch.uint8, device=slots.device)
    _lib.check(_lib.load().gm_accept_tokens(pool.handle, slots.data_ptr(), tokens.data_ptr(), slots.numel(),
                                             out.data_ptr(), _lib.stream_ptr(stream)), "gm_accept_tokens")
    return out
