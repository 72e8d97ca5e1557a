"""Device-side engine objects over the C ABI.

DeviceVocab, DeviceGrammar and DeviceCache own libgmask handles; MatcherPool
owns the device-resident stack state of every live matcher (one pool per
CUDA device, slots handed out to matchers).  compile_on_device() is the
compile pipeline: host front end -> tables upload -> K1/K1b cache build
(optionally sharded over a torch.distributed group with an NCCL all-gather of
the finished rows) -> cache assembly.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _lib
from .automaton import AutomatonOptions, CompiledTables, StateLimitError, build_tables_native, parse_grammar_native
from .vocab import Vocabulary

__all__ = ["MatcherError", "RequestErrors", "DeviceVocab", "DeviceGrammar", "DeviceCache", "CompiledDeviceGrammar",
           "MatcherPool", "compile_on_device", "compile_many_on_device", "get_pool"]


class MatcherError(RuntimeError):
    """Runtime matcher misuse (REF matcher.py:35-36)."""


class RequestErrors(MatcherError):
    """Several requests of one batched call failed; ``errors`` maps the
    request's index in the batch to its MatcherError."""

    def __init__(self, errors: dict):
        self.errors = errors
        super().__init__("; ".join(f"request {i}: {e}" for i, e in sorted(errors.items())))


def error_for_status(status: int) -> Exception:
    """MatcherError for a device-side matcher status (REF matcher.py:35-36,
    188-189, 276-277, 313-314, 379-381); GmaskError otherwise."""
    msg = _lib.load().gm_last_error().decode(errors="replace")
    if status in (_lib.GM_ERR_STATE_CAP, _lib.GM_ERR_TERMINATED, _lib.GM_ERR_ROLLBACK, _lib.GM_ERR_INVALID,
                  _lib.GM_ERR_ARENA_FULL):
        return MatcherError(msg)
    return _lib.GmaskError(status, msg)


def error_for_bits(bits: int) -> Exception:
    return error_for_status(_lib.load().gm_status_of_error_bits(C.c_uint32(bits)))


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class DeviceVocab:
    """A Vocabulary uploaded to the current CUDA device (gm_vocab)."""

    def __init__(self, vocab: Vocabulary):
        _lib.require_cuda()
        lib = _lib.load()
        self.vocab = vocab
        self.size = vocab.size
        self.words = (vocab.size + 31) // 32
        self.device = torch.device("cuda", torch.cuda.current_device())
        data, off = vocab.packed()
        special = np.asarray(sorted(vocab.special_tokens), dtype=np.int32)
        h = C.c_void_p()
        _lib.check(lib.gm_vocab_create(_ptr(data), _ptr(off), vocab.size, _ptr(special), len(special),
                                       vocab.eos_id, C.byref(h)), "gm_vocab_create")
        self.handle = h
        self._hash = vocab.content_hash()

    def content_hash(self) -> bytes:
        return self._hash

    def __del__(self):
        if getattr(self, "handle", None) is not None and _lib._lib is not None:
            _lib._lib.gm_vocab_release(self.handle)
            self.handle = None


class DeviceGrammar:
    """Automaton tables resident on the device (gm_grammar)."""

    def __init__(self, t: CompiledTables):
        lib = _lib.load()
        self.tables = t
        self._keep = [t.byte_class, t.trans_off, t.trans, t.push_pool, t.node_flags, t.node_rule,
                      t.cache_keys, t.follow_start, t.follow_next]
        st = _lib.gm_grammar_tables(
            n_nodes=t.n_nodes, n_rules=t.n_rules, n_classes=t.n_classes, start_node=t.start_node,
            byte_class=_ptr(t.byte_class), trans_off=_ptr(t.trans_off), trans=_ptr(t.trans),
            n_trans=len(t.trans) // 2, push_pool=_ptr(t.push_pool), n_push=len(t.push_pool),
            node_flags=_ptr(t.node_flags), node_rule=_ptr(t.node_rule), cache_keys=_ptr(t.cache_keys),
            n_keys=len(t.cache_keys), follow_start=_ptr(t.follow_start), follow_next=_ptr(t.follow_next),
            n_fstates=t.n_fstates,
        )
        h = C.c_void_p()
        _lib.check(lib.gm_grammar_create(C.byref(st), C.byref(h)), "gm_grammar_create")
        self.handle = h
        self.n_keys = len(t.cache_keys)

    def __del__(self):
        if getattr(self, "handle", None) is not None and _lib._lib is not None:
            _lib._lib.gm_grammar_release(self.handle)
            self.handle = None


class DeviceCache:
    """Assembled adaptive cache: dense accepted rows + dependent id lists."""

    def __init__(self, grammar: DeviceGrammar, dvocab: DeviceVocab, acc_rows: torch.Tensor,
                 dep_rows: torch.Tensor, stream=None):
        lib = _lib.load()
        h = C.c_void_p()
        stats = _lib.gm_cache_stats()
        _lib.check(lib.gm_cache_create(grammar.handle, dvocab.handle, acc_rows.data_ptr(), dep_rows.data_ptr(),
                                       C.byref(h), C.byref(stats), _lib.stream_ptr(stream)), "gm_cache_create")
        self.handle = h
        self.grammar = grammar  # keep tables alive: the cache binding points at them
        self.dvocab = dvocab
        self.stats = {
            "entries": stats.n_keys,
            "accepted_total": stats.accepted_total,
            "dependent_total": stats.dependent_total,
            "rejected_total": stats.rejected_total,
            "row_bytes": stats.row_bytes,
            "blend_keys": stats.blend_keys,  # rows the fused apply blends (mixed-chunk policy)
        }

    def export(self):
        """(acc_rows [n_keys, W] int32 device tensor, dep_off numpy, dep_ids numpy) — inspection only."""
        lib = _lib.load()
        n, w = self.grammar.n_keys, self.dvocab.words
        nd = C.c_int64()
        _lib.check(lib.gm_cache_export(self.handle, None, None, None, C.byref(nd)), "gm_cache_export")
        acc = torch.empty((max(n, 1), w), dtype=torch.int32, device=self.dvocab.device)
        off = torch.empty(n + 1, dtype=torch.int32, device=self.dvocab.device)
        ids = torch.empty(max(nd.value, 1), dtype=torch.int32, device=self.dvocab.device)
        _lib.check(lib.gm_cache_export(self.handle, acc.data_ptr(), off.data_ptr(), ids.data_ptr(), None),
                   "gm_cache_export")
        return acc[:n], off.cpu().numpy(), ids[: nd.value].cpu().numpy()

    def __del__(self):
        if getattr(self, "handle", None) is not None and _lib._lib is not None:
            _lib._lib.gm_cache_release(self.handle)
            self.handle = None


@dataclass
class CompiledDeviceGrammar:
    tables: CompiledTables
    grammar: DeviceGrammar
    cache: DeviceCache
    dvocab: DeviceVocab
    timings_ms: dict = field(default_factory=dict)

    @property
    def stats(self) -> dict:
        return {**self.tables.stats, **self.cache.stats}


def build_cache_rows(grammar: DeviceGrammar, dvocab: DeviceVocab, key_begin: int, n: int, stream=None):
    lib = _lib.load()
    acc = torch.empty((n, dvocab.words), dtype=torch.int32, device=dvocab.device)
    dep = torch.empty((n, dvocab.words), dtype=torch.int32, device=dvocab.device)
    if n:
        status = lib.gm_cache_build_rows(grammar.handle, dvocab.handle, key_begin, n, acc.data_ptr(),
                                         dep.data_ptr(), _lib.stream_ptr(stream))
        if status == _lib.GM_ERR_STATE_CAP:
            raise StateLimitError(lib.gm_last_error().decode())
        _lib.check(status, "gm_cache_build_rows")
    return acc, dep


def build_cache_rows_keys(grammar: DeviceGrammar, dvocab: DeviceVocab, keys, stream=None):
    """Rows of an arbitrary list of cache keys (position sharding)."""
    lib = _lib.load()
    keys = np.ascontiguousarray(np.asarray(keys, dtype=np.int32))
    n = len(keys)
    acc = torch.empty((n, dvocab.words), dtype=torch.int32, device=dvocab.device)
    dep = torch.empty((n, dvocab.words), dtype=torch.int32, device=dvocab.device)
    if n:
        status = lib.gm_cache_build_keys(grammar.handle, dvocab.handle, keys.ctypes.data, n, acc.data_ptr(),
                                         dep.data_ptr(), _lib.stream_ptr(stream))
        if status == _lib.GM_ERR_STATE_CAP:
            raise StateLimitError(lib.gm_last_error().decode())
        _lib.check(status, "gm_cache_build_keys")
    return acc, dep


def shard_range(n_keys: int, world: int, rank: int):
    """Contiguous block of cache keys owned by ``rank`` (kept for callers
    that want blocks; the build deals keys with ``shard_keys``)."""
    per = (n_keys + world - 1) // world if world else n_keys
    return min(rank * per, n_keys), min((rank + 1) * per, n_keys), per


def key_costs(tables: CompiledTables, vocab: Vocabulary) -> np.ndarray:
    """Estimated K1 work per cache key: the token bytes whose
    first byte the key's node can consume — a position inside a string walks
    almost the whole sorted vocabulary, a structural one dies at byte 0 of
    most tokens (SURVEY §7 hard part 3)."""
    data, off = vocab.packed()
    lens = np.diff(off)
    nonempty = lens > 0
    first = np.zeros(len(lens), dtype=np.int64)
    first[nonempty] = data[off[:-1][nonempty]]
    cls = np.asarray(tables.byte_class, dtype=np.int64)
    C = int(tables.n_classes)
    per_class = np.zeros(C, dtype=np.float64)
    np.add.at(per_class, cls[first[nonempty]], lens[nonempty].astype(np.float64))
    toff = np.asarray(tables.trans_off, dtype=np.int64)
    keys = np.asarray(tables.cache_keys, dtype=np.int64)
    out = np.empty(len(keys), dtype=np.float64)
    for i, nd in enumerate(keys):
        idx = nd * C + np.arange(C)
        live = toff[idx + 1] > toff[idx]
        out[i] = per_class[live].sum() + 1.0
    return out


def shard_keys(costs, world: int, rank: int) -> np.ndarray:
    """Keys of ``rank``: all keys sorted by decreasing estimated cost (ties by
    index), dealt round-robin over the ranks, so every rank gets
    a share of the expensive string-interior positions."""
    order = np.argsort(-np.asarray(costs, dtype=np.float64), kind="stable")
    return order[rank::world].astype(np.int32)


def _all_gather(out: torch.Tensor, inp: torch.Tensor, group):
    import torch.distributed as dist

    if dist.get_backend(group) == "gloo" and inp.is_cuda:  # gloo collectives run on host copies
        o = out.cpu()
        dist.all_gather_into_tensor(o, inp.cpu(), group=group)
        out.copy_(o)
    else:
        dist.all_gather_into_tensor(out, inp, group=group)


def sharded_rows(build, n_keys: int, words: int, device, group=None, costs=None):
    """Position-sharded cache rows: each rank builds its keys with
    ``build(keys) -> (acc, dep)`` (rows in ``keys`` order; keys None = all,
    in order, for a single rank), one all-gather
    replicates them and every rank puts them back in key order (NCCL over
    NVLink on the GPU box; gloo in the CPU tests).  The result is identical
    on every rank and bit-identical to the 1-rank build (REF SPEC.md:364).
    Returns (acc, dep) [n_keys, words] int32."""
    world = 1
    if group is not None:
        import torch.distributed as dist

        world = dist.get_world_size(group)
    if costs is None:
        costs = np.zeros(n_keys)
    if world <= 1:
        return build(None)
    import torch.distributed as dist

    rank = dist.get_rank(group)
    per = (n_keys + world - 1) // world
    mine = shard_keys(costs, world, rank)
    acc_l, dep_l = build(mine)
    pad = torch.zeros((2, per, words), dtype=torch.int32, device=device)
    pad[0, : len(mine)] = acc_l
    pad[1, : len(mine)] = dep_l
    full = torch.empty((world * 2, per, words), dtype=torch.int32, device=device)
    _all_gather(full, pad, group)
    full = full.view(world, 2, per, words)
    acc = torch.empty((n_keys, words), dtype=torch.int32, device=device)
    dep = torch.empty((n_keys, words), dtype=torch.int32, device=device)
    for r in range(world):
        keys_r = torch.from_numpy(shard_keys(costs, world, r).astype(np.int64)).to(device)
        acc.index_copy_(0, keys_r, full[r, 0, : len(keys_r)])
        dep.index_copy_(0, keys_r, full[r, 1, : len(keys_r)])
    return acc, dep


def compile_on_device(text: str, dvocab: DeviceVocab, opts: Optional[AutomatonOptions] = None, *,
                      root_rule_name: Optional[str] = None, group=None, stream=None,
                      uncached: bool = False, parsed=None) -> CompiledDeviceGrammar:
    """Front end + K1/K1b build.  With a torch.distributed ``group`` of size G
    the cache keys are dealt round-robin in decreasing order of estimated
    cost (``key_costs``) and the rows replicated with one all-gather
    (SURVEY §8e)."""
    t0 = time.perf_counter()
    tables = build_tables_native(parsed if parsed is not None else parse_grammar_native(text, root_rule_name), opts)
    t1 = time.perf_counter()
    grammar = DeviceGrammar(tables)
    n_keys = grammar.n_keys
    if uncached:
        # no cache: every token is context dependent, fill walks the whole
        # vocabulary (the reference's uncached path, REF matcher.py:446-460)
        v = dvocab.vocab
        ok = np.fromiter((t not in v.special_tokens and len(v.tokens[t]) > 0 for t in range(v.size)), bool, v.size)
        u = np.packbits(np.concatenate([ok, np.zeros(32 * dvocab.words - v.size, bool)]), bitorder="little")
        acc = torch.zeros((n_keys, dvocab.words), dtype=torch.int32, device=dvocab.device)
        dep = torch.from_numpy(u.view(np.int32).copy()).to(dvocab.device).expand(n_keys, -1).contiguous()
    else:
        costs = key_costs(tables, dvocab.vocab) if group is not None else None
        def build(keys):  # None: every key (one contiguous range)
            if keys is None:
                return build_cache_rows(grammar, dvocab, 0, n_keys, stream)
            return build_cache_rows_keys(grammar, dvocab, keys, stream)

        acc, dep = sharded_rows(build, n_keys, dvocab.words, dvocab.device, group, costs)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    cache = DeviceCache(grammar, dvocab, acc, dep, stream)
    t3 = time.perf_counter()
    timings = {"front_end": (t1 - t0) * 1e3, "cache_build": (t2 - t1) * 1e3, "assemble": (t3 - t2) * 1e3,
               "total": (t3 - t0) * 1e3}
    return CompiledDeviceGrammar(tables, grammar, cache, dvocab, timings)


def compile_many_on_device(texts, dvocab: DeviceVocab, opts: Optional[AutomatonOptions] = None, *, group=None,
                           stream=None):
    """BASELINE config 5's build: every rank ends with ALL grammars compiled,
    the work sharded by grammar position across the group ("all
    positions of all schemas").  The host front end is dealt round-robin over
    the ranks and the tables exchanged (all_gather_object); the (grammar,
    key) pairs of all grammars are dealt round-robin in decreasing order of
    estimated cost; one all-gather of the padded rows replicates them.
    Returns (list of CompiledDeviceGrammar, stats with the per-rank bytes
    moved and phase ms).  Compare: per-rank compile (each rank compiles only
    the grammars of the requests it serves; no exchange)."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if group is not None else 1
    rank = dist.get_rank(group) if group is not None else 0
    t0 = time.perf_counter()
    mine = {i: build_tables_native(parse_grammar_native(texts[i]), opts) for i in range(rank, len(texts), world)}
    t1 = time.perf_counter()
    if world > 1:
        parts = [None] * world
        dist.all_gather_object(parts, mine, group=group)
        tables = {}
        for part in parts:
            tables.update(part)
    else:
        tables = mine
    t2 = time.perf_counter()
    grammars = [DeviceGrammar(tables[i]) for i in range(len(texts))]
    pairs, costs = [], []
    for i in range(len(texts)):
        c = key_costs(tables[i], dvocab.vocab)
        pairs += [(i, k) for k in range(len(c))]
        costs.append(c)
    costs = np.concatenate(costs) if costs else np.zeros(0)
    n = len(pairs)
    W = dvocab.words

    def build(sel):
        if sel is None:
            sel = np.arange(n)
        acc = torch.empty((len(sel), W), dtype=torch.int32, device=dvocab.device)
        dep = torch.empty((len(sel), W), dtype=torch.int32, device=dvocab.device)
        by_g = {}
        for j, p in enumerate(sel):
            by_g.setdefault(pairs[p][0], []).append((j, pairs[p][1]))
        for gi, lst in by_g.items():
            a, d = build_cache_rows_keys(grammars[gi], dvocab, [k for _, k in lst], stream)
            idx = torch.tensor([j for j, _ in lst], dtype=torch.int64, device=dvocab.device)
            acc.index_copy_(0, idx, a)
            dep.index_copy_(0, idx, d)
        return acc, dep

    acc, dep = sharded_rows(build, n, W, dvocab.device, group if world > 1 else None, costs)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    out, at = [], 0
    for i, g in enumerate(grammars):
        nk = g.n_keys
        cache = DeviceCache(g, dvocab, acc[at:at + nk].contiguous(), dep[at:at + nk].contiguous(), stream)
        out.append(CompiledDeviceGrammar(tables[i], g, cache, dvocab, {}))
        at += nk
    t4 = time.perf_counter()
    per = (n + world - 1) // world
    stats = {"grammars": len(texts), "positions": n, "world": world,
             "front_end_ms": (t1 - t0) * 1e3, "tables_exchange_ms": (t2 - t1) * 1e3,
             "cache_build_ms": (t3 - t2) * 1e3, "assemble_ms": (t4 - t3) * 1e3, "total_ms": (t4 - t0) * 1e3,
             "allgather_bytes_in_per_rank": (world - 1) * per * 2 * W * 4 if world > 1 else 0}
    return out, stats


# ---------------------------------------------------------------------------
# matcher pool


class MatcherPool:
    """Device-resident matcher slots (gm_pool) with a host free list."""

    def __init__(self, capacity: int = 4096, max_stacks: int = 32, max_window: int = 64, arena_log2: int = 24):
        _lib.require_cuda()
        lib = _lib.load()
        h = C.c_void_p()
        _lib.check(lib.gm_pool_create(capacity, max_stacks, max_window, arena_log2, C.byref(h)), "gm_pool_create")
        self.handle = h
        self.capacity = capacity
        self.max_window = max_window
        self.max_stacks = max_stacks
        self.device = torch.device("cuda", torch.cuda.current_device())
        self._free = list(range(capacity - 1, -1, -1))
        self._lock = threading.Lock()
        self._flag = torch.zeros(1, dtype=torch.uint8, device=self.device)
        self._pinned_flag = torch.zeros(1, dtype=torch.uint8).pin_memory()

    def alloc(self) -> int:
        with self._lock:
            if not self._free:
                raise MatcherError(f"matcher pool exhausted ({self.capacity} slots); set GMASK_POOL_SLOTS")
            return self._free.pop()

    def free(self, slot: int):
        with self._lock:
            self._free.append(slot)

    def check(self, runtime: bool = True):
        """Raise the OR of every slot's sticky error, clearing them all (syncs).
        Pool-wide diagnostic: per-request errors use ``slot_errors``."""
        flags = C.c_int32()
        status = _lib.load().gm_pool_check(self.handle, C.byref(flags))
        if status != _lib.GM_OK:
            raise error_for_status(status)

    def slot_errors(self, slots: torch.Tensor, clear: bool = True) -> np.ndarray:
        """Per-slot error words (uint32, bit 1 << GM_ERR_*) of ``slots``
        (int32 CUDA tensor), cleared by the read.  Syncs the current stream."""
        out = torch.empty(slots.numel(), dtype=torch.int32, device=slots.device)
        _lib.check(_lib.load().gm_pool_errors(self.handle, slots.data_ptr(), slots.numel(), out.data_ptr(),
                                               1 if clear else 0, _lib.stream_ptr()), "gm_pool_errors")
        return out.cpu().numpy().view(np.uint32)

    def raise_slot_errors(self, slots: torch.Tensor, flags: Optional[np.ndarray] = None):
        """Raise for the requests among ``slots`` whose device operation
        failed (REF raises MatcherError on that matcher, matcher.py:188-189,
        379-381).  With ``flags`` (K4/K5 accepted flags, bit 1 = error) only
        a flagged batch pays the read.  One request: its MatcherError; more:
        RequestErrors carrying each request's exception."""
        if flags is not None and not (np.asarray(flags) & 2).any():
            return
        words = self.slot_errors(slots)
        bad = {i: error_for_bits(int(w)) for i, w in enumerate(words) if w}
        if not bad:
            return
        if len(bad) == 1:
            (i, exc), = bad.items()
            exc.request_index = i
            raise exc
        raise RequestErrors(bad)

    def live_slots(self) -> list:
        """Slots currently handed out to matchers."""
        with self._lock:
            free = set(self._free)
        return [s for s in range(self.capacity) if s not in free]

    def arena_stats(self) -> dict:
        """Frames in the device arena (syncs): live, tombstones, capacity."""
        live, tomb, cap = C.c_int64(), C.c_int64(), C.c_int64()
        _lib.check(_lib.load().gm_pool_arena_stats(self.handle, C.byref(live), C.byref(tomb), C.byref(cap)),
                   "gm_pool_arena_stats")
        return {"live": live.value, "tombstones": tomb.value, "capacity": cap.value,
                "occupancy": (live.value + tomb.value) / max(cap.value, 1)}

    def collect(self, stream=None, live_slots=None) -> None:
        """Reclaim the arena frames no live matcher references (REF
        pstack.py:85-111).  Stream-ordered; no step on this pool may run on
        another stream meanwhile.  ``live_slots`` defaults to every slot
        handed out."""
        live = np.ascontiguousarray(np.asarray(self.live_slots() if live_slots is None else live_slots,
                                               dtype=np.int32))
        _lib.check(_lib.load().gm_pool_collect(self.handle, live.ctypes.data if len(live) else None, len(live),
                                               _lib.stream_ptr(stream)), "gm_pool_collect")

    def maybe_collect(self, threshold: float = 0.5, stream=None) -> bool:
        """Collect when live + tombstoned frames exceed ``threshold`` of the
        arena (syncs for the count)."""
        if self.arena_stats()["occupancy"] <= threshold:
            return False
        self.collect(stream)
        return True

    def __del__(self):
        if getattr(self, "handle", None) is not None and _lib._lib is not None:
            _lib._lib.gm_pool_release(self.handle)
            self.handle = None


_pools: dict = {}


def get_pool(device=None) -> MatcherPool:
    dev = torch.cuda.current_device() if device is None else torch.device(device).index
    pool = _pools.get(dev)
    if pool is None:
        with torch.cuda.device(dev):
            pool = MatcherPool(
                capacity=int(os.environ.get("GMASK_POOL_SLOTS", "4096")),
                max_window=int(os.environ.get("GMASK_MAX_WINDOW", "64")),
                arena_log2=int(os.environ.get("GMASK_ARENA_LOG2", "24")),
            )
        _pools[dev] = pool
    return pool
