"""Host front end, part 2: expression IR -> device automaton tables.

Pipeline (own design; only the recognised language must equal the
reference's):

1. per-rule NFA over byte classes, rule calls and epsilons
   (role of REF pda.py:246-329 build_pda);
2. per-rule subset construction + Moore minimisation, which subsumes the
   reference's node merging (REF pda.py:403-535): every rule becomes a DFA
   whose symbols are byte classes and rule calls;
3. inlining of small call-free rules into their callers, to fixpoint, then
   re-determinisation (role of REF pda.py:336-396 inline_rules);
4. silent-move pre-closure: for every node the relative closure over rule
   pushes and frame-internal pops is enumerated once (the work the
   reference's closure() repeats per byte, REF cache.py:110-143), giving
   per-(node, class) transition lists (push run, target) and the POP flag;
5. the context-expansion follow automaton (REF cache.py:241-333) determinised
   over the same byte classes;
6. packing into the gm_grammar_tables layout of include/gmask.h.

All of it runs in the native front end (csrc/front_end.cpp, through
build_tables_native below); this module holds the option / table types and
the grammar-IR encoding.  The Python restatement of the pipeline, used only
by the tests to check the native tables array for array, is
tests/automaton_spec.py.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

from .grammar import Alt, Bytes, Eps, GrammarError, Lit, ParsedGrammar, Ref, Rep, Seq

__all__ = ["StateLimitError", "CompiledTables", "AutomatonOptions", "NativeParsed", "build_tables_native",
           "encode_ir", "parse_grammar_native"]

DEFAULT_STATE_CAP = 4096  # REF pda.py:53
_FOLLOW_DEAD, _FOLLOW_ANY = -1, -2
NODE_POP, NODE_DEAD_END = 1, 2


class StateLimitError(RuntimeError):
    """Silent-move closure exceeded its cap (REF pda.py:56-57), e.g. left
    recursion."""


@dataclass
class AutomatonOptions:
    determinize: bool = True      # ≙ CompileOptions.merge
    inline: bool = True           # ≙ CompileOptions.inline
    ctx_expansion: bool = True    # ≙ CompileOptions.ctx_expansion
    inline_max_rule_states: int = 32
    inline_max_result_states: int = 1024
    # also inline a rule that calls other rules when exactly one live rule
    # calls it (no code duplication): collapses call chains such as JSON's
    # element -> value -> object -> members -> member into one rule, and
    # removes the repetition ambiguity of `item*` with `item ::= ... | text+`
    inline_calls: bool = True
    max_dfa_states: int = 200_000
    max_follow_states: int = 4096
    state_cap: int = DEFAULT_STATE_CAP



@dataclass
class CompiledTables:
    n_nodes: int
    n_rules: int
    n_classes: int
    start_node: int
    root_rule: int
    rule_names: List[str]
    byte_class: np.ndarray  # uint8[256]
    trans_off: np.ndarray  # int32[n_nodes*n_classes+1]
    trans: np.ndarray  # int32[2*n_trans]
    push_pool: np.ndarray  # int32
    node_flags: np.ndarray  # uint8
    node_rule: np.ndarray  # int32
    cache_keys: np.ndarray  # int32
    follow_start: np.ndarray  # int32[n_rules]
    follow_next: np.ndarray  # int32[n_fstates*n_classes]
    n_fstates: int
    stats: dict = field(default_factory=dict)
    # per-rule DFAs before the pre-closure (bundle export, bundle_io.py):
    # node u's edges raw[raw_off[u]:raw_off[u+1]] as (symbol, dst) rows,
    # symbol >= 0 a byte class, < 0 a call of rule -(symbol+1)
    raw_off: Optional[np.ndarray] = None
    raw: Optional[np.ndarray] = None
    finals: Optional[np.ndarray] = None
    rule_start: Optional[np.ndarray] = None


def encode_ir(g: ParsedGrammar) -> Tuple[np.ndarray, Dict[str, int]]:
    """Prefix int32 IR of every rule body, in rule-id (source) order — the
    input format of gm_front_end_build (front_end.cpp header)."""
    rid_of = {nm: i for i, nm in enumerate(g.names)}
    out: List[int] = []
    stack = []

    def emit(e):
        if isinstance(e, Eps):
            out.append(0)
        elif isinstance(e, Bytes):
            m = e.mask
            out.append(1)
            out.extend((m >> (32 * k)) & 0xFFFFFFFF for k in range(8))
        elif isinstance(e, Lit):
            out.append(2)
            out.append(len(e.data))
            out.extend(e.data)
        elif isinstance(e, (Seq, Alt)):
            out.append(3 if isinstance(e, Seq) else 4)
            out.append(len(e.items))
            for item in e.items:
                emit(item)
        elif isinstance(e, Rep):
            out.extend((5, e.lo, -1 if e.hi is None else e.hi))
            emit(e.item)
        elif isinstance(e, Ref):
            out.extend((6, rid_of[e.name]))
        else:
            raise TypeError(e)

    del stack
    for nm in g.names:
        emit(g.bodies[nm])
    arr = np.asarray(out, dtype=np.int64)
    return arr.astype(np.uint32).view(np.int32) if arr.size else arr.astype(np.int32), rid_of


@dataclass
class NativeParsed:
    """A grammar parsed by the native parser (gm_grammar_parse): rule names in
    source order, the root, and the prefix IR the front end takes."""

    names: List[str]
    root: str
    ir: np.ndarray

    @property
    def bodies(self) -> Dict[str, None]:  # membership tests (compile_grammar's root choice)
        return dict.fromkeys(self.names)


def parse_grammar_native(text: str, root_rule_name: Optional[str] = None) -> NativeParsed:
    """EBNF text -> NativeParsed through libgmask's C++ parser: the same IR,
    names, root and GrammarError (message, line, column) as
    grammar.parse_grammar + encode_ir (tests/test_frontend.py)."""
    import ctypes as C

    from . import _lib

    lib = _lib.load()
    data = text.encode("utf-8", "surrogatepass")
    view = _lib.gm_parse_view()
    h = C.c_void_p()
    st = lib.gm_grammar_parse(data, len(data), root_rule_name.encode() if root_rule_name is not None else None,
                              C.byref(h), C.byref(view))
    try:
        if st == _lib.GM_ERR_GRAMMAR:
            raise GrammarError(view.error.decode("utf-8", "replace"), view.err_line or None, view.err_col or None)
        _lib.check(st, "gm_grammar_parse")
        n = view.n_rules
        off = np.ctypeslib.as_array(C.cast(view.name_off, C.POINTER(C.c_int64)), shape=(n + 1,))
        blob = C.string_at(view.names, int(off[-1]))
        names = [blob[off[i]:off[i + 1] - 1].decode() for i in range(n)]
        ir = (np.ctypeslib.as_array(C.cast(view.ir, C.POINTER(C.c_int32)), shape=(view.ir_len,)).copy()
              if view.ir_len else np.zeros(0, np.int32))
        return NativeParsed(names, names[view.root_rule], ir)
    finally:
        if h:
            lib.gm_grammar_parse_release(h)


def build_tables_native(g, opts: Optional[AutomatonOptions] = None) -> CompiledTables:
    """build_tables through libgmask's C++ front end (gm_front_end_build):
    identical tables (tests/test_frontend.py compares them array for array),
    a fraction of the host time."""
    import ctypes as C

    from . import _lib

    opts = opts or AutomatonOptions()
    if not opts.determinize:
        raise NotImplementedError("determinize=False is not supported by the device tables")
    if isinstance(g, NativeParsed):
        ir, rid_of = g.ir, {nm: i for i, nm in enumerate(g.names)}
    else:
        ir, rid_of = encode_ir(g)
    ir = np.ascontiguousarray(ir)
    fo = _lib.gm_fe_options(1, int(opts.inline), int(opts.ctx_expansion), opts.inline_max_rule_states,
                            opts.inline_max_result_states, opts.max_dfa_states, opts.max_follow_states,
                            opts.state_cap, int(opts.inline_calls))
    view = _lib.gm_fe_tables()
    h = C.c_void_p()
    lib = _lib.load()
    st = lib.gm_front_end_build(ir.ctypes.data, ir.size, len(g.names), rid_of[g.root], C.byref(fo), C.byref(h),
                                C.byref(view))
    if st != _lib.GM_OK:
        msg = lib.gm_last_error().decode(errors="replace")
        if st == _lib.GM_ERR_STATE_CAP:
            raise StateLimitError(msg)
        if st == _lib.GM_ERR_GRAMMAR:
            raise GrammarError(msg)
        _lib.check(st, "gm_front_end_build")
    try:
        def arr(ptr, n, ct, dt):
            if n == 0:
                return np.zeros(0, dtype=dt)
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ct)), shape=(n,)).astype(dt, copy=True)

        v = view
        n_idx = v.n_nodes * v.n_classes
        kept = arr(v.kept_rules, v.n_rules, C.c_int32, np.int32)
        t = CompiledTables(
            n_nodes=v.n_nodes,
            n_rules=v.n_rules,
            n_classes=v.n_classes,
            start_node=v.start_node,
            root_rule=v.root_rule,
            rule_names=[g.names[r] for r in kept],
            byte_class=arr(v.byte_class, 256, C.c_uint8, np.uint8),
            trans_off=arr(v.trans_off, n_idx + 1, C.c_int32, np.int32),
            trans=arr(v.trans, 2 * v.n_trans, C.c_int32, np.int32),
            push_pool=arr(v.push_pool, v.n_push, C.c_int32, np.int32),
            node_flags=arr(v.node_flags, v.n_nodes, C.c_uint8, np.uint8),
            node_rule=arr(v.node_rule, v.n_nodes, C.c_int32, np.int32),
            cache_keys=arr(v.cache_keys, v.n_keys, C.c_int32, np.int32),
            follow_start=arr(v.follow_start, v.n_rules, C.c_int32, np.int32),
            follow_next=arr(v.follow_next, max(v.n_fstates, 1) * v.n_classes, C.c_int32, np.int32),
            n_fstates=v.n_fstates,
        )
        t.raw_off = arr(v.raw_off, v.n_nodes + 1, C.c_int32, np.int32)
        t.raw = arr(v.raw, 2 * v.n_raw, C.c_int32, np.int32).reshape(-1, 2)
        t.finals = arr(v.finals, v.n_nodes, C.c_uint8, np.uint8)
        t.rule_start = arr(v.rule_start, v.n_rules, C.c_int32, np.int32)
    finally:
        lib.gm_front_end_release(h)
    t.stats = {
        "nodes": t.n_nodes,
        "rules": t.n_rules,
        "classes": t.n_classes,
        "transitions": len(t.trans) // 2,
        "keys": len(t.cache_keys),
        "follow_states": t.n_fstates,
    }
    return t
