"""ctypes binding of libgmask.so (include/gmask.h).

This module is the only place Python touches the C ABI.  There is no CPU
fallback: if the library is missing or no CUDA device is present, every
entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["GMASK_LIB"]) if os.environ.get("GMASK_LIB") else _HERE / "libgmask.so"

GM_OK = 0
GM_ERR_INVALID = 1
GM_ERR_CUDA = 2
GM_ERR_STATE_CAP = 3
GM_ERR_TERMINATED = 4
GM_ERR_SHAPE = 5
GM_ERR_ARENA_FULL = 6
GM_ERR_ROLLBACK = 7
GM_ERR_OOM = 8
GM_ERR_GRAMMAR = 9

GM_DTYPE_F32, GM_DTYPE_F16, GM_DTYPE_BF16 = 0, 1, 2
GM_NODE_POP, GM_NODE_DEAD_END = 1, 2
GM_FOLLOW_DEAD, GM_FOLLOW_ANY = -1, -2


class GmaskError(RuntimeError):
    """A libgmask call failed; ``code`` is the gm_status value."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


class gm_grammar_tables(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int32),
        ("n_rules", C.c_int32),
        ("n_classes", C.c_int32),
        ("start_node", C.c_int32),
        ("byte_class", C.c_void_p),
        ("trans_off", C.c_void_p),
        ("trans", C.c_void_p),
        ("n_trans", C.c_int32),
        ("push_pool", C.c_void_p),
        ("n_push", C.c_int32),
        ("node_flags", C.c_void_p),
        ("node_rule", C.c_void_p),
        ("cache_keys", C.c_void_p),
        ("n_keys", C.c_int32),
        ("follow_start", C.c_void_p),
        ("follow_next", C.c_void_p),
        ("n_fstates", C.c_int32),
    ]


class gm_fe_options(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("determinize", "inline_rules", "ctx_expansion", "inline_max_rule_states",
                                          "inline_max_result_states", "max_dfa_states", "max_follow_states",
                                          "state_cap", "inline_calls")]


class gm_fe_tables(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("n_nodes", "n_rules", "n_classes", "start_node", "root_rule", "n_trans",
                                          "n_push", "n_keys", "n_fstates")] + [
        (n, C.c_void_p) for n in ("byte_class", "trans_off", "trans", "push_pool", "node_flags", "node_rule",
                                  "cache_keys", "follow_start", "follow_next", "kept_rules", "raw_off", "raw")] + [
        ("n_raw", C.c_int32), ("finals", C.c_void_p), ("rule_start", C.c_void_p)]


class gm_parse_view(C.Structure):
    _fields_ = [("ir", C.c_void_p), ("ir_len", C.c_int64), ("n_rules", C.c_int32), ("root_rule", C.c_int32),
                ("names", C.c_void_p), ("name_off", C.c_void_p), ("error", C.c_char_p), ("err_line", C.c_int32),
                ("err_col", C.c_int32)]


class gm_cache_stats(C.Structure):
    _fields_ = [
        ("n_keys", C.c_int32),
        ("accepted_total", C.c_int64),
        ("dependent_total", C.c_int64),
        ("rejected_total", C.c_int64),
        ("row_bytes", C.c_int64),
        ("blend_keys", C.c_int32),
    ]


_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64

_SIGNATURES = {
    "gm_last_error": ([], C.c_char_p),
    "gm_version": ([], C.c_char_p),
    "gm_apply_inplace": ([_P, _I32, _I64, _I64, _I64, _P, _I64, _P, _P], _I32),
    "gm_apply_set_blend": ([_I32], _I32),
    "gm_vocab_create": ([_P, _P, _I32, _P, _I32, _I32, C.POINTER(_P)], _I32),
    "gm_vocab_release": ([_P], None),
    "gm_vocab_size": ([_P], _I32),
    "gm_vocab_universe": ([_P], _P),
    "gm_grammar_create": ([C.POINTER(gm_grammar_tables), C.POINTER(_P)], _I32),
    "gm_grammar_release": ([_P], None),
    "gm_cache_build_rows": ([_P, _P, _I32, _I32, _P, _P, _P], _I32),
    "gm_cache_build_keys": ([_P, _P, _P, _I32, _P, _P, _P], _I32),
    "gm_grammar_num_keys": ([_P], _I32),
    "gm_cache_create": ([_P, _P, _P, _P, C.POINTER(_P), C.POINTER(gm_cache_stats), _P], _I32),
    "gm_cache_release": ([_P], None),
    "gm_cache_export": ([_P, _P, _P, _P, C.POINTER(_I64)], _I32),
    "gm_pool_create": ([_I32, _I32, _I32, _I64, C.POINTER(_P)], _I32),
    "gm_pool_release": ([_P], None),
    "gm_pool_reset": ([_P, _I32, _P, _P, _P, _I32, _P], _I32),
    "gm_pool_fork": ([_P, _I32, _I32, _P], _I32),
    "gm_accept_tokens": ([_P, _P, _P, _I32, _P, _P], _I32),
    "gm_accept_bytes": ([_P, _I32, _P, _I64, _P, _P], _I32),
    "gm_fill_tokens": ([_P, _P, _I32, _P, _I64, _P, _P, _P], _I32),
    "gm_rollback": ([_P, _P, _P, _I32, _P], _I32),
    "gm_fill_apply_tokens": ([_P, _P, _I32, _P, _I64, _P, _P, _I32, _I64, _I64, _P], _I32),
    "gm_pool_recycle": ([_P, _P, _I32, _P], _I32),
    "gm_step_tokens": ([_P, _P, _I32, _P, _P, _I32, _P, _I64, _P, _P, _I32, _I64, _I64, _P], _I32),
    "gm_step_tokens_host_slots": ([_P, _P, _I32, _P, _P, _I32, _P, _I64, _P, _I32, _I64, _I64, _P], _I32),
    "gm_decoder_create": ([_P, _P, _I32, _I32, _P, _I64, _P, _I32, _I64, _I64, _I32, C.POINTER(_P)], _I32),
    "gm_decoder_step": ([_P, _I32, _P, _P], _I32),
    "gm_decoder_flags": ([_P, _I32, _P, _I32], _I32),
    "gm_decoder_release": ([_P], None),
    "gm_pool_slot_info": ([_P, _I32, _P, _P, _I32], _I32),
    "gm_pool_materialize": ([_P, _I32, _P, _I32, _P], _I32),
    "gm_pool_first_bytes": ([_P, _I32, _P, _P], _I32),
    "gm_pool_check": ([_P, _P], _I32),
    "gm_pool_errors": ([_P, _P, _I32, _P, _I32, _P], _I32),
    "gm_status_of_error_bits": ([C.c_uint32], _I32),
    "gm_pool_arena_used": ([_P], _I64),
    "gm_pool_arena_stats": ([_P, _P, _P, _P], _I32),
    "gm_pool_collect": ([_P, _P, _I32, _P], _I32),
    "gm_pool_trace": ([_P, _P, _I64], _I32),
    "gm_front_end_build": ([_P, _I64, _I32, _I32, C.POINTER(gm_fe_options), C.POINTER(_P),
                            C.POINTER(gm_fe_tables)], _I32),
    "gm_front_end_release": ([_P], None),
    "gm_grammar_parse": ([_P, _I64, C.c_char_p, C.POINTER(_P), C.POINTER(gm_parse_view)], _I32),
    "gm_grammar_parse_release": ([_P], None),
}

_lib = None


def load() -> C.CDLL:
    """Load libgmask.so (building it first if the sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    if os.environ.get("GMASK_NO_BUILD") != "1":
        from . import build as _build

        try:
            _build.build()
        except RuntimeError:
            if not LIB_PATH.exists():
                raise
    if not LIB_PATH.exists():
        raise ImportError(f"libgmask.so not built at {LIB_PATH}; run paper_2411_15100_b200/build.py")
    lib = C.CDLL(str(LIB_PATH))
    for name, (args, res) in _SIGNATURES.items():
        if os.environ.get("GMASK_LIB") and not hasattr(lib, name):
            continue  # diagnostics: an older library variant (tools/ab_libs.sh)
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    if os.environ.get("GMASK_APPLY_BLEND") and hasattr(lib, "gm_apply_set_blend"):
        lib.gm_apply_set_blend(int(os.environ["GMASK_APPLY_BLEND"]))  # K0, and the fused apply of caches built later
    return lib


def exported_symbols() -> list:
    return list(_SIGNATURES)


def check(status: int, what: str = ""):
    if status != GM_OK:
        msg = load().gm_last_error().decode(errors="replace")
        raise GmaskError(status, f"{what}: {msg}" if what else msg)


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2411_15100_b200 needs a CUDA device (sm_100a); there is no CPU fallback"
        )


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
