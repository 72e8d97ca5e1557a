"""Token bitmask helpers: allocation and the K0 apply kernel.

Signatures follow XGrammar 0.2.0 (xgrammar/matcher.py:15-188), the names
`north_star` asks for.  Differences, all deliberate:

* ``allocate_token_bitmask`` allocates on the current CUDA device (the fill
  kernel writes the mask straight into HBM; XGrammar fills on the CPU).
* the fill zeroes bits >= vocab_size like grammask's TokenMask._trim
  (REF matcher.py:57-60).
"""

from __future__ import annotations

import math
from typing import List, Optional, Sequence, Tuple, Union

import torch

from . import _lib

bitmask_dtype = torch.int32

_DTYPES = {torch.float32: _lib.GM_DTYPE_F32, torch.float16: _lib.GM_DTYPE_F16, torch.bfloat16: _lib.GM_DTYPE_BF16}


def get_bitmask_shape(batch_size: int, vocab_size: int) -> Tuple[int, int]:
    """(batch_size, ceil(vocab_size / 32)) — XGrammar matcher.py:19-21."""
    return (batch_size, math.ceil(vocab_size / 32))


def allocate_token_bitmask(batch_size: int, vocab_size: int, device=None) -> torch.Tensor:
    """int32 bitmask of shape get_bitmask_shape(...), all tokens allowed (-1).

    XGrammar allocates on the CPU (matcher.py:27-50); this build allocates on
    ``device`` (default: the current CUDA device) because the mask is filled
    and consumed in HBM."""
    if device is None:
        _lib.require_cuda()
        device = torch.device("cuda", torch.cuda.current_device())
    return torch.full(get_bitmask_shape(batch_size, vocab_size), -1, dtype=bitmask_dtype, device=device)


def reset_token_bitmask(bitmask: torch.Tensor) -> None:
    bitmask.fill_(-1)


def _as_index_tensor(indices, device) -> Optional[torch.Tensor]:
    if indices is None:
        return None
    if isinstance(indices, torch.Tensor):
        return indices.to(device=device, dtype=torch.int32)
    return torch.tensor(list(indices), dtype=torch.int32, device=device)


def apply_token_bitmask_inplace(
    logits: torch.Tensor,
    bitmask: torch.Tensor,
    *,
    vocab_size: Optional[int] = None,
    indices: Optional[Union[Sequence[int], torch.Tensor]] = None,
    backend: str = "auto",
    stream=None,
) -> None:
    """Set logits[r, j] = -inf wherever bit j of bitmask[r] is 0 (K0 kernel).

    Semantics of XGrammar's apply (matcher.py:58-142): vocab_size defaults to
    min(logits.shape[-1], 32 * bitmask.shape[-1]); ``indices`` selects rows;
    allowed logits are left untouched bit for bit.  ``backend`` is accepted for
    signature compatibility and ignored: there is exactly one implementation,
    the sm_100a kernel.  CPU tensors raise (no CPU fallback)."""
    del backend
    if logits.device != bitmask.device:
        raise ValueError(
            f"logits and bitmask should be on the same device. But got logits.device: {logits.device}, "
            f"bitmask.device: {bitmask.device}"
        )
    if logits.device.type != "cuda":
        raise RuntimeError("apply_token_bitmask_inplace runs on CUDA tensors only (no CPU fallback)")
    if bitmask.dtype != torch.int32:
        raise TypeError("bitmask must be of type int32")
    if logits.dtype not in _DTYPES:
        raise TypeError(f"unsupported logits dtype {logits.dtype}")
    lg = logits if logits.dim() == 2 else logits.view(1, -1)
    bm = bitmask if bitmask.dim() == 2 else bitmask.view(1, -1)
    if lg.stride(-1) != 1 or bm.stride(-1) != 1:
        raise ValueError("logits and bitmask must be contiguous in the vocabulary dimension")
    detected = min(lg.shape[-1], bm.shape[-1] * 32)
    if vocab_size is None:
        vocab_size = detected
    elif vocab_size > detected:
        raise ValueError(f"vocab_size {vocab_size} is larger than the detected vocab_size {detected}")
    idx = _as_index_tensor(indices, lg.device)
    n_rows = idx.numel() if idx is not None else lg.shape[0]
    if idx is None and bm.shape[0] < n_rows:
        raise ValueError("bitmask has fewer rows than logits")
    lib = _lib.load()
    _lib.check(
        lib.gm_apply_inplace(
            lg.data_ptr(), _DTYPES[lg.dtype], n_rows, vocab_size, lg.stride(0), bm.data_ptr(), bm.stride(0),
            idx.data_ptr() if idx is not None else None, _lib.stream_ptr(stream),
        ),
        "apply_token_bitmask_inplace",
    )
