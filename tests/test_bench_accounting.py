"""bench.py's byte accounting for the apply roofline (CPU): the algorithmic
count and the 32-byte-sector count of bench.physical_apply_bytes on masks
whose answer is known by hand."""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def test_physical_bytes_by_hand():
    W = 2
    # all masked: mask words + one 32-B write per sector (16 bf16 logits each)
    assert bench.physical_apply_bytes(torch.zeros(1, 1, W, dtype=torch.int32), 64) == 8 + 32 * 4
    # all allowed: the mask words only
    assert bench.physical_apply_bytes(torch.full((1, 1, W), -1, dtype=torch.int32), 64) == 8
    # alternating tokens: every sector mixed (read + write), averaged over steps
    assert bench.physical_apply_bytes(torch.full((3, 1, W), 0x55555555, dtype=torch.int32), 64) == 8 + 64 * 4
    # a ragged vocabulary: the sectors past it are padding, not traffic
    assert bench.physical_apply_bytes(torch.zeros(1, 1, W, dtype=torch.int32), 40) == 8 + 32 * 3
    # fp32 logits: 8 per sector
    assert bench.physical_apply_bytes(torch.zeros(1, 1, 1, dtype=torch.int32), 32, es=4) == 4 + 32 * 4


def test_physical_bytes_bound_the_algorithmic_count():
    g = torch.Generator().manual_seed(3)
    m = torch.randint(-2**31, 2**31 - 1, (2, 4, 100), dtype=torch.int32, generator=g)
    m[:, 1] = 0
    m[:, 2] = -1
    V = 100 * 32
    allowed = bench.unpack_allowed(m.view(-1, 100), V)
    algo = (m.numel() * 4 + 2 * int((~allowed).sum())) / m.shape[0]
    assert bench.physical_apply_bytes(m, V) >= algo
