"""K0 apply parity: exact vs torch.where(bit, logits, -inf) (the
reference has no apply; XGrammar's semantics, xgrammar/matcher.py:58-142)."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _unpack(bitmask, vocab):
    bits = (bitmask.unsqueeze(-1) >> torch.arange(32, device=bitmask.device, dtype=torch.int32)) & 1
    return bits.reshape(bitmask.shape[0], -1)[:, :vocab].bool()


def _expect(logits, bitmask, vocab, rows=None):
    out = logits.clone()
    allowed = _unpack(bitmask, vocab)
    sel = range(logits.shape[0]) if rows is None else rows
    for r in sel:
        out[r, :vocab] = torch.where(allowed[r], logits[r, :vocab], torch.tensor(float("-inf"), dtype=logits.dtype, device=logits.device))
    return out


@pytest.mark.parametrize("dtype", [torch.float32, torch.float16, torch.bfloat16])
@pytest.mark.parametrize("vocab", [1, 31, 32, 33, 1000, 32000, 128256, 128257])
def test_apply_exact(dtype, vocab):
    from paper_2411_15100_b200 import apply_token_bitmask_inplace

    g = torch.Generator(device="cuda").manual_seed(vocab)
    B = 7
    W = (vocab + 31) // 32
    logits = torch.randn(B, vocab, device="cuda", dtype=torch.float32, generator=g).to(dtype)
    bitmask = torch.randint(-2**31, 2**31 - 1, (B, W), device="cuda", dtype=torch.int32, generator=g)
    bitmask[1] = -1
    bitmask[2] = 0
    want = _expect(logits, bitmask, vocab)
    apply_token_bitmask_inplace(logits, bitmask)
    assert torch.equal(logits.view(torch.int8 if dtype == torch.float32 else torch.int8), want.view(torch.int8))


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_apply_indices_padding_and_strides(dtype):
    from paper_2411_15100_b200 import apply_token_bitmask_inplace

    g = torch.Generator(device="cuda").manual_seed(5)
    vocab, padded = 1000, 1024 + 3  # padded logits, odd stride -> unaligned path
    base = torch.randn(6, padded, device="cuda", generator=g).to(dtype)
    bitmask = torch.randint(-2**31, 2**31 - 1, (6, 40), device="cuda", dtype=torch.int32, generator=g)
    want = _expect(base, bitmask, vocab, rows=[1, 4])
    logits = base.clone()
    apply_token_bitmask_inplace(logits, bitmask, vocab_size=vocab, indices=[1, 4])
    assert torch.equal(logits.view(torch.int8), want.view(torch.int8))
    # columns >= vocab are untouched
    assert torch.equal(logits[:, vocab:].view(torch.int8), base[:, vocab:].view(torch.int8))


def test_apply_rejects_cpu():
    from paper_2411_15100_b200 import apply_token_bitmask_inplace

    with pytest.raises(RuntimeError):
        apply_token_bitmask_inplace(torch.zeros(1, 32), torch.zeros(1, 1, dtype=torch.int32))
