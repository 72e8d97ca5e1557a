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


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("policy", [0, 1, 528, 0x0F10])
@pytest.mark.parametrize("vocab", [128256, 32011])
def test_apply_mixed_chunk_policy_exact(dtype, policy, vocab):
    """K0's runtime mixed-chunk policy (gm_apply_set_blend): element stores,
    blend always, the default and a strict threshold give the same exact
    result on masks with dense, sparse and heavily masked mixed chunks, also
    with a ragged last word; logits past the vocabulary and rows not listed
    stay untouched."""
    from paper_2411_15100_b200 import _lib, apply_token_bitmask_inplace

    lib = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(policy + vocab)
    B = 9
    W = (vocab + 31) // 32
    width = (vocab + 7) // 8 * 8 + 8  # 16-byte aligned rows (the tiled kernel), columns past the vocabulary
    logits = torch.randn(B, width, device="cuda", generator=g).to(dtype)
    bm = torch.randint(-2**31, 2**31 - 1, (B, W), device="cuda", dtype=torch.int32, generator=g)  # dense mixed
    bm[1] = bm[1] | 0x7F7F7F7F        # mixed chunks with one masked element
    bm[2] = bm[2] & 0x01010101        # heavily masked mixed chunks
    bm[3, ::2] = -1                   # bimodal words
    bm[3, 1::2] = 0
    bm[4] = -1
    bm[5] = 0
    want = _expect(logits, bm, vocab, rows=[0, 1, 2, 3, 4, 5, 7])
    old = lib.gm_apply_set_blend(policy)
    try:
        y = logits.clone()
        apply_token_bitmask_inplace(y, bm, vocab_size=vocab, indices=[0, 1, 2, 3, 4, 5, 7])
    finally:
        lib.gm_apply_set_blend(old)
    assert torch.equal(y.view(torch.int8), want.view(torch.int8))
