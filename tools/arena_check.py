import os, sys
sys.path.insert(0, os.getcwd())
os.environ["GMASK_NO_BUILD"] = "1"
import torch, bench
import paper_2411_15100_b200 as gm
from paper_2411_15100_b200 import _lib
from paper_2411_15100_b200.engine import get_pool
from paper_2411_15100_b200.matcher import batch_step
torch.cuda.set_device(0)
vocab = gm.synth_vocab(128256)
info = gm.TokenizerInfo.from_vocabulary(vocab)
compiled = gm.GrammarCompiler(info).compile_builtin_json_grammar()
pool = get_pool(); lib = _lib.load()
print("arena after compile", lib.gm_pool_arena_used(pool.handle), "mask+1", 1 << 24)
B = 128
ms = [gm.GrammarMatcher(compiled, max_rollback_tokens=1) for _ in range(B)]
slots = torch.tensor([m.slot for m in ms], dtype=torch.int32, device="cuda")
print("arena after reset", lib.gm_pool_arena_used(pool.handle))
W = (vocab.size + 31) // 32
bm = torch.empty((B, W), dtype=torch.int32, device="cuda"); acc = torch.empty(B, dtype=torch.uint8, device="cuda")
structural = torch.from_numpy(bench.structural_flags(vocab, bench.STRUCTURAL)).cuda()
rows = torch.arange(B, device="cuda")
toks = None
for s in range(200):
    batch_step(pool, slots, toks, acc if toks is not None else None, bm, None, recycle=True)
    toks = bench.sample_tokens(bench.unpack_allowed(bm, vocab.size), structural, s, rows).to(torch.int32)
    if s in (10, 50, 199): print("step", s, "arena", lib.gm_pool_arena_used(pool.handle))
