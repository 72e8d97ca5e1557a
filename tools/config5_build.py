"""BASELINE config 5's cache build, both strategies, on the ranks of one
torchrun job (or one process):

* per-rank: each rank compiles only the schemas of the requests it serves
  (schemas[rank::world]) — no exchange (what bench_config5.py runs);
* sharded: every rank ends with ALL schemas compiled, the host front end
  dealt over the ranks + tables exchanged, all (schema, position) pairs dealt
  by estimated cost + one all-gather of the rows
  (engine.compile_many_on_device).

Checks that both give identical caches and prints one JSON line (rank 0):
per-rank ms, sharded phase ms, bytes all-gathered per rank.

    python tools/config5_build.py --schemas 128
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/config5_build.py --backend gloo
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--schemas", type=int, default=128)
    ap.add_argument("--vocab", type=int, default=128256)
    ap.add_argument("--backend", default="nccl")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % torch.cuda.device_count())
    group = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group(args.backend)
        group = dist.group.WORLD
    import paper_2411_15100_b200 as gm
    from bench_config5 import mutate_schema
    from paper_2411_15100_b200.engine import DeviceVocab, compile_many_on_device, compile_on_device
    from paper_2411_15100_b200.schema import schema_to_grammar_text

    vocab = gm.synth_vocab(args.vocab)
    dv = DeviceVocab(vocab)
    texts = [schema_to_grammar_text(json.dumps(mutate_schema(i))) for i in range(args.schemas)]
    compile_on_device(texts[0], dv)  # warm-up (kernel attributes, allocator)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mine = {i: compile_on_device(texts[i], dv) for i in range(rank, len(texts), world)}
    torch.cuda.synchronize()
    per_rank_ms = (time.perf_counter() - t0) * 1e3
    if group is not None:
        torch.distributed.barrier()
    all_c, st = compile_many_on_device(texts, dv, group=group)
    same = True
    for i, c in mine.items():
        a, b = c.cache.export(), all_c[i].cache.export()
        same &= bool(torch.equal(a[0], b[0]) and (a[1] == b[1]).all() and (a[2] == b[2]).all())
    rows_bytes = sum(int(c.grammar.n_keys) for c in all_c) * dv.words * 4
    out = {"schemas": args.schemas, "world": world, "backend": args.backend if world > 1 else None,
           "per_rank_compile_ms": per_rank_ms, "per_rank_schemas": len(mine),
           "sharded": st, "caches_identical": same, "all_rows_bytes": rows_bytes,
           "note": "per-rank: each rank compiles the schemas it serves (no exchange); sharded: every rank holds "
                   "all schemas' caches (positions dealt by cost + one all-gather)"}
    if group is not None:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    if rank == 0:
        print(json.dumps(out))


if __name__ == "__main__":
    main()
