"""The position-sharded cache build for real: two processes on
cuda:0 (gloo, the only backend that takes two ranks on one device) run
compile_on_device(group=WORLD) — K1 over their cost-dealt keys, one
all-gather, reassembly in key order.  The assembled cache must equal the
1-rank build bit for bit (REF SPEC.md:364: a parallel build is identical to
the sequential one) and reproduce the reference's golden masks."""

import hashlib
import os
import socket

import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, fixture):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from workloads import grammar_text, load_fixture, vocab_by_name

        from paper_2411_15100_b200.compat import Matcher, compile_bundle

        fx = load_fixture(fixture)
        vocab = vocab_by_name(fx["vocab"])
        sharded = compile_bundle(grammar_text(fx["grammar"]), vocab, group=dist.group.WORLD)
        single = compile_bundle(grammar_text(fx["grammar"]), vocab)
        a = sharded.compiled.cache.export()
        b = single.compiled.cache.export()
        same = (torch.equal(a[0], b[0]) and (a[1] == b[1]).all() and (a[2] == b[2]).all())
        checked = bad = 0
        if rank == 0:  # the sharded cache serves the reference's masks
            for traj in fx["trajectories"]:
                m = Matcher(sharded, vocab, history_window=1)
                for step, rec in enumerate(traj["masks"]):
                    raw = m.next_token_mask().to_bytes()
                    bad += hashlib.sha256(raw).hexdigest() != rec["sha256"]
                    checked += 1
                    if step >= len(traj["tokens"]) or traj["tokens"][step] == vocab.eos_id:
                        break
                    m.accept_token(traj["tokens"][step])
                m.close()
        q.put((rank, bool(same), checked, bad, sharded.compiled.tables.cache_keys.size))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fixture", ["masks_json_32000_text.json.gz", "masks_schema_32000_text.json.gz"])
def test_two_rank_sharded_compile_equals_single(fixture):
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, fixture)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    for rank, same, checked, bad, n_keys in results:
        assert same, f"rank {rank}: sharded cache differs from the 1-rank build"
        assert n_keys > 1
    assert results[0][2] > 0 and results[0][3] == 0
