"""Multi-rank cache-build assembly on CPU with gloo, world size 2:
each rank builds its key block, one all-gather replicates the rows, and the
result equals the single-process build."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2411_15100_b200.engine import shard_range, sharded_rows

N_KEYS, WORDS = 11, 37


def fake_build(lo, n):
    k = torch.arange(lo, lo + n, dtype=torch.int32).view(-1, 1)
    w = torch.arange(WORDS, dtype=torch.int32).view(1, -1)
    return (k * 1000 + w), (k * 7 - w)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        acc, dep = sharded_rows(fake_build, N_KEYS, WORDS, torch.device("cpu"), dist.group.WORLD)
        q.put((rank, acc.numpy().tobytes(), dep.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


def test_shard_ranges_cover_keys():
    for n in (0, 1, 5, 46, 91):
        for world in (1, 2, 3, 8):
            got = [shard_range(n, world, r)[:2] for r in range(world)]
            covered = [k for lo, hi in got for k in range(lo, hi)]
            assert covered == list(range(n))


@pytest.mark.parametrize("world", [2])
def test_sharded_rows_gloo_equals_single(world):
    want_acc, want_dep = fake_build(0, N_KEYS)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=90) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for _, acc, dep in results:
        assert acc == want_acc.numpy().tobytes()
        assert dep == want_dep.numpy().tobytes()
