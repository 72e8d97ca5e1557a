"""Multi-rank cache-build assembly on CPU with gloo, world size 2:
keys are dealt round-robin in decreasing order of estimated cost, each rank
builds its keys, one all-gather replicates the rows, and every rank puts
them back in key order — equal to the single-process build."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import numpy as np

from paper_2411_15100_b200.engine import shard_keys, shard_range, sharded_rows

N_KEYS, WORDS = 11, 37
COSTS = [5, 1, 9, 9, 0, 3, 7, 2, 8, 4, 6]


def fake_build(keys):
    if keys is None:
        keys = range(N_KEYS)
    k = torch.as_tensor(np.asarray(keys, dtype=np.int64)).to(torch.int32).view(-1, 1)
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
        acc, dep = sharded_rows(fake_build, N_KEYS, WORDS, torch.device("cpu"), dist.group.WORLD, COSTS)
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
    want_acc, want_dep = fake_build(range(N_KEYS))
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


def test_shard_keys_cost_sorted_round_robin():
    """Every key exactly once; the most expensive keys are spread over the
    ranks (rank r gets the r-th, (r+G)-th ... most expensive)."""
    for world in (1, 2, 3, 8):
        got = [shard_keys(COSTS, world, r) for r in range(world)]
        flat = sorted(int(k) for g in got for k in g)
        assert flat == list(range(N_KEYS))
        order = np.argsort(-np.asarray(COSTS), kind="stable")
        for r in range(world):
            assert list(got[r]) == list(order[r::world])
    # two-rank split of these costs: [9,9,8,7,6,5,4,3,2,1,0] dealt alternately
    a, b = shard_keys(COSTS, 2, 0), shard_keys(COSTS, 2, 1)
    assert abs(sum(COSTS[k] for k in a) - sum(COSTS[k] for k in b)) <= max(COSTS)


def test_key_costs_rank_string_interior_first():
    """The cost estimate ranks a position that can start any token above a
    structural one that only takes a few bytes (JSON: inside a string vs
    after a value)."""
    from paper_2411_15100_b200.automaton import AutomatonOptions, build_tables_native
    from paper_2411_15100_b200.engine import key_costs
    from paper_2411_15100_b200.grammar import parse_grammar
    from paper_2411_15100_b200.vocab import synth_vocab

    g = parse_grammar('root ::= "{" [a-z]* "}" ","')
    t = build_tables_native(g, AutomatonOptions())
    c = key_costs(t, synth_vocab(4000, profile="mixed"))
    assert len(c) == len(t.cache_keys)
    assert c.max() > 20 * c.min()
