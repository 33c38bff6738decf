"""Multi-process (gloo, world_size 2, CPU) checks of the N>1 host logic in
paper_2409_05477_b200/shard.py.

The GPU path cannot run here, so the per-rank compute is the oracle (the CPU restatement of
the reference -- this is a test, the checker is allowed).  What is under test is the plan:
whole-batch contiguous query shards + stream_base must give, concatenated in rank order,
exactly the single-process rows (recent and uniform), and the timing reduction must be the
max over ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2409_05477_b200 import shard


def test_shard_ranges_partition_whole_batches():
    for q, b, w in ((1800 * 263, 1800, 8), (12000 * 7 + 5, 12000, 4), (10, 3, 4), (0, 5, 2)):
        ranges = [shard.shard_range(q, b, w, r) for r in range(w)]
        assert ranges[0][0] == 0 and ranges[-1][1] == q
        for (a0, a1), (b0, _) in zip(ranges, ranges[1:]):
            assert a1 == b0 and a0 <= a1
        for lo, hi in ranges:
            assert lo % b == 0 and (hi % b == 0 or hi == q)
    with pytest.raises(ValueError):
        shard.shard_range(10, 3, 2, 2)
    assert shard.chunks(5, 17, 5) == [(5, 10), (10, 15), (15, 17)]
    assert shard.weak_neg_seed(7, 0) == 7 and shard.weak_neg_seed(7, 3) == 10


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        E, V, B = 30000, 400, 600
        ev = O.make_random_stream(E, V, 42)
        g = O.build(ev, V, True)
        nodes, times = O.make_queries(ev, 0, E, B, V)
        lo, hi = shard.shard_range(len(nodes), 3 * B, world, rank)
        rows = {}
        for strat, k, l in (("recent", 10, 11), ("random", 20, 21)):
            parts = []
            for s, e in shard.chunks(lo, hi, 7 * 3 * B):
                r = O.sample_assemble(g, nodes[s:e], times[s:e], k, strat, 9, l, E + 1,
                                      stream_base=s)
                parts.append(r["node_index"])
            mine = np.concatenate(parts) if parts else np.zeros((0, l), np.int64)
            gathered = [None] * world
            dist.all_gather_object(gathered, mine)
            rows[strat] = np.concatenate(gathered)
        t = shard.max_over_ranks([1.0 + rank, 5.0 - rank])
        s = shard.sum_over_ranks([float(hi - lo)])
        if rank == 0:
            np.savez(os.path.join(out_dir, "rows.npz"), **rows, t=np.array(t), s=np.array(s))
    finally:
        dist.destroy_process_group()


def test_sharded_sampling_equals_single_process(tmp_path):
    from oracle import oracle as O
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    got = np.load(os.path.join(tmp_path, "rows.npz"))
    E, V, B = 30000, 400, 600
    ev = O.make_random_stream(E, V, 42)
    g = O.build(ev, V, True)
    nodes, times = O.make_queries(ev, 0, E, B, V)
    for strat, k, l in (("recent", 10, 11), ("random", 20, 21)):
        want = O.sample_assemble(g, nodes, times, k, strat, 9, l, E + 1)["node_index"]
        assert np.array_equal(got[strat], want), strat
    assert got["t"].tolist() == [2.0, 5.0]          # max over ranks, element-wise
    assert got["s"].tolist() == [float(len(nodes))]  # shards cover every query once


def test_partition_plan_balances_entries():
    """plan_bounds / plan_offsets (partition.py), pure host arithmetic."""
    from paper_2409_05477_b200 import partition as P
    deg = torch.tensor([50, 1, 1, 1, 30, 2, 2, 2, 2, 9], dtype=torch.int64)
    for world in (1, 2, 3, 4, 8):
        b = P.plan_bounds(deg, world)
        assert b[0] == 0 and b[-1] == len(deg) and bool((b[1:] >= b[:-1]).all())
        assert len(b) == world + 1
    b = P.plan_bounds(deg, 2)
    assert b.tolist() == [0, 1, 10]  # the hub (50 of 100 entries) fills rank 0
    counts = torch.tensor([[3, 1], [0, 2], [4, 0]], dtype=torch.int64)
    offs, send = P.plan_offsets(counts, 2)
    assert send.tolist() == [7, 3]
    assert offs.tolist() == [[0, 7], [3, 8], [3, 10]]
