"""Multi-GPU plumbing for the hot path (one process per GPU, torch.distributed).

The sampler shards by query: each rank takes whole forward_concat batches
([src | dst | neg] x B, proj/src/training.cpp:193-209) and samples them against its own
replica of the T-CSR.  Uniform sampling draws from CounterRng(seed, stream) with stream = the
query's index inside its logical sample_batch call (proj/src/sampler.cpp:100-101); a rank
passes stream_base = the global index of its first query, so the rows a rank produces are
bit-identical to the rows one GPU would produce for the same queries, at any world size.
No collective touches the data path; the only collective is the timing reduction (max over
ranks), as the measurement rules require.

Two plans:
  * strong (fixed total work): contiguous whole-batch query ranges of one pass (shard_range);
  * weak (fixed work per rank, bench.py's default for N > 1): every rank runs a full pass
    over the stream with its own negatives (neg_seed + rank), i.e. N data-parallel workers.
"""
from __future__ import annotations

import os
from dataclasses import dataclass


@dataclass(frozen=True)
class Dist:
    world: int
    rank: int
    local: int


def dist_env() -> Dist:
    """RANK / WORLD_SIZE / LOCAL_RANK from the torchrun environment (defaults: one process)."""
    return Dist(int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
                int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(num_queries: int, batch_queries: int, world: int, rank: int):
    """Contiguous [lo, hi) query range of `rank`, cut at whole-batch boundaries so no
    forward_concat batch straddles two ranks; ranges partition [0, num_queries) in rank order."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if batch_queries < 1:
        raise ValueError("batch_queries must be >= 1")
    nb = -(-num_queries // batch_queries)
    b0 = nb * rank // world
    b1 = nb * (rank + 1) // world
    return min(num_queries, b0 * batch_queries), min(num_queries, b1 * batch_queries)


def chunks(lo: int, hi: int, chunk: int):
    """[lo, hi) cut into launches of at most `chunk` queries (stream_base = chunk start)."""
    return [(s, min(hi, s + chunk)) for s in range(lo, hi, chunk)]


def weak_neg_seed(neg_seed: int, rank: int) -> int:
    """Negative-sampling seed of a rank's pass in the weak-scaling plan (rank 0 = the
    single-GPU workload)."""
    return neg_seed + rank


def max_over_ranks(values, device=None):
    """Element-wise max of a list of floats over all ranks (identity without a process
    group).  Used for device-timed step times: the job is as slow as its slowest rank."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(values)
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def sum_over_ranks(values, device=None):
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(values)
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.tolist()
