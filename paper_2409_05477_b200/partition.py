"""Node-range-partitioned multi-GPU T-CSR build (MAG-scale).

One process per GPU.  Rank r holds the r-th contiguous chunk of the event stream (rank order
= stream order).  The build is one exchange step:

  1. degrees      tgfx_degree_hist_device on the local chunk, all_reduce(SUM)   [NCCL]
  2. node ranges  contiguous, balanced by entry count (plan_bounds)
  3. partition    tgfx_partition_count/scatter_device: the chunk's entries, stably split into
                  per-owner buckets of 32-byte records (eid, owner-local node, other, t)
  4. exchange     all_to_all of the bucket sizes, then one all_to_all_single of the records
                  [NCCL over NVLink]; received buckets are concatenated in rank order, i.e.
                  in global stream order
  5. local build  tgfx_build_range_device: an ordinary stable build of the owned range
                  (reverse = 0 over the records; neighbour ids stay global)
  6. replicate    (optional) every owner broadcasts its columns into their slice of the full
                  columns on every rank (what query-sharded sampling needs); global indptr =
                  exclusive scan of the all-reduced degrees.

The owned range of rank r is bit-identical to the slices [indptr[b_r], indptr[b_{r+1}]) of the
single-GPU build (tests/test_gpu_partition.py), because every node's entries arrive in
emission order.  The compute is libtgfx's kernels; torch supplies device memory, small
metadata arithmetic (cumsum / searchsorted on V counters) and torch.distributed.
"""
from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

from ._lib import TGFX_TRUSTED, check, lib


def plan_bounds(deg: torch.Tensor, world: int) -> torch.Tensor:
    """Node-range bounds [world+1] (int64): rank d owns nodes [b[d], b[d+1]).  Cuts where the
    exclusive prefix of entries crosses d*m/world, so every rank owns ~m/world entries (a
    single node's slice cannot be split: the Zipf hub bounds the balance)."""
    V = deg.numel()
    csum = torch.cumsum(deg.to(torch.int64), 0)
    m = int(csum[-1].item()) if V else 0
    targets = torch.tensor([m * d // world for d in range(1, world)], dtype=torch.int64,
                           device=deg.device)
    cuts = torch.searchsorted(csum, targets, right=False) + 1 if V else targets * 0
    b = torch.cat([torch.zeros(1, dtype=torch.int64, device=deg.device),
                   torch.clamp(cuts, 0, V),
                   torch.full((1,), V, dtype=torch.int64, device=deg.device)])
    return torch.cummax(b, 0).values  # monotone


def plan_offsets(counts: torch.Tensor, world: int):
    """counts[nw, world] per-warp bucket sizes -> (offsets[nw, world] first slot of each warp's
    records in the send buffer, send_sizes[world]).  Buckets are laid out by destination
    rank, warps (stream order) inside a bucket."""
    totals = counts.sum(0)
    base = torch.cumsum(totals, 0) - totals
    offs = torch.cumsum(counts, 0) - counts + base[None, :]
    return offs.contiguous(), totals


def _ptr(t):
    return C.c_void_p(t.data_ptr())


def _stream(stream):
    return C.c_void_p(stream.cuda_stream if stream is not None else
                      torch.cuda.current_stream().cuda_stream)


def build_partitioned(ev_local: torch.Tensor, num_nodes: int, reverse: bool, num_edges: int,
                      replicate: bool = True, exchange_on_host: bool = False):
    """Partitioned build.  ev_local: this rank's chunk of the stream, uint8 device tensor of
    n*32 bytes (TemporalEvent layout).  Returns dict(local=TCsr of the owned range,
    bounds=[world+1], degrees, full=TCsr replicated on every rank (if replicate)).
    exchange_on_host: stage the all_to_all through host memory (gloo test mode)."""
    from .tgformer import TCsr
    L = lib()
    world, rank = dist.get_world_size(), dist.get_rank()
    dev = ev_local.device
    n = ev_local.numel() // 32
    s = _stream(None)
    rev = 1 if reverse else 0

    deg = torch.empty(max(num_nodes, 1), dtype=torch.int64, device=dev)
    check(L.tgfx_degree_hist_device(_ptr(ev_local), n, num_nodes, rev, _ptr(deg), s))
    deg = deg[:num_nodes]
    _all_reduce(deg, exchange_on_host)
    bounds = plan_bounds(deg, world)

    nw = int(L.tgfx_partition_warps(max(n, 1)))
    counts = torch.zeros((nw, world), dtype=torch.int64, device=dev)
    if n:
        check(L.tgfx_partition_count_device(_ptr(ev_local), n, rev, _ptr(bounds), world, nw,
                                            _ptr(counts), s))
    offs, send = plan_offsets(counts, world)
    sent = int(send.sum().item())
    records = torch.empty(max(sent, 1) * 32, dtype=torch.uint8, device=dev)
    check(L.tgfx_partition_scatter_device(_ptr(ev_local), n, rev, _ptr(bounds), world, nw,
                                          _ptr(offs), _ptr(records), s))

    recv_counts = torch.empty_like(send)
    _all_to_all(recv_counts, send, None, None, exchange_on_host)
    recv = torch.empty(max(int(recv_counts.sum().item()), 1) * 32, dtype=torch.uint8, device=dev)
    _all_to_all(recv, records[:sent * 32], (recv_counts * 32).tolist(), (send * 32).tolist(),
                exchange_on_host)
    n_recv = int(recv_counts.sum().item())

    lo, hi = int(bounds[rank].item()), int(bounds[rank + 1].item())
    h = C.c_void_p()
    check(L.tgfx_build_range_device(_ptr(recv), n_recv, hi - lo, num_nodes, num_edges, s, 0,
                                    C.byref(h)))
    local = TCsr(h.value)
    out = dict(local=local, bounds=bounds, degrees=deg, range=(lo, hi), sent_records=sent)
    if replicate:
        out["full"] = _replicate(local, deg, bounds, num_nodes, num_edges, reverse,
                                 exchange_on_host)
    return out


def replicate(part: dict, num_nodes: int, num_edges: int, reverse: bool,
              exchange_on_host: bool = False):
    """The full T-CSR on every rank from a build_partitioned(replicate=False) result."""
    return _replicate(part["local"], part["degrees"], part["bounds"], num_nodes, num_edges,
                      reverse, exchange_on_host)


def _replicate(local, deg, bounds, num_nodes, num_edges, reverse, on_host):
    """Every rank's owned columns broadcast straight into their slice of the full columns
    (one broadcast per owner and column: no padding to the largest part, no concatenation
    copy), then imported as one device T-CSR per rank (node directory, bucket tables and gather
    records built on the device)."""
    from .device import graph_tensors
    from .tgformer import TCsr
    L = lib()
    world, rank = dist.get_world_size(), dist.get_rank()
    dev = deg.device
    indptr = torch.zeros(num_nodes + 1, dtype=torch.int64, device=dev)
    torch.cumsum(deg, 0, out=indptr[1:])
    m = int(indptr[-1].item())
    starts = indptr[bounds].tolist()  # entry offset of each owner's range, [world + 1]
    _, nb, ed, ts = graph_tensors(local)
    cols = [torch.empty(max(m, 1), dtype=torch.int64, device=dev) for _ in range(3)]
    for col, mine in zip(cols, (nb, ed, ts.view(torch.int64))):
        col[starts[rank]:starts[rank + 1]].copy_(mine)
        for d in range(world):
            if starts[d + 1] > starts[d]:
                _broadcast(col[starts[d]:starts[d + 1]], d, on_host)
    h = C.c_void_p()
    check(L.tgfx_graph_from_device(num_nodes, num_edges, 1 if reverse else 0, m, _ptr(indptr),
                                   _ptr(cols[0]), _ptr(cols[1]), _ptr(cols[2]), _stream(None),
                                   TGFX_TRUSTED, C.byref(h)))
    torch.cuda.synchronize()
    return TCsr(h.value)


# -------------------------------------------------------------------- collectives
def _all_reduce(t, on_host):
    if on_host:
        c = t.cpu()
        dist.all_reduce(c)
        t.copy_(c)
    else:
        dist.all_reduce(t)


def _all_to_all(out, inp, out_splits, in_splits, on_host):
    if on_host:
        o = torch.empty(out.shape, dtype=out.dtype)
        dist.all_to_all_single(o, inp.cpu(), out_splits, in_splits)
        out.copy_(o)
    else:
        dist.all_to_all_single(out, inp, out_splits, in_splits)


def _broadcast(t, src, on_host):
    if on_host:
        c = t.cpu()
        dist.broadcast(c, src)
        t.copy_(c)
    else:
        dist.broadcast(t, src)
