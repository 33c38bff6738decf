"""Node-range-partitioned multi-GPU T-CSR build (MAG-scale).

One process per GPU.  Rank r holds the r-th contiguous chunk of the event stream (rank order
= stream order).  The build is one exchange step:

  1. degrees      tgfx_degree_hist_device on the local chunk, all_reduce(SUM)   [NCCL]
  2. ownership    rank d owns the global entry positions [d*m/N, (d+1)*m/N) exactly
                  (plan_entry_ranges): contiguous node ranges, plus the <= N-1 nodes a cut
                  falls inside (the Zipf hubs), split by entry position -- the positions of a
                  chunk's entries of such a node come from a tiny all-gather of their per-chunk
                  counts (the node's entries in earlier chunks precede this chunk's)
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

Rank r's columns are bit-identical to the entries [P_r, P_{r+1}) of the single-GPU build
(tests/test_gpu_partition.py), because every node's entries arrive in emission order; every
rank holds m/N entries (+-1) whatever the degree skew.  The compute is libtgfx's kernels; torch supplies device memory, small
metadata arithmetic (cumsum / searchsorted on V counters) and torch.distributed.
"""
from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

from ._lib import TGFX_TRUSTED, check, lib


def plan_entry_ranges(deg: torch.Tensor, world: int):
    """Balanced ownership by GLOBAL entry position: rank d owns [P[d], P[d+1]), P[d] = d*m/world.
    Returns (P [world+1], bounds [world+1], split nodes [ns], indptr [V+1]): bounds[d] = the
    node containing position P[d] (the first node rank d touches); a node whose slice has a
    cut strictly inside is split between ranks (ns <= world-1), every other node belongs to
    the rank whose node range [bounds[d], bounds[d+1]) holds it."""
    V = deg.numel()
    dev = deg.device
    indptr = torch.zeros(V + 1, dtype=torch.int64, device=dev)
    if V:
        torch.cumsum(deg.to(torch.int64), 0, out=indptr[1:])
    m = int(indptr[-1].item())
    P = torch.tensor([m * d // world for d in range(world + 1)], dtype=torch.int64, device=dev)
    # node containing position P[d]: the first node whose slice ends after P[d]
    c = torch.searchsorted(indptr[1:], P, right=True) if V else P * 0
    bounds = torch.clamp(c, 0, V)
    bounds[0] = 0
    bounds[world] = V
    inner = bounds[1:world]
    split = inner[(inner < V) & (indptr[torch.clamp(inner, max=V)] < P[1:world])] if world > 1 \
        else inner
    return P, bounds, torch.unique(split), indptr


def plan_bounds(deg: torch.Tensor, world: int) -> torch.Tensor:
    """Node-range bounds of plan_entry_ranges (kept for callers that only need them)."""
    return plan_entry_ranges(deg, world)[1]


def plan_offsets(counts: torch.Tensor, world: int):
    """counts[nw, world] per-warp bucket sizes -> (offsets[nw, world] first slot of each warp's
    records in the send buffer, send_sizes[world]).  Buckets are laid out by destination
    rank, warps (stream order) inside a bucket."""
    totals = counts.sum(0)
    base = torch.cumsum(totals, 0) - totals
    offs = torch.cumsum(counts, 0) - counts + base[None, :]
    return offs.contiguous(), totals


def split_counts_per_rank(scounts, gp, P, world):
    """Per-warp entries of the split nodes per destination rank: split node i's entries of
    warp w occupy global positions [gp[i] + occ[w, i], + scounts[w, i]); rank d takes their
    overlap with [P[d], P[d+1]).  Returns (occ [nw, 7], per_rank [nw, world])."""
    occ = torch.cumsum(scounts, 0) - scounts
    start = gp[None, :] + occ
    end = start + scounts
    per_rank = torch.stack([(torch.clamp(torch.minimum(end, P[d + 1]) -
                                         torch.maximum(start, P[d]), min=0)).sum(1)
                            for d in range(world)], 1)
    return occ.contiguous(), per_rank


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

    deg_local = torch.empty(max(num_nodes, 1), dtype=torch.int64, device=dev)
    check(L.tgfx_degree_hist_device(_ptr(ev_local), n, num_nodes, rev, _ptr(deg_local), s))
    deg_local = deg_local[:num_nodes]
    deg = deg_local.clone()
    _all_reduce(deg, exchange_on_host)
    P, bounds, split, indptr = plan_entry_ranges(deg, world)
    ns = int(split.numel())
    # this chunk's first entry of each split node: indptr + the node's entries in earlier chunks
    sdeg = torch.zeros(8, dtype=torch.int64, device=dev)
    if ns:
        sdeg[:ns] = deg_local[split]
    gathered = torch.empty(world * 8, dtype=torch.int64, device=dev)
    _all_gather(gathered, sdeg, exchange_on_host)
    before = gathered.view(world, 8)[:rank].sum(0)[:7]
    gp = torch.zeros(7, dtype=torch.int64, device=dev)
    if ns:
        gp[:ns] = indptr[split] + before[:ns]
    tab = torch.zeros(24, dtype=torch.int64, device=dev)
    tab[0] = ns
    tab[1:1 + ns] = split
    tab[8:15] = gp
    tab[15:15 + world + 1] = P

    nw = int(L.tgfx_partition_warps(max(n, 1)))
    counts = torch.zeros((nw, world), dtype=torch.int64, device=dev)
    scounts = torch.zeros((nw, 7), dtype=torch.int64, device=dev)
    if n:
        check(L.tgfx_partition_count_device(_ptr(ev_local), n, rev, _ptr(bounds), world, nw,
                                            _ptr(tab), _ptr(counts), _ptr(scounts), s))
    occ, per_rank = split_counts_per_rank(scounts, gp, P, world)
    offs, send = plan_offsets(counts + per_rank, world)
    sent = int(send.sum().item())
    records = torch.empty(max(sent, 1) * 32, dtype=torch.uint8, device=dev)
    check(L.tgfx_partition_scatter_device(_ptr(ev_local), n, rev, _ptr(bounds), world, nw,
                                          _ptr(tab), _ptr(occ), _ptr(offs), _ptr(records), s))

    recv_counts = torch.empty_like(send)
    _all_to_all(recv_counts, send, None, None, exchange_on_host)
    recv = torch.empty(max(int(recv_counts.sum().item()), 1) * 32, dtype=torch.uint8, device=dev)
    _all_to_all(recv, records[:sent * 32], (recv_counts * 32).tolist(), (send * 32).tolist(),
                exchange_on_host)
    n_recv = int(recv_counts.sum().item())

    Ph = P.tolist()
    lo = int(bounds[rank].item())
    # last node this rank touches: the one holding its last position P[rank+1] - 1
    hi = int(torch.searchsorted(indptr[1:], P[rank + 1] - 1, right=True).item()) + 1 \
        if Ph[rank + 1] > Ph[rank] else lo
    h = C.c_void_p()
    check(L.tgfx_build_range_device(_ptr(recv), n_recv, max(hi - lo, 0), num_nodes, num_edges, s,
                                    0, C.byref(h)))
    local = TCsr(h.value)
    out = dict(local=local, bounds=bounds, degrees=deg, range=(lo, hi), positions=P,
               split_nodes=split, sent_records=sent, received_records=n_recv)
    if replicate:
        out["full"] = _replicate(local, deg, P, num_nodes, num_edges, reverse, exchange_on_host)
    return out


def replicate(part: dict, num_nodes: int, num_edges: int, reverse: bool,
              exchange_on_host: bool = False):
    """The full T-CSR on every rank from a build_partitioned(replicate=False) result."""
    return _replicate(part["local"], part["degrees"], part["positions"], num_nodes, num_edges,
                      reverse, exchange_on_host)


def _replicate(local, deg, P, num_nodes, num_edges, reverse, on_host):
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
    starts = P.tolist()  # each owner's global entry range [P[d], P[d+1])
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


def _all_gather(out, inp, on_host):
    if on_host:
        parts = [torch.empty(inp.shape, dtype=inp.dtype) for _ in range(dist.get_world_size())]
        dist.all_gather(parts, inp.cpu())
        out.copy_(torch.cat(parts))
    else:
        dist.all_gather_into_tensor(out, inp)


def _broadcast(t, src, on_host):
    if on_host:
        c = t.cpu()
        dist.broadcast(c, src)
        t.copy_(c)
    else:
        dist.broadcast(t, src)
