"""Asynchronous device-pointer API over libtgfx (include/tgfx.h *_device calls).

PyTorch is plumbing here: it owns the big device buffers (events, queries, outputs) and
supplies the CUDA stream; every computation is a libtgfx kernel launched on
torch.cuda.current_stream().  Used by bench.py and the GPU tests.
"""
from __future__ import annotations

import ctypes as C

import torch

from ._lib import TGFX_INDEX64, TGFX_TRUSTED, check, lib
from .tgformer import TCsr, _strategy_code

EVENT_BYTES = 32


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _p(t):
    return C.c_void_p(0 if t is None else t.data_ptr())


class _CAI:
    """__cuda_array_interface__ wrapper so torch can view library-owned device memory."""

    def __init__(self, ptr, n, typestr, owner):
        self.__cuda_array_interface__ = dict(shape=(n,), typestr=typestr, data=(ptr, False),
                                             version=3, strides=None)
        self._owner = owner


def random_stream(num_edges, num_nodes, seed, zipf=1.2, stream=None):
    """make_random_stream (synthetic.cpp:12-43) generated on the device -> uint8 [E*32]."""
    ev = torch.empty(max(num_edges, 1) * EVENT_BYTES, dtype=torch.uint8, device="cuda")
    check(lib().tgfx_make_random_stream_device(num_edges, num_nodes, seed, zipf, _p(ev),
                                               _stream(stream)))
    return ev[: num_edges * EVENT_BYTES]


def event_view(ev):
    """uint8 [E*32] -> int64 [E, 4] view (edge_id, src, dst, timestamp bits)."""
    return ev.view(torch.int64).view(-1, 4)


def build(ev, num_nodes, reverse=True, trusted=False, stream=None):
    """T-CSR build from device events (uint8 [E*32])."""
    n = ev.numel() // EVENT_BYTES
    h = C.c_void_p()
    check(lib().tgfx_build_device(_p(ev), n, num_nodes, 1 if reverse else 0, _stream(stream),
                                  TGFX_TRUSTED if trusted else 0, C.byref(h)))
    return TCsr(h.value)


def rebuild(g, ev, trusted=True, stream=None):
    """Rebuild g in place from events of the same shape (no allocation)."""
    check(lib().tgfx_rebuild_device(g.handle, _p(ev), _stream(stream),
                                    TGFX_TRUSTED if trusted else 0))


def graph_tensors(g):
    """Zero-copy torch views (indptr, nbr, eid, ts) of the device T-CSR (nbr / eid are
    materialised from the gather records on first request; call again after a rebuild)."""
    ip, nb, ed, ts = g.device_arrays()
    m = g.num_entries()
    mk = lambda p, n, t, dt: torch.as_tensor(_CAI(p, n, t, g), device="cuda")  # noqa: E731
    return (mk(ip, g.num_nodes + 1, "<i8", torch.int64), mk(nb, m, "<i8", torch.int64),
            mk(ed, m, "<i8", torch.int64), mk(ts, m, "<f8", torch.float64))


def make_queries(ev, e0, e1, batch, num_nodes, neg_seed=7, nodes=None, times=None, stream=None):
    """forward_concat query layout (training.cpp:193-209) for events [e0, e1)."""
    q = 3 * (e1 - e0)
    nodes = torch.empty(max(q, 1), dtype=torch.int64, device="cuda") if nodes is None else nodes
    times = torch.empty(max(q, 1), dtype=torch.float64, device="cuda") if times is None else times
    check(lib().tgfx_make_queries_device(_p(ev), e0, e1, batch, num_nodes, neg_seed, _p(nodes),
                                         _p(times), _stream(stream)))
    return nodes[:q], times[:q]


def mix_streams(a, b, c):
    """training.cpp:16-18 (train_epoch's seed derivation), via libtgfx."""
    return int(lib().tgfx_mix_streams(a & (2**64 - 1), b & (2**64 - 1), c & (2**64 - 1)))


def make_train_queries(ev, n, b0, b1, batch_size, neg_per_pos, workers, num_nodes, batch_seed,
                       nodes=None, times=None, stream=None):
    """train_epoch's sample_batch queries for batches [b0, b1) of the n-event training stream
    ev (make_batches negatives, workers shards, forward_concat layout per call), on device."""
    q = (min(n, b1 * batch_size) - b0 * batch_size) * (2 + neg_per_pos)
    nodes = torch.empty(max(q, 1), dtype=torch.int64, device="cuda") if nodes is None else nodes
    times = torch.empty(max(q, 1), dtype=torch.float64, device="cuda") if times is None else times
    check(lib().tgfx_make_train_queries_device(_p(ev), n, b0, b1, batch_size, neg_per_pos, workers,
                                               num_nodes, batch_seed & (2**64 - 1), _p(nodes),
                                               _p(times), _stream(stream)))
    return nodes[:q], times[:q]


def train_calls(n, batch_size, neg_per_pos, workers, cfg_seed, epoch):
    """(offset, size, sample_seed) of every sample_batch call of train_epoch (training.cpp:
    425-446) in the make_train_queries layout."""
    out, off = [], 0
    nb = -(-n // batch_size)
    for step in range(nb):
        bs = min(batch_size, n - step * batch_size)
        m = min(workers, bs)
        for h in range(m):
            pb = (h + 1) * bs // m - h * bs // m
            size = pb * (2 + neg_per_pos)
            out.append((off, size, mix_streams(cfg_seed, epoch * 0x10001 + step, h)))
            off += size
    return out


def alloc_rows(q, l, index64=False, dt32=True, dt64=False):
    it = torch.int64 if index64 else torch.int32
    d = dict(node_index=torch.empty((q, l), dtype=it, device="cuda"),
             edge_index=torch.empty((q, l), dtype=it, device="cuda"),
             valid_len=torch.empty(q, dtype=it, device="cuda"))
    if dt32:
        d["time_delta"] = torch.empty((q, l), dtype=torch.float32, device="cuda")
    if dt64:
        d["time_delta64"] = torch.empty((q, l), dtype=torch.float64, device="cuda")
    return d


def first_bad_word():
    """Device word for sample_assemble(first_bad=...): ~0 = no failing query yet."""
    return torch.full((1,), -1, dtype=torch.int64, device="cuda")


def query_error(nodes, first_bad, stream_base=0, stream=None):
    """Raise the reference's ValidationError if a fused-check call recorded a bad query."""
    check(lib().tgfx_query_error(_p(nodes), stream_base & (2**64 - 1), _p(first_bad),
                                 _stream(stream)))


def sample_assemble(g, nodes, times, k, strategy, seed, l, self_edge_index, out=None,
                    stream_base=0, trusted=False, index64=False, dt64=False, stream=None,
                    first_bad=None):
    """Fused sample_batch + build_sequence_batch into device rows [Q, l].  first_bad: a
    first_bad_word() tensor -> the query node check runs inside the sampler kernel (no
    separate pass, no sync); raise with query_error() before using the rows."""
    q = nodes.numel()
    if out is None:
        out = alloc_rows(q, l, index64=index64, dt64=dt64)
    flags = (TGFX_TRUSTED if trusted else 0) | (TGFX_INDEX64 if index64 else 0)
    if first_bad is not None:
        check(lib().tgfx_sample_assemble_checked_device(
            g.handle, _p(nodes), _p(times), q, k, _strategy_code(strategy), seed & (2**64 - 1),
            stream_base & (2**64 - 1), l, self_edge_index, _p(out["node_index"]),
            _p(out["edge_index"]), _p(out.get("time_delta")), _p(out.get("time_delta64")),
            _p(out["valid_len"]), _p(first_bad), _stream(stream), flags))
        return out
    check(lib().tgfx_sample_assemble_device(
        g.handle, _p(nodes), _p(times), q, k, _strategy_code(strategy), seed & (2**64 - 1),
        stream_base & (2**64 - 1), l, self_edge_index, _p(out["node_index"]),
        _p(out["edge_index"]), _p(out.get("time_delta")), _p(out.get("time_delta64")),
        _p(out["valid_len"]), _stream(stream), flags))
    return out


def sample_assemble_batched(g, nodes, times, batch_q, k, strategy, seeds, l, self_edge_index,
                            out=None, trusted=False, index64=False, dt64=False, stream=None):
    """One launch for many forward_concat batches of batch_q queries; batch b uses seeds[b]
    (int64/uint64 device tensor) -- equal to one sample_assemble call per batch."""
    q = nodes.numel()
    if out is None:
        out = alloc_rows(q, l, index64=index64, dt64=dt64)
    flags = (TGFX_TRUSTED if trusted else 0) | (TGFX_INDEX64 if index64 else 0)
    check(lib().tgfx_sample_assemble_batched_device(
        g.handle, _p(nodes), _p(times), q, batch_q, k, _strategy_code(strategy), _p(seeds), l,
        self_edge_index, _p(out["node_index"]), _p(out["edge_index"]), _p(out.get("time_delta")),
        _p(out.get("time_delta64")), _p(out["valid_len"]), _stream(stream), flags))
    return out


def sample_batch(g, nodes, times, k, strategy, seed, stream_base=0, trusted=False, stream=None):
    """sample_batch into padded device arrays: counts [Q], nbr/eid/ts [Q, k]."""
    q = nodes.numel()
    counts = torch.empty(max(q, 1), dtype=torch.int64, device="cuda")
    nb = torch.empty((max(q, 1), k), dtype=torch.int64, device="cuda")
    ed = torch.empty((max(q, 1), k), dtype=torch.int64, device="cuda")
    ts = torch.empty((max(q, 1), k), dtype=torch.float64, device="cuda")
    check(lib().tgfx_sample_batch_device(g.handle, _p(nodes), _p(times), q, k,
                                         _strategy_code(strategy), seed & (2**64 - 1),
                                         stream_base & (2**64 - 1), _p(counts), _p(nb), _p(ed),
                                         _p(ts), _stream(stream),
                                         TGFX_TRUSTED if trusted else 0))
    return counts[:q], nb[:q], ed[:q], ts[:q]


def two_hop(g, roots, times, k1, k2, strategy, seed, l, self_edge_index, seed2=None, out=None,
            trusted=False, stream=None):
    q = roots.numel()
    if out is None:
        out = dict(h1=alloc_rows(q, l), h2=alloc_rows(q * k1, l))
    h1, h2 = out["h1"], out["h2"]
    check(lib().tgfx_sample_two_hop_device(
        g.handle, _p(roots), _p(times), q, k1, k2, _strategy_code(strategy), seed,
        seed if seed2 is None else seed2, l, self_edge_index, _p(h1["node_index"]),
        _p(h1["edge_index"]), _p(h1["time_delta"]), _p(h1["valid_len"]), _p(h2["node_index"]),
        _p(h2["edge_index"]), _p(h2["time_delta"]), _p(h2["valid_len"]), _stream(stream),
        TGFX_TRUSTED if trusted else 0))
    return out



_DT = {torch.float32: 0, torch.float64: 1, torch.bfloat16: 2}


def assemble_inputs(rows, node_table, edge_table, omega, phi, concat=False, z_dtype=torch.float32,
                    trusted=False, stream=None):
    """tgf::assemble_inputs (proj/src/attention.cpp:414-451) on the device: the sampler's rows
    (dict with node_index, edge_index, valid_len and time_delta or time_delta64) ->
    z [q*l, d] with d = d_t (sum) or d_v + d_e + d_t (concat)."""
    ni, ei, vl = rows["node_index"], rows["edge_index"], rows["valid_len"]
    dt = rows.get("time_delta64", rows.get("time_delta"))
    q, l = ni.shape
    d_v, d_e, d_t = node_table.shape[1], edge_table.shape[1], omega.numel()
    d = d_v + d_e + d_t if concat else d_t
    z = torch.empty((q * l, d), dtype=z_dtype, device="cuda")
    om = omega.to(torch.float64).contiguous()
    ph = phi.to(torch.float64).contiguous()
    check(lib().tgfx_assemble_inputs_device(
        q, l, _p(ni), _p(ei), _p(dt), _p(vl), 1 if ni.dtype == torch.int64 else 0, _DT[dt.dtype],
        _p(node_table), node_table.shape[0], _p(edge_table), edge_table.shape[0],
        _DT[node_table.dtype], _p(om), _p(ph), d_v, d_e, d_t, 1 if concat else 0, _p(z),
        _DT[z_dtype], _stream(stream), TGFX_TRUSTED if trusted else 0))
    return z


def sample_inputs(g, nodes, times, k, strategy, seed, l, self_edge_index, node_table, edge_table,
                  omega, phi, concat=False, z_dtype=torch.float32, stream_base=0, trusted=False,
                  stream=None):
    """forward_concat's sample_batch + build_sequence_batch + assemble_inputs in one call
    (tgfx_sample_inputs_device): -> (z [q*l, d], valid_len int32 [q])."""
    q = nodes.numel()
    d_v, d_e, d_t = node_table.shape[1], edge_table.shape[1], omega.numel()
    d = d_v + d_e + d_t if concat else d_t
    z = torch.empty((max(q * l, 1), d), dtype=z_dtype, device="cuda")
    vl = torch.empty(max(q, 1), dtype=torch.int32, device="cuda")
    om = omega.to(torch.float64).contiguous()
    ph = phi.to(torch.float64).contiguous()
    check(lib().tgfx_sample_inputs_device(
        g.handle, _p(nodes), _p(times), q, k, _strategy_code(strategy), seed & (2**64 - 1),
        stream_base & (2**64 - 1), l, self_edge_index, _p(node_table), node_table.shape[0],
        _p(edge_table), edge_table.shape[0], _DT[node_table.dtype], _p(om), _p(ph), d_v, d_e,
        d_t, 1 if concat else 0, _p(z), _DT[z_dtype], _p(vl), _stream(stream),
        TGFX_TRUSTED if trusted else 0))
    return z[:q * l], vl[:q]
