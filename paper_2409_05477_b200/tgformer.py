"""Host-side mirror of the reference's hot-path API (tgformer, proj/include/tgformer/*.hpp)
over the C ABI (include/tgfx.h).  Same names, argument meaning and error behaviour, so the
parity tests read like the reference's own tests; every computation runs in libtgfx's
sm_100a kernels (no CPU path).

    reference                                  here
    tgf::EventStream      event_stream.hpp:26  EventStream(events, num_nodes)
    tgf::build_sequential tcsr.hpp:37          build_sequential(stream, reverse)
    tgf::build_parallel   tcsr.hpp:43          build_parallel(stream, reverse, num_threads)
    tgf::TCsr             tcsr.hpp:20-33       TCsr (device-resident; host columns on demand)
    tgf::sample_recent    sampler.hpp:32       sample_recent(g, u, t, k)
    tgf::sample_random    sampler.hpp:37-38    sample_random(g, u, t, k, seed, stream)
    tgf::sample_batch     sampler.hpp:42-45    sample_batch(g, nodes, times, k, strategy, seed)
    tgf::build_sequence_batch sequence.hpp:45  build_sequence_batch(samples, l, self_edge_index)
    tgf::build_mask       sequence.hpp:50      build_mask(batch, kind)
    tgf::make_random_stream synthetic.hpp:17   make_random_stream(E, V, seed, zipf)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, NamedTuple

import numpy as np

from ._lib import (TGFX_INDEX64, TGFX_RANDOM, TGFX_RECENT, TGFX_TRUSTED, FormatError,
                   ParseError, TgfxError, ValidationError, check, lib)

EVENT_DTYPE = np.dtype([("edge_id", "<i8"), ("src", "<i8"), ("dst", "<i8"), ("timestamp", "<f8")])

__all__ = ["EventStream", "TCsr", "NeighborEntry", "NeighborSample", "SequenceBatch",
           "build_sequential", "build_parallel", "build_device", "sample_recent", "sample_random",
           "sample_batch", "sample_batch_arrays", "sample_assemble", "sample_two_hop",
           "build_sequence", "build_sequence_batch", "build_mask", "make_random_stream",
           "parse_strategy", "parse_mask_kind", "ValidationError", "FormatError", "TgfxError",
           "ParseError", "load_csv",
           "EVENT_DTYPE"]


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _events(ev):
    ev = np.ascontiguousarray(ev)
    if ev.dtype != EVENT_DTYPE:
        ev = ev.astype(EVENT_DTYPE)
    return ev


@dataclass
class EventStream:
    """proj/include/tgformer/event_stream.hpp:26-39 (events + num_nodes; features unused here)."""

    events: np.ndarray
    num_nodes: int

    def size(self):
        return len(self.events)


def parse_strategy(name):
    """tgf::parse_strategy (proj/src/sampler.cpp:35-39)"""
    if name == "recent":
        return "recent"
    if name == "random":
        return "random"
    raise ValidationError(f"unknown sampling strategy '{name}'")


def parse_mask_kind(name):
    """tgf::parse_mask_kind (proj/src/sequence.cpp:48-53)"""
    if name in ("causal", "tgat", "self_loop"):
        return name
    raise ValidationError(f"unknown mask kind '{name}'")


def _strategy_code(strategy):
    if isinstance(strategy, int):
        return strategy
    return TGFX_RECENT if parse_strategy(strategy) == "recent" else TGFX_RANDOM


class TCsr:
    """Device-resident T-CSR (proj/include/tgformer/tcsr.hpp:20-33).  Host columns
    (indptr, neighbor_ids, edge_ids, timestamps) are exported lazily on first access."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)
        n = C.c_int64()
        e = C.c_int64()
        m = C.c_int64()
        r = C.c_int()
        check(lib().tgfx_graph_info(self._h, C.byref(n), C.byref(e), C.byref(m), C.byref(r)))
        self.num_nodes, self.num_edges, self._m, self.reverse = n.value, e.value, m.value, bool(r.value)
        self._host = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().tgfx_graph_free(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def num_entries(self):
        return self._m

    @property
    def build_path(self):
        return int(lib().tgfx_graph_build_path(self._h))

    def _export(self):
        if self._host is None:
            m = self._m
            ip = np.zeros(self.num_nodes + 1, np.int64)
            nb = np.zeros(max(m, 1), np.int64)
            ed = np.zeros(max(m, 1), np.int64)
            ts = np.zeros(max(m, 1), np.float64)
            check(lib().tgfx_graph_export(self._h, _ptr(ip), _ptr(nb), _ptr(ed), _ptr(ts)))
            self._host = (ip, nb[:m], ed[:m], ts[:m])
        return self._host

    @property
    def indptr(self):
        return self._export()[0]

    @property
    def neighbor_ids(self):
        return self._export()[1]

    @property
    def edge_ids(self):
        return self._export()[2]

    @property
    def timestamps(self):
        return self._export()[3]

    def degree(self, u):
        ip = self.indptr
        return int(ip[u + 1] - ip[u])

    def device_arrays(self):
        """Raw device pointers (indptr, nbr, eid, ts) as ints."""
        ps = [C.c_void_p() for _ in range(4)]
        check(lib().tgfx_graph_device_arrays(self._h, *(C.byref(p) for p in ps)))
        return tuple(p.value for p in ps)

    def validate(self):
        """TCsr::validate (proj/src/tcsr.cpp:54-81), on the device."""
        check(lib().tgfx_graph_validate(self._h))

    @classmethod
    def from_host(cls, num_nodes, num_edges, reverse, indptr, nbr, eid, ts):
        h = C.c_void_p()
        arrs = [np.ascontiguousarray(a, dtype=t) for a, t in
                ((indptr, np.int64), (nbr, np.int64), (eid, np.int64), (ts, np.float64))]
        check(lib().tgfx_graph_from_host(num_nodes, num_edges, 1 if reverse else 0, len(arrs[1]),
                                         *(_ptr(a) for a in arrs), C.byref(h)))
        return cls(h.value)


def _stream_args(stream, num_nodes):
    if isinstance(stream, EventStream):
        return _events(stream.events), stream.num_nodes
    if num_nodes is None:
        raise ValidationError("num_nodes required")
    return _events(stream), num_nodes


def build_sequential(stream, reverse=True, num_nodes=None):
    """tgf::build_sequential (proj/src/tcsr.cpp:83-105), computed on the GPU."""
    ev, V = _stream_args(stream, num_nodes)
    h = C.c_void_p()
    check(lib().tgfx_build_sequential(_ptr(ev), len(ev), V, 1 if reverse else 0, C.byref(h)))
    return TCsr(h.value)


def build_parallel(stream, reverse, num_threads, num_nodes=None):
    """tgf::build_parallel (proj/src/tcsr.cpp:107-151): num_threads < 1 -> ValidationError."""
    ev, V = _stream_args(stream, num_nodes)
    h = C.c_void_p()
    check(lib().tgfx_build_parallel(_ptr(ev), len(ev), V, 1 if reverse else 0, num_threads,
                                    C.byref(h)))
    return TCsr(h.value)


def build_device(events_ptr, n, num_nodes, reverse=True, stream=0, trusted=False):
    """Build from device-resident events (int pointer to n x 32 bytes)."""
    h = C.c_void_p()
    check(lib().tgfx_build_device(C.c_void_p(events_ptr), n, num_nodes, 1 if reverse else 0,
                                  C.c_void_p(stream), TGFX_TRUSTED if trusted else 0, C.byref(h)))
    return TCsr(h.value)


class NeighborEntry(NamedTuple):
    """proj/include/tgformer/sampler.hpp:12-16"""

    neighbor: int
    edge: int
    timestamp: float


@dataclass
class NeighborSample:
    """proj/include/tgformer/sampler.hpp:20-24"""

    query_node: int = 0
    query_time: float = 0.0
    neighbors: List[NeighborEntry] = field(default_factory=list)


def sample_batch_arrays(g, nodes, times, k, strategy="recent", seed=0, stream_base=0):
    """Padded form of sample_batch: (counts[Q], nbr[Q,k], eid[Q,k], ts[Q,k])."""
    nodes = np.ascontiguousarray(nodes, dtype=np.int64)
    times = np.ascontiguousarray(times, dtype=np.float64)
    if len(nodes) != len(times):
        raise ValidationError("node and time lists differ in length")  # sampler.cpp:88-90
    q = len(nodes)
    kp = max(int(k), 1)
    counts = np.zeros(q, np.int64)
    nb = np.zeros(q * kp, np.int64)
    ed = np.zeros(q * kp, np.int64)
    ts = np.zeros(q * kp, np.float64)
    check(lib().tgfx_sample_batch(g.handle, _ptr(nodes), _ptr(times), q, k,
                                  _strategy_code(strategy), seed & (2**64 - 1),
                                  stream_base & (2**64 - 1), _ptr(counts), _ptr(nb), _ptr(ed),
                                  _ptr(ts)))
    return counts, nb.reshape(q, kp), ed.reshape(q, kp), ts.reshape(q, kp)


def sample_batch(g, nodes, times, k, strategy="recent", seed=0, num_threads=0, stream_base=0):
    """tgf::sample_batch (proj/src/sampler.cpp:84-104); num_threads is accepted and ignored."""
    nodes = np.ascontiguousarray(nodes, dtype=np.int64)
    times = np.ascontiguousarray(times, dtype=np.float64)
    counts, nb, ed, ts = sample_batch_arrays(g, nodes, times, k, strategy, seed, stream_base)
    out = []
    for i in range(len(nodes)):
        c = int(counts[i])
        out.append(NeighborSample(int(nodes[i]), float(times[i]),
                                  [NeighborEntry(int(nb[i, j]), int(ed[i, j]), float(ts[i, j]))
                                   for j in range(c)]))
    return out


def sample_recent(g, u, t, k):
    """tgf::sample_recent (proj/src/sampler.cpp:41-52)"""
    return sample_batch(g, [u], [t], k, "recent")[0]


def sample_random(g, u, t, k, seed, stream=0):
    """tgf::sample_random (proj/src/sampler.cpp:54-82) with the (seed, stream) counter RNG"""
    return sample_batch(g, [u], [t], k, "random", seed, stream_base=stream)[0]


@dataclass
class SequenceBatch:
    """proj/include/tgformer/sequence.hpp:20-30 (numpy; time_delta is batch x l)."""

    batch: int
    l: int
    node_index: np.ndarray
    edge_index: np.ndarray
    time_delta: np.ndarray
    valid_len: np.ndarray
    target_row: np.ndarray


def build_sequence_batch(samples, l, self_edge_index):
    """tgf::build_sequence_batch (proj/src/sequence.cpp:55-86), on the GPU."""
    q = len(samples)
    kp = max([len(s.neighbors) for s in samples] + [1])
    counts = np.zeros(q, np.int64)
    nb = np.zeros((q, kp), np.int64)
    ed = np.zeros((q, kp), np.int64)
    ts = np.zeros((q, kp), np.float64)
    qn = np.zeros(q, np.int64)
    qt = np.zeros(q, np.float64)
    for i, s in enumerate(samples):
        counts[i] = len(s.neighbors)
        qn[i], qt[i] = s.query_node, s.query_time
        for j, e in enumerate(s.neighbors):
            nb[i, j], ed[i, j], ts[i, j] = e.neighbor, e.edge, e.timestamp
    return assemble_arrays(counts, nb, ed, ts, qn, qt, l, self_edge_index)


def assemble_arrays(counts, nbr, eid, ts, qnodes, qtimes, l, self_edge_index):
    q = len(counts)
    kp = nbr.shape[1] if nbr.ndim == 2 else 1
    ni = np.zeros(max(q * l, 1), np.int64)
    ei = np.zeros(max(q * l, 1), np.int64)
    dt = np.zeros(max(q * l, 1), np.float64)
    vl = np.zeros(max(q, 1), np.int64)
    tr = np.zeros(max(q, 1), np.int64)
    a = [np.ascontiguousarray(x, dtype=t) for x, t in
         ((counts, np.int64), (nbr, np.int64), (eid, np.int64), (ts, np.float64),
          (qnodes, np.int64), (qtimes, np.float64))]
    check(lib().tgfx_assemble(q, kp, *(_ptr(x) for x in a), l, self_edge_index, _ptr(ni),
                              _ptr(ei), _ptr(dt), _ptr(vl), _ptr(tr)))
    return SequenceBatch(q, l, ni[:q * l].reshape(q, l), ei[:q * l].reshape(q, l),
                         dt[:q * l].reshape(q, l), vl[:q], tr[:q])


def build_sequence(sample, l, self_edge_index):
    """tgf::build_sequence (proj/src/sequence.cpp:88-91)"""
    return build_sequence_batch([sample], l, self_edge_index)


def build_mask(batch, kind):
    """tgf::build_mask (proj/src/sequence.cpp:93-111): (batch*l) x l of {0, -inf}."""
    kinds = {"causal": 0, "tgat": 1, "self_loop": 2}
    kind = parse_mask_kind(kind)
    q, l = batch.batch, batch.l
    mask = np.zeros(max(q * l * l, 1), np.float64)
    vl = np.ascontiguousarray(batch.valid_len, np.int64)
    tr = np.ascontiguousarray(batch.target_row, np.int64)
    check(lib().tgfx_build_mask(q, l, _ptr(vl), _ptr(tr), kinds[kind], _ptr(mask)))
    return mask[:q * l * l].reshape(q * l, l)


def sample_assemble(g, nodes, times, k, strategy, seed, l, self_edge_index, stream_base=0,
                    dt64=False):
    """sample_batch + build_sequence_batch fused (the forward_concat pair,
    proj/src/training.cpp:211-214).  int32 ids, fp32 (and optionally fp64) deltas."""
    nodes = np.ascontiguousarray(nodes, dtype=np.int64)
    times = np.ascontiguousarray(times, dtype=np.float64)
    if len(nodes) != len(times):
        raise ValidationError("node and time lists differ in length")
    q = len(nodes)
    ni = np.zeros((max(q, 1), l), np.int32)
    ei = np.zeros((max(q, 1), l), np.int32)
    d32 = np.zeros((max(q, 1), l), np.float32)
    d64 = np.zeros((max(q, 1), l), np.float64) if dt64 else None
    vl = np.zeros(max(q, 1), np.int32)
    check(lib().tgfx_sample_assemble(g.handle, _ptr(nodes), _ptr(times), q, k,
                                     _strategy_code(strategy), seed & (2**64 - 1),
                                     stream_base & (2**64 - 1), l, self_edge_index, _ptr(ni),
                                     _ptr(ei), _ptr(d32), _ptr(d64), _ptr(vl)))
    out = dict(node_index=ni[:q], edge_index=ei[:q], time_delta=d32[:q], valid_len=vl[:q])
    if dt64:
        out["time_delta64"] = d64[:q]
    return out


def sample_two_hop(g, roots, times, k1, k2, strategy, seed, l, self_edge_index, seed2=None):
    """2-hop composition: hop-1 rows [Q, l], hop-2 rows [Q, k1, l]."""
    roots = np.ascontiguousarray(roots, dtype=np.int64)
    times = np.ascontiguousarray(times, dtype=np.float64)
    q = len(roots)
    s2 = seed if seed2 is None else seed2
    h1 = [np.zeros((max(q, 1), l), t) for t in (np.int32, np.int32, np.float32)]
    h1l = np.zeros(max(q, 1), np.int32)
    h2 = [np.zeros((max(q, 1), k1, l), t) for t in (np.int32, np.int32, np.float32)]
    h2l = np.zeros((max(q, 1), k1), np.int32)
    check(lib().tgfx_sample_two_hop(g.handle, _ptr(roots), _ptr(times), q, k1, k2,
                                    _strategy_code(strategy), seed, s2, l, self_edge_index,
                                    *(_ptr(a) for a in h1), _ptr(h1l), *(_ptr(a) for a in h2),
                                    _ptr(h2l)))
    hop1 = dict(node_index=h1[0][:q], edge_index=h1[1][:q], time_delta=h1[2][:q],
                valid_len=h1l[:q])
    hop2 = dict(node_index=h2[0][:q], edge_index=h2[1][:q], time_delta=h2[2][:q],
                valid_len=h2l[:q])
    return hop1, hop2


def make_random_stream(num_edges, num_nodes, seed, zipf_exponent=1.2):
    """tgf::make_random_stream (proj/src/synthetic.cpp:12-43), generated on the GPU."""
    ev = np.zeros(max(num_edges, 1), EVENT_DTYPE)
    check(lib().tgfx_make_random_stream(num_edges, num_nodes, seed, zipf_exponent, _ptr(ev)))
    return EventStream(ev[:num_edges], num_nodes)


def load_csv(path, has_features=False):
    """tgf::load_csv (proj/src/event_stream.cpp:85-154), parsed on the device ->
    EventStream (events in the reference's layout) and the edge features [n, d_e]."""
    h = C.c_void_p()
    check(lib().tgfx_load_csv(str(path).encode(), 1 if has_features else 0, C.byref(h)))
    try:
        n, v, de = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().tgfx_csv_info(h, C.byref(n), C.byref(v), C.byref(de)))
        ev = np.zeros(n.value, dtype=EVENT_DTYPE)
        feats = np.zeros((n.value, de.value), dtype=np.float64)
        check(lib().tgfx_csv_export(h, _ptr(ev) if n.value else None,
                                    _ptr(feats) if feats.size else None))
    finally:
        lib().tgfx_csv_free(h)
    return EventStream(ev, v.value), feats
