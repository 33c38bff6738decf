"""ctypes bindings for the CPU oracle (liboracle.so) and the compiled reference (_ref/libtgf_ref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs -- as the checker or the CPU baseline, never as the
product path.  The product (paper_2409_05477_b200, libtgfx.so) never imports this module.

Array conventions follow the reference (proj/include/tgformer/*.hpp): ids int64, times
float64, events as the 32-byte TemporalEvent record (event_stream.hpp:13-18).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtgf_ref.so")
# the same reference build for the GPU box's host CPU (Emerald Rapids): -march=native there
REF_SO_NATIVE = os.path.join(HERE, "_ref", "libtgf_ref_emr.so")


def host_has_native_isa():
    """True when this CPU runs the -march=emeraldrapids build (AMX + AVX512-FP16 present)."""
    try:
        with open("/proc/cpuinfo") as f:
            flags = next((ln for ln in f if ln.startswith("flags")), "")
    except OSError:
        return False
    need = ("avx512_fp16", "amx_tile", "avx512_bf16", "avx512_vbmi2", "avx_vnni", "movdir64b")
    return all(n in flags.split() for n in need)


def ref_so_path(native=False):
    """native=True: the box-tuned build when it exists and this CPU can run it."""
    if native and os.path.exists(REF_SO_NATIVE) and host_has_native_isa():
        return REF_SO_NATIVE
    return REF_SO

EVENT_DTYPE = np.dtype([("edge_id", "<i8"), ("src", "<i8"), ("dst", "<i8"), ("timestamp", "<f8")])

_P = C.c_void_p
_I64 = C.c_int64
_U64 = C.c_uint64


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def build_oracle():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_orc = None
_ref = None


def _setup_fromchars(L):
    L.orc_from_chars_f64.argtypes = [C.c_char_p, _I64, C.POINTER(C.c_double)]
    L.orc_from_chars_i64.argtypes = [C.c_char_p, _I64, C.POINTER(C.c_int64)]


def lib():
    """The C restatement (oracle.c)."""
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            build_oracle()
        L = C.CDLL(ORACLE_SO)
        _setup_fromchars(L)
        L.orc_mix64.restype = _U64
        L.orc_mix64.argtypes = [_U64]
        L.orc_rng_state.restype = _U64
        L.orc_rng_state.argtypes = [_U64, _U64]
        L.orc_rng_draw.restype = _U64
        L.orc_rng_draw.argtypes = [_U64, _U64]
        L.orc_mulhi64.restype = _U64
        L.orc_mulhi64.argtypes = [_U64, _U64]
        L.orc_make_random_stream.argtypes = [_I64, _I64, _U64, C.c_double, _P]
        L.orc_zipf_cdf.argtypes = [_I64, C.c_double, _P]
        L.orc_build.argtypes = [_P, _I64, _I64, C.c_int, _P, _P, _P, _P, _P]
        L.orc_validate.argtypes = [_I64, _I64, _I64, _P, _P, _P, _P]
        L.orc_prefix_end.restype = _I64
        L.orc_prefix_end.argtypes = [_P, _P, _I64, C.c_double]
        L.orc_sample_batch.argtypes = [_I64, _P, _P, _P, _P, _P, _P, _I64, _I64, C.c_int, _U64,
                                       _U64, _P, _P, _P, _P, _P]
        L.orc_build_sequence_batch.argtypes = [_I64, _I64, _P, _P, _P, _P, _P, _P, _I64, _I64,
                                               _P, _P, _P, _P, _P]
        L.orc_build_mask.argtypes = [_I64, _I64, _P, _P, C.c_int, _P]
        L.orc_make_queries.argtypes = [_P, _I64, _I64, _I64, _I64, _U64, _P, _P]
        _orc = L
    return _orc


def ref_available():
    return os.path.exists(REF_SO)


_ref_path = None


def ref(native=False):
    """The reference's own hot path (compiled from /root/reference by oracle/Makefile).
    native=True (first call only) loads the build tuned for the GPU box's host CPU."""
    global _ref, _ref_path
    if _ref is None:
        path = ref_so_path(native)
        if not os.path.exists(path):
            raise RuntimeError(f"reference build {path} missing (run make -C oracle)")
        L = C.CDLL(path)
        _ref_path = path
        L.ref_last_error.restype = C.c_char_p
        L.ref_make_random_stream.argtypes = [_I64, _I64, _U64, C.c_double, _P]
        L.ref_stream_create.restype = _P
        L.ref_stream_create.argtypes = [_P, _I64, _I64]
        L.ref_stream_free.argtypes = [_P]
        L.ref_build.argtypes = [_P, C.c_int, C.c_int, C.POINTER(_P), C.POINTER(C.c_double)]
        L.ref_build_parallel_raw.argtypes = [_P, C.c_int, C.c_int, C.POINTER(_P)]
        L.ref_graph_free.argtypes = [_P]
        L.ref_graph_info.argtypes = [_P, _P]
        L.ref_graph_export.argtypes = [_P, _P, _P, _P, _P]
        L.ref_graph_validate.argtypes = [_P]
        L.ref_graph_from_columns.restype = _P
        L.ref_graph_from_columns.argtypes = [_I64, _I64, C.c_int, _I64, _P, _P, _P, _P]
        L.ref_sample_batch.argtypes = [_P, _P, _P, _I64, _I64, C.c_int, _U64, C.c_int, _P, _P, _P,
                                       _P, C.POINTER(C.c_double)]
        L.ref_sample_random.argtypes = [_P, _I64, C.c_double, _I64, _U64, _U64, _P, _P, _P, _P]
        L.ref_sample_assemble.argtypes = [_P, _P, _P, _I64, _I64, C.c_int, _U64, C.c_int, _I64,
                                          _I64, _P, _P, _P, _P, C.POINTER(C.c_double)]
        L.ref_build_sequence_batch.argtypes = [_I64, _I64, _P, _P, _P, _P, _P, _P, _I64, _I64, _P,
                                               _P, _P, _P, _P]
        L.ref_build_mask.argtypes = [_I64, _I64, _P, _P, C.c_int, _P]
        L.ref_load_csv.argtypes = [C.c_char_p, C.c_int, _P, _P, _P, _P, _P]
        L.ref_assemble_inputs.argtypes = [_I64, _I64, _P, _P, _P, _P, _P, _I64, _P, _I64, _P, _P,
                                          _I64, _I64, _I64, C.c_int, _P]
        L.ref_train_queries.argtypes = [_P, _I64, _I64, _I64, _I64, _U64, _P, _P, _P]
        _ref = L
    return _ref


class OracleError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


# --------------------------------------------------------------------------- restatement

def mix64(x):
    return lib().orc_mix64(x)


def make_random_stream(num_edges, num_nodes, seed, zipf=1.2):
    ev = np.zeros(num_edges, dtype=EVENT_DTYPE)
    rc = lib().orc_make_random_stream(num_edges, num_nodes, seed, zipf, _ptr(ev))
    if rc:
        raise OracleError(1, "bad stream dimensions")
    return ev


_M64 = 2**64 - 1


def mix_streams(a, b, c):
    """proj/src/training.cpp:16-18 (train_epoch's seed derivation)."""
    return mix64((mix64((a ^ 0x8f1bbcdcbfa53e0b) & _M64) ^ mix64(b & _M64) ^
                  ((c * 0x2545f4914f6cdd1d) & _M64)) & _M64)


def make_train_queries(events, batch_size, neg_per_pos, workers, num_nodes, batch_seed):
    """The sample_batch queries of one train_epoch, concatenated in call order:
    make_batches (proj/src/training.cpp:157-182; negatives CounterRng(batch_seed, batch index)
    .next_below(num_nodes), rng.hpp:23-38), split into min(workers, b) shards
    [h*b/m, (h+1)*b/m) (:425-440), each in forward_concat's layout [src | dst | neg]
    (:193-209).  Pure restatement (small inputs)."""
    events = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
    n = len(events)
    nodes, times = [], []
    for b, start in enumerate(range(0, n, batch_size)):
        stop = min(start + batch_size, n)
        s0 = mix64((mix64(batch_seed) ^ ((b * 0xd6e8feb86659fd93) & _M64)) & _M64)
        bs = stop - start
        neg = [lib().orc_mulhi64(mix64((s0 + d * 0x9e3779b97f4a7c15) & _M64), num_nodes)
               for d in range(bs * neg_per_pos)]
        ev = events[start:stop]
        m = min(workers, bs)
        for h in range(m):
            lo, hi = h * bs // m, (h + 1) * bs // m
            part = ev[lo:hi]
            nodes += list(part["src"]) + list(part["dst"]) + neg[lo * neg_per_pos:hi * neg_per_pos]
            times += (list(part["timestamp"]) * 2 +
                      [float(ev["timestamp"][lo + j // neg_per_pos])
                       for j in range((hi - lo) * neg_per_pos)])
    return np.array(nodes, np.int64), np.array(times, np.float64)


def zipf_cdf(num_nodes, zipf=1.2):
    cdf = np.zeros(num_nodes, dtype=np.float64)
    lib().orc_zipf_cdf(num_nodes, zipf, _ptr(cdf))
    return cdf


def events_from(src, dst, ts, eid=None):
    n = len(src)
    ev = np.zeros(n, dtype=EVENT_DTYPE)
    ev["edge_id"] = np.arange(n) if eid is None else eid
    ev["src"], ev["dst"], ev["timestamp"] = src, dst, ts
    return ev


def build(events, num_nodes, reverse=True):
    """build_sequential (tcsr.cpp:83-105) -> dict(indptr, nbr, eid, ts)."""
    events = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
    n = len(events)
    m = n * (2 if reverse else 1)
    indptr = np.zeros(num_nodes + 1, dtype=np.int64)
    nbr = np.zeros(max(m, 1), dtype=np.int64)
    eid = np.zeros(max(m, 1), dtype=np.int64)
    ts = np.zeros(max(m, 1), dtype=np.float64)
    bad = np.zeros(1, dtype=np.int64)
    rc = lib().orc_build(_ptr(events), n, num_nodes, 1 if reverse else 0, _ptr(indptr), _ptr(nbr),
                         _ptr(eid), _ptr(ts), _ptr(bad))
    if rc:
        raise OracleError(1, f"event {int(bad[0])} endpoint out of range")
    return dict(num_nodes=num_nodes, num_edges=n, reverse=bool(reverse), indptr=indptr,
                nbr=nbr[:m], eid=eid[:m], ts=ts[:m])


def validate(g):
    rc = lib().orc_validate(g["num_nodes"], g["num_edges"], len(g["nbr"]), _ptr(g["indptr"]),
                            _ptr(g["nbr"]), _ptr(g["eid"]), _ptr(g["ts"]))
    return rc == 0


def sample_batch(g, nodes, times, k, strategy="recent", seed=0, stream_base=0):
    """sample_batch (sampler.cpp:84-104) -> (counts[Q], nbr[Q,k], eid[Q,k], ts[Q,k])."""
    nodes = np.ascontiguousarray(nodes, dtype=np.int64)
    times = np.ascontiguousarray(times, dtype=np.float64)
    q = len(nodes)
    kp = max(k, 1)
    counts = np.zeros(q, dtype=np.int64)
    nb = np.zeros(q * kp, dtype=np.int64)
    ed = np.zeros(q * kp, dtype=np.int64)
    tt = np.zeros(q * kp, dtype=np.float64)
    bad = np.zeros(1, dtype=np.int64)
    rc = lib().orc_sample_batch(g["num_nodes"], _ptr(g["indptr"]), _ptr(g["nbr"]), _ptr(g["eid"]),
                                _ptr(g["ts"]), _ptr(nodes), _ptr(times), q, k,
                                0 if strategy == "recent" else 1, seed, stream_base, _ptr(counts),
                                _ptr(nb), _ptr(ed), _ptr(tt), _ptr(bad))
    if rc == 1:
        raise OracleError(1, f"query node {int(bad[0])} out of range")
    if rc == 2:
        raise OracleError(1, "k must be at least 1")
    return counts, nb.reshape(q, kp), ed.reshape(q, kp), tt.reshape(q, kp)


def build_sequence_batch(counts, nbr, eid, ts, qnodes, qtimes, l, self_edge_index):
    """build_sequence_batch (sequence.cpp:55-86) -> dict of int64/float64 arrays."""
    q, kp = nbr.shape
    ni = np.zeros(q * l, dtype=np.int64)
    ei = np.zeros(q * l, dtype=np.int64)
    dt = np.zeros(q * l, dtype=np.float64)
    vl = np.zeros(q, dtype=np.int64)
    tr = np.zeros(q, dtype=np.int64)
    c = [np.ascontiguousarray(a) for a in (counts, nbr, eid, ts)]
    qn = np.ascontiguousarray(qnodes, dtype=np.int64)
    qt = np.ascontiguousarray(qtimes, dtype=np.float64)
    rc = lib().orc_build_sequence_batch(q, kp, _ptr(c[0]), _ptr(c[1]), _ptr(c[2]), _ptr(c[3]),
                                        _ptr(qn), _ptr(qt), l, self_edge_index, _ptr(ni), _ptr(ei),
                                        _ptr(dt), _ptr(vl), _ptr(tr))
    if rc:
        raise OracleError(1, "sequence length must be at least 2")
    return dict(node_index=ni.reshape(q, l), edge_index=ei.reshape(q, l),
                time_delta=dt.reshape(q, l), valid_len=vl, target_row=tr)


def sample_assemble(g, nodes, times, k, strategy, seed, l, self_edge_index, stream_base=0):
    counts, nb, ed, tt = sample_batch(g, nodes, times, k, strategy, seed, stream_base)
    return build_sequence_batch(counts, nb, ed, tt, nodes, times, l, self_edge_index)


def build_mask(valid_len, target_row, l, kind):
    kinds = {"causal": 0, "tgat": 1, "self_loop": 2}
    q = len(valid_len)
    mask = np.zeros(q * l * l, dtype=np.float64)
    vl = np.ascontiguousarray(valid_len, dtype=np.int64)
    tr = np.ascontiguousarray(target_row, dtype=np.int64)
    lib().orc_build_mask(q, l, _ptr(vl), _ptr(tr), kinds[kind], _ptr(mask))
    return mask.reshape(q * l, l)


def make_queries(events, e0, e1, batch, num_nodes, neg_seed=7):
    events = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
    n = 3 * (e1 - e0)
    nodes = np.zeros(n, dtype=np.int64)
    times = np.zeros(n, dtype=np.float64)
    lib().orc_make_queries(_ptr(events), e0, e1, batch, num_nodes, neg_seed, _ptr(nodes),
                           _ptr(times))
    return nodes, times


def two_hop(g, roots, rtimes, k1, k2, strategy, seed, l, self_edge_index, seed2=None):
    """2-hop composition defined over reference calls:

    hop-1 = sample_batch(roots, k1); hop-2 query for hop-1 entry j of root q is
    (nbr_j, ts_j) sampled with k2 (recent) or sample_random(seed2, stream = q*k1 + j).
    Returns hop-1 rows [Q, l] and hop-2 rows [Q, k1, l] (absent slots zero, valid_len 0).
    """
    q = len(roots)
    c1, n1, e1, t1 = sample_batch(g, roots, rtimes, k1, strategy, seed)
    hop1 = build_sequence_batch(c1, n1, e1, t1, roots, rtimes, l, self_edge_index)
    ni = np.zeros((q, k1, l), np.int64)
    ei = np.zeros((q, k1, l), np.int64)
    dt = np.zeros((q, k1, l), np.float64)
    vl = np.zeros((q, k1), np.int64)
    qi, ji = np.nonzero(np.arange(k1)[None, :] < c1[:, None])
    if len(qi):
        hn = n1[qi, ji]
        ht = t1[qi, ji]
        if strategy == "recent":
            c2, n2, e2, t2 = sample_batch(g, hn, ht, k2, "recent", 0)
        else:
            s2 = seed if seed2 is None else seed2
            c2 = np.zeros(len(qi), np.int64)
            n2 = np.zeros((len(qi), k2), np.int64)
            e2 = np.zeros((len(qi), k2), np.int64)
            t2 = np.zeros((len(qi), k2), np.float64)
            for r in range(len(qi)):
                cc, a, b, c = sample_batch(g, hn[r:r + 1], ht[r:r + 1], k2, "random", s2,
                                           stream_base=int(qi[r]) * k1 + int(ji[r]))
                c2[r], n2[r], e2[r], t2[r] = cc[0], a[0], b[0], c[0]
        h2 = build_sequence_batch(c2, n2, e2, t2, hn, ht, l, self_edge_index)
        ni[qi, ji] = h2["node_index"]
        ei[qi, ji] = h2["edge_index"]
        dt[qi, ji] = h2["time_delta"]
        vl[qi, ji] = h2["valid_len"]
    return hop1, dict(node_index=ni, edge_index=ei, time_delta=dt, valid_len=vl)


# --------------------------------------------------------------------------- reference

class RefGraph:
    """A tgf::TCsr built by the compiled reference."""

    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_graph_free(self.h)
            self.h = None

    def info(self):
        out = np.zeros(4, np.int64)
        ref().ref_graph_info(self.h, _ptr(out))
        return dict(num_nodes=int(out[0]), num_edges=int(out[1]), num_entries=int(out[2]),
                    reverse=bool(out[3]))

    def export(self):
        inf = self.info()
        m = inf["num_entries"]
        indptr = np.zeros(inf["num_nodes"] + 1, np.int64)
        nbr = np.zeros(max(m, 1), np.int64)
        eid = np.zeros(max(m, 1), np.int64)
        ts = np.zeros(max(m, 1), np.float64)
        ref().ref_graph_export(self.h, _ptr(indptr), _ptr(nbr), _ptr(eid), _ptr(ts))
        return dict(num_nodes=inf["num_nodes"], num_edges=inf["num_edges"],
                    reverse=inf["reverse"], indptr=indptr, nbr=nbr[:m], eid=eid[:m], ts=ts[:m])


def ref_validate_columns(num_nodes, num_edges, reverse, indptr, nbr, eid, ts):
    """TCsr::validate (tcsr.cpp:54-81) of the reference on the given columns -> message or ''."""
    arrs = [np.ascontiguousarray(a, dtype=t) for a, t in
            ((indptr, np.int64), (nbr, np.int64), (eid, np.int64), (ts, np.float64))]
    h = ref().ref_graph_from_columns(num_nodes, num_edges, 1 if reverse else 0, len(arrs[1]),
                                     *(_ptr(a) for a in arrs))
    g = RefGraph(h)
    rc = ref().ref_graph_validate(g.h)
    return ref().ref_last_error().decode() if rc else ""


def _ref_err(rc):
    msg = ref().ref_last_error().decode()
    raise OracleError(rc, msg)


def ref_make_random_stream(num_edges, num_nodes, seed, zipf=1.2):
    ev = np.zeros(num_edges, dtype=EVENT_DTYPE)
    rc = ref().ref_make_random_stream(num_edges, num_nodes, seed, zipf, _ptr(ev))
    if rc:
        _ref_err(rc)
    return ev


class RefStream:
    def __init__(self, events, num_nodes):
        self.events = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
        self.h = ref().ref_stream_create(_ptr(self.events), len(self.events), num_nodes)

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_stream_free(self.h)
            self.h = None

    def build(self, reverse=True, threads=0):
        """threads <= 0: build_sequential; else build_parallel(threads). -> (RefGraph, secs)."""
        g = C.c_void_p()
        s = C.c_double()
        rc = ref().ref_build(self.h, 1 if reverse else 0, threads, C.byref(g), C.byref(s))
        if rc:
            _ref_err(rc)
        return RefGraph(g.value), s.value

    def build_parallel_raw(self, reverse, threads):
        g = C.c_void_p()
        rc = ref().ref_build_parallel_raw(self.h, 1 if reverse else 0, threads, C.byref(g))
        if rc:
            _ref_err(rc)
        return RefGraph(g.value)


def ref_sample_batch(rg, nodes, times, k, strategy="recent", seed=0, threads=0):
    nodes = np.ascontiguousarray(nodes, dtype=np.int64)
    times = np.ascontiguousarray(times, dtype=np.float64)
    q = len(nodes)
    kp = max(k, 1)
    counts = np.zeros(q, np.int64)
    nb = np.zeros(q * kp, np.int64)
    ed = np.zeros(q * kp, np.int64)
    tt = np.zeros(q * kp, np.float64)
    s = C.c_double()
    rc = ref().ref_sample_batch(rg.h, _ptr(nodes), _ptr(times), q, k,
                                0 if strategy == "recent" else 1, seed, threads, _ptr(counts),
                                _ptr(nb), _ptr(ed), _ptr(tt), C.byref(s))
    if rc:
        _ref_err(rc)
    return (counts, nb.reshape(q, kp), ed.reshape(q, kp), tt.reshape(q, kp)), s.value


def ref_sample_random(rg, u, t, k, seed, stream):
    cnt = np.zeros(1, np.int64)
    nb = np.zeros(max(k, 1), np.int64)
    ed = np.zeros(max(k, 1), np.int64)
    tt = np.zeros(max(k, 1), np.float64)
    rc = ref().ref_sample_random(rg.h, u, t, k, seed, stream, _ptr(cnt), _ptr(nb), _ptr(ed),
                                 _ptr(tt))
    if rc:
        _ref_err(rc)
    c = int(cnt[0])
    return nb[:c], ed[:c], tt[:c]


def ref_sample_assemble(rg, nodes, times, k, strategy, seed, l, self_edge_index, threads=0,
                        want_outputs=True):
    nodes = np.ascontiguousarray(nodes, dtype=np.int64)
    times = np.ascontiguousarray(times, dtype=np.float64)
    q = len(nodes)
    if want_outputs:
        ni = np.zeros(q * l, np.int64)
        ei = np.zeros(q * l, np.int64)
        dt = np.zeros(q * l, np.float64)
        vl = np.zeros(q, np.int64)
    else:
        ni = ei = dt = vl = None
    s = C.c_double()
    rc = ref().ref_sample_assemble(rg.h, _ptr(nodes), _ptr(times), q, k,
                                   0 if strategy == "recent" else 1, seed, threads, l,
                                   self_edge_index, _ptr(ni), _ptr(ei), _ptr(dt), _ptr(vl),
                                   C.byref(s))
    if rc:
        _ref_err(rc)
    out = None
    if want_outputs:
        out = dict(node_index=ni.reshape(q, l), edge_index=ei.reshape(q, l),
                   time_delta=dt.reshape(q, l), valid_len=vl)
    return out, s.value


def ref_build_sequence_batch(counts, nbr, eid, ts, qnodes, qtimes, l, self_edge_index):
    q, kp = nbr.shape
    ni = np.zeros(q * l, np.int64)
    ei = np.zeros(q * l, np.int64)
    dt = np.zeros(q * l, np.float64)
    vl = np.zeros(q, np.int64)
    tr = np.zeros(q, np.int64)
    c = [np.ascontiguousarray(a) for a in (counts, nbr, eid, ts)]
    qn = np.ascontiguousarray(qnodes, dtype=np.int64)
    qt = np.ascontiguousarray(qtimes, dtype=np.float64)
    rc = ref().ref_build_sequence_batch(q, kp, _ptr(c[0]), _ptr(c[1]), _ptr(c[2]), _ptr(c[3]),
                                        _ptr(qn), _ptr(qt), l, self_edge_index, _ptr(ni),
                                        _ptr(ei), _ptr(dt), _ptr(vl), _ptr(tr))
    if rc:
        _ref_err(rc)
    return dict(node_index=ni.reshape(q, l), edge_index=ei.reshape(q, l),
                time_delta=dt.reshape(q, l), valid_len=vl, target_row=tr)


def ref_build_mask(valid_len, target_row, l, kind):
    kinds = {"causal": 0, "tgat": 1, "self_loop": 2}
    q = len(valid_len)
    mask = np.zeros(q * l * l, np.float64)
    vl = np.ascontiguousarray(valid_len, dtype=np.int64)
    tr = np.ascontiguousarray(target_row, dtype=np.int64)
    rc = ref().ref_build_mask(q, l, _ptr(vl), _ptr(tr), kinds[kind], _ptr(mask))
    if rc:
        _ref_err(rc)
    return mask.reshape(q * l, l)


# ---------------------------------------------------------------------- assemble_inputs
def assemble_inputs(node_index, edge_index, time_delta, valid_len, node_table, edge_table,
                    omega, phi, concat):
    """Restatement of tgf::assemble_inputs (proj/src/attention.cpp:414-451) in numpy fp64:
    z[b*l+j] for j < valid_len[b] = node_table[ni] + edge_table[ei] + cos(omega*dt + phi)
    (sum) or [node_table[ni] | edge_table[ei] | cos(omega*dt + phi)] (concat); other rows 0.
    Raises OracleError on an index outside its table (attention.cpp:427-431)."""
    ni = np.asarray(node_index, np.int64)
    ei = np.asarray(edge_index, np.int64)
    dt = np.asarray(time_delta, np.float64)
    q, l = ni.shape
    vl = np.asarray(valid_len, np.int64)
    live = np.arange(l)[None, :] < vl[:, None]
    nt = np.asarray(node_table, np.float64)
    et = np.asarray(edge_table, np.float64)
    if np.any(live & ((ni < 0) | (ni >= len(nt)) | (ei < 0) | (ei >= len(et)))):
        raise OracleError(1, "sequence index outside embedding tables")
    om = np.asarray(omega, np.float64).reshape(-1)
    ph = np.asarray(phi, np.float64).reshape(-1)
    nrow = nt[np.where(live, ni, 0)]
    erow = et[np.where(live, ei, 0)]
    # omega * dt + phi is contracted to one fma by the reference's compiler (-march with FMA,
    # GCC's default -ffp-contract=fast) and by nvcc: emulate the single rounding in extended
    # precision.  Then glibc cos (math.cos, = std::cos); numpy's vectorised cos is less
    # accurate for the large arguments omega * dt reaches.
    ld = np.longdouble
    arg = (om.astype(ld)[None, None, :] * dt.astype(ld)[:, :, None]
           + ph.astype(ld)[None, None, :]).astype(np.float64)
    enc = np.frompyfunc(math.cos, 1, 1)(arg).astype(np.float64)
    z = (np.concatenate([nrow, erow, enc], axis=2) if concat else (nrow + erow) + enc)
    z[~live] = 0.0
    return z.reshape(q * l, -1)


def ref_assemble_inputs(node_index, edge_index, time_delta, valid_len, node_table, edge_table,
                        omega, phi, concat):
    """The reference's own assemble_inputs (oracle/_ref, attention.cpp compiled in place)."""
    ni = np.ascontiguousarray(node_index, np.int64)
    ei = np.ascontiguousarray(edge_index, np.int64)
    dt = np.ascontiguousarray(time_delta, np.float64)
    vl = np.ascontiguousarray(valid_len, np.int64)
    nt = np.ascontiguousarray(node_table, np.float64)
    et = np.ascontiguousarray(edge_table, np.float64)
    om = np.ascontiguousarray(omega, np.float64).reshape(-1)
    ph = np.ascontiguousarray(phi, np.float64).reshape(-1)
    q, l = ni.shape
    d_v, d_e, d_t = nt.shape[1], et.shape[1], len(om)
    d = d_v + d_e + d_t if concat else d_t
    z = np.zeros((q * l, d), np.float64)
    rc = ref().ref_assemble_inputs(q, l, _ptr(ni), _ptr(ei), _ptr(dt), _ptr(vl), _ptr(nt),
                                   len(nt), _ptr(et), len(et), _ptr(om), _ptr(ph), d_v, d_e, d_t,
                                   1 if concat else 0, _ptr(z))
    if rc:
        _ref_err(rc)
    return z


# ---------------------------------------------------------------------- CSV ingestion
def ref_train_queries(events, num_nodes, batch_size, neg_per_pos, workers, batch_seed):
    """The reference's own make_batches (training.cpp:157-182, compiled in oracle/_ref), split
    and laid out per call as train_epoch + forward_concat do (ref_harness.cpp)."""
    events = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
    n = len(events)
    q = n * (2 + neg_per_pos)
    nodes = np.zeros(max(q, 1), np.int64)
    times = np.zeros(max(q, 1), np.float64)
    tot = np.zeros(1, np.int64)
    st = ref().ref_stream_create(_ptr(events), n, num_nodes)
    try:
        rc = ref().ref_train_queries(st, batch_size, neg_per_pos, workers, num_nodes,
                                     batch_seed, _ptr(nodes), _ptr(times), _ptr(tot))
    finally:
        ref().ref_stream_free(st)
    if rc:
        raise OracleError(rc, ref().ref_last_error().decode())
    return nodes[:int(tot[0])], times[:int(tot[0])]


def ref_load_csv(path, has_features=False):
    """The reference's own load_csv (event_stream.cpp:85-154, compiled in oracle/_ref) ->
    (events, num_nodes, features [n, d_e]).  Raises OracleError(code, message) with code 1
    ValidationError, 6 ParseError (the reference's message texts)."""
    n, v, de = (np.zeros(1, np.int64) for _ in range(3))
    rc = ref().ref_load_csv(path.encode(), 1 if has_features else 0, _ptr(n), _ptr(v), _ptr(de),
                            None, None)
    if rc:
        raise OracleError(rc, ref().ref_last_error().decode())
    ev = np.zeros(int(n[0]), dtype=EVENT_DTYPE)
    feats = np.zeros((int(n[0]), int(de[0])), np.float64)
    rc = ref().ref_load_csv(path.encode(), 1 if has_features else 0, _ptr(n), _ptr(v), _ptr(de),
                            _ptr(ev) if len(ev) else _ptr(np.zeros(1, EVENT_DTYPE)),
                            _ptr(feats) if feats.size else None)
    if rc:
        raise OracleError(rc, ref().ref_last_error().decode())
    return ev, int(v[0]), feats


def from_chars(strings, kind):
    """std::from_chars over a list of byte strings (oracle/fromchars.cpp): (ok[n], values[n])
    with ok False where load_csv's parse_int / parse_real would throw."""
    n = len(strings)
    ok = np.zeros(n, bool)
    vals = np.zeros(n, np.float64 if kind == "real" else np.int64)
    f = lib().orc_from_chars_f64 if kind == "real" else lib().orc_from_chars_i64
    out = (C.c_double if kind == "real" else C.c_int64)()
    for i, b in enumerate(strings):
        if f(b, len(b), C.byref(out)) == 0:
            ok[i] = True
            vals[i] = out.value
    return ok, vals
