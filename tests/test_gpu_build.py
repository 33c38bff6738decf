"""GPU parity: T-CSR build (CUDA, through the C ABI) vs the reference's golden vectors and the
CPU oracle.  Bit-exact: indptr/nbr/eid int64 equal, ts compared bit-for-bit."""
import glob
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, events_of

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    from paper_2409_05477_b200 import tgformer
    return tgformer


def assert_same(g, want, tag=""):
    assert np.array_equal(g.indptr, want["indptr"]), tag
    assert np.array_equal(g.neighbor_ids, want["nbr"]), tag
    assert np.array_equal(g.edge_ids, want["eid"]), tag
    assert g.timestamps.view(np.uint64).tobytes() == np.asarray(want["ts"]).view(np.uint64).tobytes(), tag


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "build_*.npz"))))
def test_build_matches_reference_golden(T, path):
    g = dict(np.load(path))
    ev = events_of(g["events"])
    V = int(g["num_nodes"])
    for rev in (0, 1):
        want = {k: g[f"rev{rev}_{k}"] for k in ("indptr", "nbr", "eid", "ts")}
        got = T.build_sequential(T.EventStream(ev, V), bool(rev))
        assert_same(got, want, (path, rev))
        got.validate()
        gp = T.build_parallel(T.EventStream(ev, V), bool(rev), 8)
        assert_same(gp, want, (path, rev, "parallel"))


def test_reference_unit_known_answers(T):
    """proj/tests/test_tcsr.cpp:50-97"""
    three = T.EventStream(np.array([(1, 0, 2, 3.0), (2, 1, 2, 4.0), (0, 0, 1, 5.0)],
                                   dtype=T.EVENT_DTYPE), 3)
    g = T.build_sequential(three, False)
    assert g.indptr.tolist() == [0, 2, 3, 3]
    assert g.timestamps[:2].tolist() == [3.0, 5.0] and g.neighbor_ids[:2].tolist() == [2, 1]
    g = T.build_sequential(three, True)
    assert g.num_entries() == 6 and g.indptr.tolist() == [0, 2, 4, 6]
    assert g.neighbor_ids[4:6].tolist() == [0, 1] and g.timestamps[4:6].tolist() == [3.0, 4.0]
    sl = T.build_sequential(T.EventStream(np.array([(0, 1, 1, 4.0)], dtype=T.EVENT_DTYPE), 2), True)
    assert sl.degree(0) == 0 and sl.degree(1) == 2
    assert sl.edge_ids.tolist() == [0, 0] and sl.neighbor_ids[0] == 1
    empty = T.build_sequential(T.EventStream(np.zeros(0, T.EVENT_DTYPE), 4), True)
    assert empty.indptr.tolist() == [0, 0, 0, 0, 0] and empty.num_entries() == 0


def test_build_errors_match_reference(T):
    with open(os.path.join(GOLDEN, "errors.json")) as f:
        errs = json.load(f)
    bad = T.EventStream(np.array([(0, 0, 7, 1.0)], dtype=T.EVENT_DTYPE), 2)
    with pytest.raises(T.ValidationError, match=errs["bad_endpoint"]):
        T.build_sequential(bad, False)
    with pytest.raises(T.ValidationError, match=errs["bad_endpoint"]):
        T.build_parallel(bad, False, 2)
    ok = T.EventStream(np.array([(0, 0, 1, 1.0)], dtype=T.EVENT_DTYPE), 2)
    with pytest.raises(T.ValidationError, match=errs["bad_threads"]):
        T.build_parallel(ok, True, 0)
    # first offending event in stream order is reported (check_endpoints, tcsr.cpp:44-50)
    ev = np.array([(10, 0, 1, 1.0), (11, 0, 9, 2.0), (12, -1, 0, 3.0)], dtype=T.EVENT_DTYPE)
    with pytest.raises(T.ValidationError, match="event 11 endpoint out of range"):
        T.build_sequential(T.EventStream(ev, 2), True)


def _acceptance_stream(O, i):
    """proj/tests/acceptance.cpp:44-55 schedule_stream(i)"""
    if i < 90:
        n = 1000 + O.mix64(i) % 9000
        v = 50 + O.mix64(i + 7) % 2000
        return O.make_random_stream(n, v, 1000 + i), v
    if i < 98:
        return O.make_random_stream(100000, 20000, 2000 + i), 20000
    return O.make_random_stream(1000000, 100000, 3000 + i), 100000


@pytest.mark.parametrize("i", [0, 1, 2, 17, 45, 89, 90, 97, 98, 99])
def test_acceptance_schedule_vs_oracle(T, oracle_mod, i):
    """acceptance `builder` criterion (acceptance.cpp:63-95) on a subset of its schedule:
    includes the 1e6-edge / 1e5-node streams, which exceed the shared-memory cursor budget and
    take the large-V path."""
    ev, v = _acceptance_stream(oracle_mod, i)
    for rev in (False, True):
        want = oracle_mod.build(ev, v, rev)
        got = T.build_sequential(T.EventStream(ev, v), rev)
        assert_same(got, want, (i, rev))
        assert got.build_path == (2 if v > 45000 else 0)


@pytest.mark.parametrize("V", [700, 120000])
def test_unsorted_streams_take_the_general_path(T, oracle_mod, V):
    rng = np.random.default_rng(V)
    ev = oracle_mod.make_random_stream(60000, V, 77)
    shuffled = ev[rng.permutation(len(ev))].copy()
    for rev in (False, True):
        want = oracle_mod.build(shuffled, V, rev)
        got = T.build_sequential(T.EventStream(shuffled, V), rev)
        assert_same(got, want, (V, rev))
        assert got.build_path == (1 if V <= 45000 else 2)


def test_degenerate_shapes(T, oracle_mod):
    # one node, all self-loops; node ids at the boundary; V much larger than used
    for ev, V in ((oracle_mod.events_from([0] * 50, [0] * 50, np.arange(50.0)), 1),
                  (oracle_mod.events_from([4, 0, 4], [0, 4, 4], [1.0, 1.0, 1.0]), 5),
                  (oracle_mod.events_from([3, 2], [2, 3], [0.0, 0.0]), 45000),
                  (oracle_mod.events_from([3, 2], [2, 3], [0.0, 0.0]), 45001)):
        for rev in (False, True):
            assert_same(T.build_sequential(T.EventStream(ev, V), rev), oracle_mod.build(ev, V, rev))


def test_gdelt_shape_prefix_vs_oracle(T, oracle_mod):
    """GDELT-shaped (V = 16,682, Zipf 1.2) 8M-event prefix: full bit-exact comparison."""
    ev = oracle_mod.make_random_stream(8_000_000, 16682, 42)
    want = oracle_mod.build(ev, 16682, True)
    got = T.build_sequential(T.EventStream(ev, 16682), True)
    assert_same(got, want)


def test_full_gdelt_size_properties():
    """Full GDELT-shaped build (191,290,882 events, rev=1) on the device: size-independent
    properties -- validate() (sorted slices, ranges, indptr endpoints), degree histogram equal
    to a bincount of the endpoints, and the multiset checksum of (nbr, eid) per entry equal to
    that of the emitted entries."""
    import torch
    from paper_2409_05477_b200 import device as D
    E, V = 191_290_882, 16682
    ev = D.random_stream(E, V, 42)
    g = D.build(ev, V, True)
    g.validate()
    ip, nb, ed, ts = D.graph_tensors(g)
    raw = ev.view(torch.int64).view(E, 4)
    deg = torch.bincount(raw[:, 1], minlength=V) + torch.bincount(raw[:, 2], minlength=V)
    assert torch.equal(torch.diff(ip), deg)
    # checksum of checksums: per-entry hash summed (order-independent), equal on both sides
    def h(a, b):
        return ((a * 0x9E3779B1 + b * 0x85EBCA77) & 0xFFFFFFFF).sum()
    want = h(raw[:, 2], raw[:, 0]) + h(raw[:, 1], raw[:, 0])
    assert int(h(nb, ed)) == int(want)


def test_permuted_ids_and_reverse_settings(T, oracle_mod):
    """Hub nodes at arbitrary ids (a random relabelling of a Zipf stream), both reverse
    settings, several sizes: the builder's hot-node selection must not depend on ids."""
    rng = np.random.default_rng(8)
    for E, V, seed in ((300_000, 5000, 3), (2_000_000, 16682, 4), (50_000, 65535, 5)):
        ev = oracle_mod.make_random_stream(E, V, seed)
        perm = rng.permutation(V)
        ev["src"] = perm[ev["src"]]
        ev["dst"] = perm[ev["dst"]]
        for rev in (True, False):
            assert_same(T.build_parallel(T.EventStream(ev, V), rev, 4), oracle_mod.build(ev, V, rev))


def test_rebuild_refreshes_lazily_widened_columns(oracle_mod):
    """The tile scatter writes 16-byte gather records instead of the int64 nbr / eid columns;
    those are widened on demand (export, device views, validate).  A rebuild from another
    stream of the same shape must invalidate them: views taken after the rebuild, the export
    and the sampler all see the new graph."""
    import torch
    from paper_2409_05477_b200 import device as D
    E, V = 400_000, 3000
    ev1 = D.random_stream(E, V, 21)
    ev2 = D.random_stream(E, V, 22)
    g = D.build(ev1, V, True)
    for seed, ev in ((21, ev1), (22, ev2), (21, ev1)):
        D.rebuild(g, ev, trusted=True)
        og = oracle_mod.build(oracle_mod.make_random_stream(E, V, seed), V, True)
        ip, nb, ed, ts = D.graph_tensors(g)
        assert np.array_equal(ip.cpu().numpy(), og["indptr"])
        assert np.array_equal(nb.cpu().numpy(), og["nbr"])
        assert np.array_equal(ed.cpu().numpy(), og["eid"])
        assert np.array_equal(ts.cpu().numpy(), og["ts"])
        g.validate()
        nodes, times = D.make_queries(ev, 0, 20_000, 600, V)
        out = D.sample_assemble(g, nodes, times, 10, "recent", 9, 11, E + 1, index64=True,
                                dt64=True)
        want = oracle_mod.sample_assemble(og, nodes.cpu().numpy(), times.cpu().numpy(), 10,
                                          "recent", 9, 11, E + 1)
        assert np.array_equal(out["node_index"].cpu().numpy(), want["node_index"])
        assert np.array_equal(out["edge_index"].cpu().numpy(), want["edge_index"])
        assert np.array_equal(out["time_delta64"].cpu().numpy(), want["time_delta"])
    torch.cuda.synchronize()


@pytest.mark.parametrize("variant", ["50", "45", "10"])
def test_scatter_variants_build_the_same_tcsr(variant):
    """The A/B scatter variants (TGFX_SCATTER_VARIANT, read once per process, so each runs in
    its own process) build the default's T-CSR bit for bit on a GDELT-like shape (Zipf hubs,
    cold tail, reverse = 1): 50 = one pass over hub labels + a warp-sorted remainder."""
    import os
    import subprocess
    import sys
    code = (
        "import sys, hashlib; sys.path.insert(0, %r)\n"
        "from paper_2409_05477_b200 import device as D\n"
        "ev = D.random_stream(3_000_000, 16682, 42)\n"
        "g = D.build(ev, 16682, True)\n"
        "h = hashlib.sha256()\n"
        "for t in D.graph_tensors(g): h.update(t.cpu().numpy().tobytes())\n"
        "print(h.hexdigest())\n" % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    out = {}
    for v in ("43", variant):
        env = dict(os.environ, TGFX_SCATTER_VARIANT=v)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        out[v] = r.stdout.strip().splitlines()[-1]
    assert out[variant] == out["43"]


def test_pageable_host_round_trip_through_the_staging_ring(T):
    """Host-buffer build from a pageable 640 MB event array and export into pageable 320 MB
    columns (both above the 256 MB threshold of the pinned staging ring: host threads fill and
    drain 64 MB chunks beside the DMA) equal the device-buffer build's columns bit for bit."""
    import torch
    from paper_2409_05477_b200 import device as D
    E, V = 20_000_000, 16682
    st = T.make_random_stream(E, V, 5)  # host (pageable) events
    assert st.events.nbytes >= 256 << 20
    g = T.build_parallel(st, True, 8)
    dev_ev = torch.from_numpy(st.events.view(np.uint8).reshape(-1)).cuda()
    gd = D.build(dev_ev, V, True)
    ip, nb, ed, ts = (t.cpu().numpy() for t in D.graph_tensors(gd))
    assert g.neighbor_ids.nbytes >= 256 << 20
    assert np.array_equal(g.indptr, ip)
    assert np.array_equal(g.neighbor_ids, nb)
    assert np.array_equal(g.edge_ids, ed)
    assert g.timestamps.tobytes() == ts.view(np.float64).tobytes()


def test_large_v_fused_key_pass_errors_and_reuse(T, oracle_mod):
    """Large-V path (V > 45,000): the flags pass that also writes the sort keys reports the
    first bad endpoint with the reference's text, and the graph built right after from a valid
    stream (same allocator, buffers reused) is bit-exact."""
    V = 200_000
    ev = oracle_mod.make_random_stream(300_000, V, 31)
    bad = ev.copy()
    bad["dst"][123_456] = V + 3
    for rev in (False, True):
        with pytest.raises(T.ValidationError, match="event %d endpoint out of range"
                           % int(bad["edge_id"][123_456])):
            T.build_parallel(T.EventStream(bad, V), rev, 4)
        got = T.build_parallel(T.EventStream(ev, V), rev, 4)
        assert got.build_path == 2
        assert_same(got, oracle_mod.build(ev, V, rev), rev)
