"""GPU parity: sampler + fused assembler (CUDA via the C ABI) vs the reference's golden vectors
and the CPU oracle.  Indices bit-exact; fp64 deltas bit-exact; fp32 deltas equal to the fp64
reference rounded to nearest (|rel err| <= 2^-24 < 1e-6, the north-star tolerance)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden

pytestmark = pytest.mark.gpu

RTOL = 1e-6  # north_star: fp32 time deltas within 1e-6 relative


@pytest.fixture(scope="module")
def T():
    from paper_2409_05477_b200 import tgformer
    return tgformer


def check_rows(got, want, tag=""):
    """got: int32/fp32 rows (+ optional fp64); want: reference int64/fp64 SequenceBatch."""
    assert np.array_equal(got["node_index"].astype(np.int64), want["node_index"]), tag
    assert np.array_equal(got["edge_index"].astype(np.int64), want["edge_index"]), tag
    assert np.array_equal(got["valid_len"].astype(np.int64), want["valid_len"]), tag
    ref = want["time_delta"]
    d32 = got["time_delta"].astype(np.float64)
    with np.errstate(invalid="ignore", divide="ignore"):
        err = np.abs(d32 - ref) / np.abs(ref)
    assert np.all((d32 == ref) | (err <= RTOL)), (tag, float(np.nanmax(err)))
    assert np.array_equal(got["time_delta"], ref.astype(np.float32)), tag  # fp64->fp32 RN
    if "time_delta64" in got:
        assert got["time_delta64"].view(np.uint64).tobytes() == ref.view(np.uint64).tobytes(), tag


@pytest.mark.parametrize("name", ["sample_4000_150_31", "sample_3000_40_32"])
def test_sampler_matches_reference_golden(T, oracle_mod, name):
    g = golden(name)
    e, v, seed = (int(x) for x in name.split("_")[1:])
    stream = T.make_random_stream(e, v, seed)
    graph = T.build_sequential(stream, True)
    for strat in ("recent", "random"):
        for k in (1, 6, 20, 40):
            for tag, nn, tt in (("rand", g["qn"], g["qt"]), ("event", g["en"], g["et"])):
                c, nb, ed, ts = T.sample_batch_arrays(graph, nn, tt, k, strat, 9)
                p = f"{strat}_k{k}_{tag}"
                assert np.array_equal(c, g[p + "_counts"]), p
                assert np.array_equal(nb, g[p + "_nbr"]), p
                assert np.array_equal(ed, g[p + "_eid"]), p
                assert np.array_equal(ts, g[p + "_ts"]), p
    for strat, k, l in (("recent", 10, 11), ("random", 20, 21), ("random", 10, 5),
                        ("recent", 40, 33)):
        got = T.sample_assemble(graph, g["en"], g["et"], k, strat, 9, l, e + 1, dt64=True)
        want = {kk: g[f"asm_{strat}_k{k}_l{l}_{kk}"] for kk in
                ("node_index", "edge_index", "time_delta", "valid_len")}
        check_rows(got, want, (name, strat, k, l))


def test_two_hop_matches_reference_golden(T):
    g = golden("two_hop_6000_200_51")
    graph = T.build_sequential(T.make_random_stream(6000, 200, 51), True)
    for strat in ("recent", "random"):
        h1, h2 = T.sample_two_hop(graph, g["roots"], g["rtimes"], 10, 10, strat, 9, 11, 6001,
                                  seed2=0x5eed2)
        check_rows(h1, {kk: g[f"{strat}_hop1_{kk}"] for kk in
                        ("node_index", "edge_index", "time_delta", "valid_len")}, strat)
        q = len(g["roots"])
        flat = {kk: h2[kk].reshape(q * 10, *h2[kk].shape[2:]) for kk in h2}
        want = {kk: g[f"{strat}_hop2_{kk}"].reshape(q * 10, *g[f"{strat}_hop2_{kk}"].shape[2:])
                for kk in ("node_index", "edge_index", "time_delta", "valid_len")}
        check_rows(flat, want, strat)


def test_reference_unit_known_answers(T):
    """proj/tests/test_sampler.cpp:32-87, 264-272"""
    ev = np.array([(1, 0, 2, 3.0), (2, 1, 2, 4.0), (0, 0, 1, 5.0)], dtype=T.EVENT_DTYPE)
    g = T.build_sequential(T.EventStream(ev, 3), False)
    mid = T.sample_recent(g, 0, 4.0, 5)
    assert [(e.neighbor, e.timestamp) for e in mid.neighbors] == [(2, 3.0)]
    assert T.sample_recent(g, 0, 3.0, 5).neighbors == []
    assert T.sample_recent(g, 0, 0.5, 5).neighbors == []
    assert [e.timestamp for e in T.sample_recent(g, 0, 99.0, 5).neighbors] == [3.0, 5.0]
    got = T.sample_recent(g, 0, 5.0, 10)  # strict inequality
    assert [e.timestamp for e in got.neighbors] == [3.0]
    for seed in range(20):
        assert all(e.timestamp < 5.0 for e in T.sample_random(g, 0, 5.0, 1, seed).neighbors)
    for seed in (0, 7, 123456):
        assert [e.timestamp for e in T.sample_random(g, 0, 99.0, 5, seed).neighbors] == [3.0, 5.0]
    ten = np.array([(i, 0, i + 1, float(i)) for i in range(10)], dtype=T.EVENT_DTYPE)
    g10 = T.build_sequential(T.EventStream(ten, 12), False)
    assert [e.timestamp for e in T.sample_recent(g10, 0, 100.0, 3).neighbors] == [7.0, 8.0, 9.0]


def test_uniformity_over_seeds(T):
    """proj/tests/test_sampler.cpp:144-165 and acceptance.cpp:120-147 (distributional)."""
    ev = np.array([(i, 0, i + 1, float(i)) for i in range(100)], dtype=T.EVENT_DTYPE)
    g = T.build_sequential(T.EventStream(ev, 101), False)
    seeds = 10000
    hits = np.zeros(100)
    # one batch per seed would be slow; stream_base varies the stream instead of the seed, and
    # a second pass varies the seed with a fixed stream
    for s in range(0, seeds, 1000):
        c, nb, ed, ts = T.sample_batch_arrays(g, np.zeros(1000, np.int64), np.full(1000, 1e9),
                                              10, "random", 12345, stream_base=s)
        assert (c == 10).all()
        np.add.at(hits, ed.ravel(), 1)
    share = hits / (seeds * 10)
    appear = hits / seeds
    assert np.abs(share - 0.01).max() <= 0.01 and np.abs(appear - 0.1).max() <= 0.02


def test_sampler_errors_match_reference(T):
    with open(os.path.join(GOLDEN, "errors.json")) as f:
        errs = json.load(f)
    ev = np.array([(1, 0, 2, 3.0), (2, 1, 2, 4.0), (0, 0, 1, 5.0)], dtype=T.EVENT_DTYPE)
    g = T.build_sequential(T.EventStream(ev, 3), False)
    with pytest.raises(T.ValidationError, match=errs["bad_node"]):
        T.sample_recent(g, 99, 1.0, 3)
    with pytest.raises(T.ValidationError, match=errs["bad_k"]):
        T.sample_recent(g, 0, 1.0, 0)
    with pytest.raises(T.ValidationError, match="node and time lists differ in length"):
        T.sample_batch(g, [0, 1], [1.0], 3)
    with pytest.raises(T.ValidationError, match=errs["bad_l"]):
        T.sample_assemble(g, [0], [1.0], 3, "recent", 0, 1, 4)
    with pytest.raises(T.ValidationError, match="query node -1 out of range"):
        T.sample_batch(g, [0, 1, -1, 7], [1.0] * 4, 3)
    with pytest.raises(T.ValidationError):
        T.parse_strategy("nope")


def _workload(O, E, V, seed, batch, n_events=None):
    ev = O.make_random_stream(E, V, seed)
    e1 = E if n_events is None else n_events
    nodes, times = O.make_queries(ev, 0, e1, batch, V)
    return ev, nodes, times


@pytest.mark.parametrize("strat,k,l", [("recent", 10, 11), ("random", 20, 21), ("recent", 1, 2),
                                       ("random", 64, 33), ("random", 128, 129),
                                       ("recent", 128, 11), ("random", 200, 40)])
def test_wikipedia_shape_vs_oracle(T, oracle_mod, strat, k, l):
    """Config W (9,227 nodes, 157,474 edges) event-derived queries, all events."""
    ev, nodes, times = _workload(oracle_mod, 157474, 9227, 42, 600)
    og = oracle_mod.build(ev, 9227, True)
    graph = T.build_sequential(T.EventStream(ev, 9227), True)
    for b0 in (0, 200 * 1800):
        nn, tt = nodes[b0:b0 + 1800 * 20], times[b0:b0 + 1800 * 20]
        want = oracle_mod.sample_assemble(og, nn, tt, k, strat, 9 + b0, l, 157475,
                                          stream_base=b0)
        got = T.sample_assemble(graph, nn, tt, k, strat, 9 + b0, l, 157475, stream_base=b0,
                                dt64=True)
        check_rows(got, want, (strat, k, l, b0))
        cw = oracle_mod.sample_batch(og, nn, tt, k, strat, 9, stream_base=b0)
        cg = T.sample_batch_arrays(graph, nn, tt, k, strat, 9, stream_base=b0)
        for a, b in zip(cg, cw):
            assert np.array_equal(a, b), (strat, k)


def test_lastfm_shape_uniform20_vs_oracle(T, oracle_mod):
    """Config L (1,980 nodes, 1.29M edges, heavy hub): uniform-20, batch 4,000, l = 21."""
    ev, nodes, times = _workload(oracle_mod, 1293103, 1980, 42, 4000, n_events=40000)
    og = oracle_mod.build(ev, 1980, True)
    graph = T.build_sequential(T.EventStream(ev, 1980), True)
    for b in range(0, 10):  # 10 batches of 12,000 queries, seed 9 + b, stream = index in batch
        nn, tt = nodes[b * 12000:(b + 1) * 12000], times[b * 12000:(b + 1) * 12000]
        want = oracle_mod.sample_assemble(og, nn, tt, 20, "random", 9 + b, 21, 1293104)
        got = T.sample_assemble(graph, nn, tt, 20, "random", 9 + b, 21, 1293104, dt64=True)
        check_rows(got, want, b)


def test_edge_case_queries(T, oracle_mod):
    ev = oracle_mod.make_random_stream(5000, 60, 5)
    og = oracle_mod.build(ev, 60, True)
    graph = T.build_sequential(T.EventStream(ev, 60), True)
    rng = np.random.default_rng(1)
    nodes = rng.integers(0, 60, 4500)
    times = np.concatenate([np.full(500, np.nan), np.full(500, -np.inf), np.full(500, np.inf),
                            np.full(500, 0.0), np.full(500, -0.0), ev["timestamp"][:1500],
                            rng.uniform(0, 3000, 500)])
    for strat, k, l in (("recent", 5, 6), ("random", 5, 3), ("random", 33, 40),
                        ("recent", 300, 301)):
        want = oracle_mod.sample_assemble(og, nodes, times, k, strat, 3, l, 5001)
        got = T.sample_assemble(graph, nodes, times, k, strat, 3, l, 5001, dt64=True)
        check_rows(got, want, (strat, k, l))
    # empty graph and single-node graph
    e0 = T.build_sequential(T.EventStream(np.zeros(0, T.EVENT_DTYPE), 3), True)
    out = T.sample_assemble(e0, [0, 1, 2], [1.0, 2.0, 3.0], 4, "recent", 0, 5, 1)
    assert out["valid_len"].tolist() == [1, 1, 1]
    assert out["node_index"][:, 0].tolist() == [1, 2, 3]
    out = T.sample_assemble(e0, [], [], 4, "random", 0, 5, 1)
    assert out["valid_len"].shape == (0,)


def test_fused_int64_outputs_and_device_api(T, oracle_mod):
    import torch
    from paper_2409_05477_b200 import device as D
    ev = D.random_stream(200000, 5000, 4001)
    g = D.build(ev, 5000, True)
    nodes, times = D.make_queries(ev, 0, 200000, 600, 5000)
    h_ev = oracle_mod.make_random_stream(200000, 5000, 4001)
    hn, ht = oracle_mod.make_queries(h_ev, 0, 200000, 600, 5000)
    assert np.array_equal(nodes.cpu().numpy(), hn) and np.array_equal(times.cpu().numpy(), ht)
    og = oracle_mod.build(h_ev, 5000, True)
    out = D.sample_assemble(g, nodes, times, 10, "recent", 0, 11, 200001, index64=True, dt64=True)
    want = oracle_mod.sample_assemble(og, hn, ht, 10, "recent", 0, 11, 200001)
    assert np.array_equal(out["node_index"].cpu().numpy(), want["node_index"])
    assert np.array_equal(out["edge_index"].cpu().numpy(), want["edge_index"])
    assert np.array_equal(out["valid_len"].cpu().numpy(), want["valid_len"])
    assert np.array_equal(out["time_delta64"].cpu().numpy(), want["time_delta"])
    torch.cuda.synchronize()


def test_gdelt_full_size_sampler_vs_oracle(T, oracle_mod):
    """Full GDELT-shaped T-CSR (191,290,882 events, rev=1; hub slice ~78 M entries) built on
    the device; recent-10 rows for event-derived queries from the start, middle and end of the
    stream and uniform-20 rows for a slice of them, checked bit-exactly against the oracle run
    on the exported T-CSR (exercises the interpolation search on the deep hub slices)."""
    import torch
    from paper_2409_05477_b200 import device as D
    E, V = 191_290_882, 16682
    ev = D.random_stream(E, V, 42)
    g = D.build(ev, V, True)
    ip, nb, ed, ts = D.graph_tensors(g)
    og = {"indptr": ip.cpu().numpy(), "nbr": nb.cpu().numpy(), "eid": ed.cpu().numpy(),
          "ts": ts.cpu().numpy(), "num_nodes": V, "num_edges": E}
    for e0 in (0, E // 2, E - 60_000):
        nodes, times = D.make_queries(ev, e0, e0 + 60_000, 600, V)
        hn, ht = nodes.cpu().numpy(), times.cpu().numpy()
        out = D.sample_assemble(g, nodes, times, 10, "recent", 9, 11, E + 1, dt64=True)
        want = oracle_mod.sample_assemble(og, hn, ht, 10, "recent", 9, 11, E + 1)
        got = {k: v.cpu().numpy() for k, v in out.items()}
        check_rows(got, want, ("recent", e0))
        out = D.sample_assemble(g, nodes[:30000], times[:30000], 20, "random", 9, 21, E + 1,
                                dt64=True)
        want = oracle_mod.sample_assemble(og, hn[:30000], ht[:30000], 20, "random", 9, 21, E + 1)
        got = {k: v.cpu().numpy() for k, v in out.items()}
        check_rows(got, want, ("random", e0))
    del og, ip, nb, ed, ts
    torch.cuda.synchronize()


def test_exact_search_on_unsorted_or_nan_slices(T, oracle_mod):
    """A T-CSR imported from the host whose slices hold NaN timestamps or are out of order is
    outside the interpolation search's precondition: the sampler must then replay
    std::lower_bound's own bisection (sampler.cpp:16-20) and match the oracle exactly."""
    ev = oracle_mod.make_random_stream(20000, 90, 77)
    og = oracle_mod.build(ev, 90, True)
    rng = np.random.default_rng(3)
    ts = og["ts"].copy()
    ts[rng.choice(len(ts), 300, replace=False)] = np.nan        # NaN entries
    ip = og["indptr"]
    for u in range(0, 90, 7):                                   # reversed slices
        ts[ip[u]:ip[u + 1]] = ts[ip[u]:ip[u + 1]][::-1].copy()
    bad = dict(og, ts=ts)
    g = T.TCsr.from_host(90, 20000, True, og["indptr"], og["nbr"], og["eid"], ts)
    nodes = rng.integers(0, 90, 5000)
    times = np.concatenate([rng.uniform(0, 10000, 4000), np.full(500, np.nan),
                            ev["timestamp"][:500]])
    for strat, k, l in (("recent", 10, 11), ("random", 12, 13)):
        want = oracle_mod.sample_assemble(bad, nodes, times, k, strat, 5, l, 20001)
        got = T.sample_assemble(g, nodes, times, k, strat, 5, l, 20001, dt64=True)
        assert np.array_equal(got["node_index"].astype(np.int64), want["node_index"]), strat
        assert np.array_equal(got["valid_len"].astype(np.int64), want["valid_len"]), strat
        # NaN entries: compare as values (the payload bits of a NaN result are not specified)
        assert np.array_equal(got["time_delta64"], want["time_delta"], equal_nan=True), strat


def test_batched_launch_equals_one_call_per_batch(T, oracle_mod):
    """tgfx_sample_assemble_batched_device: many forward_concat batches in one launch, batch b
    sampled with seeds[b] and stream = index within the batch -- must equal one
    sample_batch + build_sequence_batch per batch (the oracle, and the per-batch device call)."""
    import torch
    from paper_2409_05477_b200 import device as D
    E, V, B = 200_000, 1980, 4000
    ev = D.random_stream(E, V, 42)
    g = D.build(ev, V, True)
    nodes, times = D.make_queries(ev, 0, 60_000, B, V)
    qb = 3 * B
    nb = -(-nodes.numel() // qb)
    seeds = torch.tensor([(0x9E3779B97F4A7C15 * (b + 1)) & (2**63 - 1) for b in range(nb)],
                         dtype=torch.int64, device="cuda")
    h_ev = ev.cpu().numpy().view(oracle_mod.EVENT_DTYPE)
    og = oracle_mod.build(h_ev, V, True)
    hn, ht = nodes.cpu().numpy(), times.cpu().numpy()
    for strat, k, l in (("random", 20, 21), ("recent", 10, 11), ("random", 64, 40)):
        out = D.sample_assemble_batched(g, nodes, times, qb, k, strat, seeds, l, E + 1, dt64=True)
        for b in range(nb):
            s, e = b * qb, min(nodes.numel(), (b + 1) * qb)
            want = oracle_mod.sample_assemble(og, hn[s:e], ht[s:e], k, strat,
                                              int(seeds[b].item()), l, E + 1)
            got = {kk: v[s:e].cpu().numpy() for kk, v in out.items()}
            check_rows(got, want, (strat, b))


def test_time_buckets_on_adversarial_slices(T, oracle_mod):
    """The per-slice time buckets (build_node_dir) narrow each search to [bkt[j], bkt[j+1]];
    exactness rests on bucket_of being monotone and evaluated identically by the builder and
    the sampler.  Slices built to stress that: uniform, bursty tie clusters, all ties, a
    geometric 1.5^i spread up to 1e264, a span of a few ulps, negative times, +-inf ends,
    subnormal spans, -0.0/0.0 ties, slices just under / over the bucket threshold; queries at
    every entry time, its neighbours one ulp away, midpoints, and the bucket edges."""
    rng = np.random.default_rng(12)
    slices = [
        np.sort(rng.uniform(0, 1e4, 5000)),
        np.sort(np.concatenate([np.full(1000, 10.0), np.full(1000, 20.0), np.full(1000, 30.5),
                                rng.uniform(0, 40, 300)])),
        np.full(2000, 7.0),
        1.5 ** np.arange(1500, dtype=np.float64),
        1.0 + np.arange(100) * np.spacing(1.0),
        np.sort(rng.uniform(-1e6, -1, 3000)),
        np.concatenate([[-np.inf], np.sort(rng.uniform(0, 5, 200)), [np.inf]]),
        np.arange(64, dtype=np.float64) * 5e-324,
        np.sort(rng.uniform(0, 1, 31)),
        np.sort(rng.uniform(0, 1, 33)),
        np.array([-0.0, 0.0] * 40),
        np.zeros(0),
        np.sort(rng.exponential(1.0, 4000)) * 1e-300,
        np.sort(np.round(rng.uniform(0, 50, 6000))),
    ]
    V = len(slices)
    lens = np.array([len(s) for s in slices])
    indptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    m = int(indptr[-1])
    ts = np.concatenate(slices).astype(np.float64)
    nbr = rng.integers(0, V, m).astype(np.int64)
    eid = rng.permutation(m).astype(np.int64)
    g = T.TCsr.from_host(V, m, False, indptr, nbr, eid, ts)
    og = {"indptr": indptr, "nbr": nbr, "eid": eid, "ts": ts, "num_nodes": V, "num_edges": m}
    qn, qt = [], []
    for u, s in enumerate(slices):
        fin = s[np.isfinite(s)]
        cand = [s, np.nextafter(s, np.inf), np.nextafter(s, -np.inf), [np.inf, -np.inf, np.nan]]
        if len(fin) > 1:
            cand.append((fin[1:] + fin[:-1]) / 2)
            for R in (4, 8, 16):  # bucket edges for the bucket sizes the sampler may use
                nb = -(-len(s) // R)
                w = (fin[-1] - fin[0]) / nb
                e = fin[0] + np.arange(nb + 1) * w
                cand += [e, np.nextafter(e, np.inf), np.nextafter(e, -np.inf)]
        c = np.concatenate([np.asarray(x, np.float64) for x in cand])
        qn.append(np.full(len(c), u, np.int64))
        qt.append(c)
    nodes, times = np.concatenate(qn), np.concatenate(qt)
    for strat, k, l in (("recent", 10, 11), ("random", 12, 13), ("recent", 40, 33)):
        want = oracle_mod.sample_assemble(og, nodes, times, k, strat, 5, l, m + 1)
        got = T.sample_assemble(g, nodes, times, k, strat, 5, l, m + 1, dt64=True)
        assert np.array_equal(got["node_index"].astype(np.int64), want["node_index"]), strat
        assert np.array_equal(got["edge_index"].astype(np.int64), want["edge_index"]), strat
        assert np.array_equal(got["valid_len"].astype(np.int64), want["valid_len"]), strat
        assert np.array_equal(got["time_delta64"], want["time_delta"], equal_nan=True), strat
    c, nb, ed, tsr = T.sample_batch_arrays(g, nodes, times, 10, "recent", 5)
    cw, nw, ew, tw = oracle_mod.sample_batch(og, nodes, times, 10, "recent", 5)
    assert np.array_equal(c, cw) and np.array_equal(nb, nw) and np.array_equal(ed, ew)


@pytest.mark.parametrize("k,l", [(1, 2), (5, 3), (8, 9), (16, 5), (20, 21), (24, 32), (31, 32),
                                 (32, 11), (32, 32)])
def test_uniform_lane_kernel_int32_rows_vs_oracle(T, oracle_mod, k, l):
    """Uniform-k with int32 / fp32-only rows takes the one-query-per-lane kernel
    (k_random_lane): Floyd draws, ranks and the keep-the-most-recent-l-1 rule must match the
    oracle bit for bit, including whole-prefix queries (qm <= k), empty slices, times before
    every entry and absent hop-2 slots."""
    ev, nodes, times = _workload(oracle_mod, 120_000, 700, 13, 600, n_events=30_000)
    og = oracle_mod.build(ev, 700, True)
    graph = T.build_sequential(T.EventStream(ev, 700), True)
    rng = np.random.default_rng(k * 100 + l)
    nodes = np.concatenate([nodes, rng.integers(0, 700, 3000)])
    times = np.concatenate([times, rng.uniform(-10, ev["timestamp"][-1] + 10, 3000)])
    for b0, seed in ((0, 5), (60_000, 77)):
        nn, tt = nodes[b0:b0 + 33_000], times[b0:b0 + 33_000]
        want = oracle_mod.sample_assemble(og, nn, tt, k, "random", seed, l, 120_001,
                                          stream_base=b0)
        got = T.sample_assemble(graph, nn, tt, k, "random", seed, l, 120_001, stream_base=b0)
        assert np.array_equal(got["node_index"].astype(np.int64), want["node_index"])
        assert np.array_equal(got["edge_index"].astype(np.int64), want["edge_index"])
        assert np.array_equal(got["valid_len"].astype(np.int64), want["valid_len"])
        assert np.array_equal(got["time_delta"], want["time_delta"].astype(np.float32))


def test_uniform_lane_kernel_device_batched(T, oracle_mod):
    """The lane kernel under per-batch seeds (one launch for many forward_concat batches); its
    hop-2 use (absent virtual queries) is covered by test_two_hop_matches_reference_golden,
    whose rows are int32 / fp32."""
    import torch
    from paper_2409_05477_b200 import device as D
    E, V = 200_000, 4000
    ev = D.random_stream(E, V, 31)
    g = D.build(ev, V, True)
    h_ev = oracle_mod.make_random_stream(E, V, 31)
    og = oracle_mod.build(h_ev, V, True)
    nodes, times = D.make_queries(ev, 0, 40_000, 600, V)
    qb = 1800
    nb = -(-nodes.numel() // qb)
    seeds = torch.arange(100, 100 + nb, dtype=torch.int64, device="cuda")
    out = D.sample_assemble_batched(g, nodes, times, qb, 20, "random", seeds, 21, E + 1)
    hn, ht = nodes.cpu().numpy(), times.cpu().numpy()
    for b in range(nb):
        s, e = b * qb, min((b + 1) * qb, len(hn))
        want = oracle_mod.sample_assemble(og, hn[s:e], ht[s:e], 20, "random", 100 + b, 21, E + 1)
        assert np.array_equal(out["node_index"][s:e].cpu().numpy().astype(np.int64),
                              want["node_index"]), b
        assert np.array_equal(out["time_delta"][s:e].cpu().numpy(),
                              want["time_delta"].astype(np.float32)), b
    torch.cuda.synchronize()


def test_host_sample_assemble_reports_the_first_bad_query(T):
    """tgfx_sample_assemble validates query nodes on the device inside its copy pipeline
    (4 M-query sub-chunks): the error must still name the first out-of-range query in query
    order (sampler.cpp:88-93), wherever it falls, and query 0 / k keep the reference's order."""
    ev = np.array([(1, 0, 2, 3.0), (2, 1, 2, 4.0), (0, 0, 1, 5.0)], dtype=T.EVENT_DTYPE)
    g = T.build_sequential(T.EventStream(ev, 3), False)
    q = 9_000_000
    nodes = np.zeros(q, np.int64)
    times = np.full(q, 4.5)
    nodes[8_500_000] = 7        # third sub-chunk
    nodes[4_200_000] = -3       # second sub-chunk: the first bad one
    nodes[8_999_999] = 11
    with pytest.raises(T.ValidationError, match="query node -3 out of range"):
        T.sample_assemble(g, nodes, times, 3, "recent", 0, 4, 4)
    nodes[4_200_000] = 0
    with pytest.raises(T.ValidationError, match="query node 7 out of range"):
        T.sample_assemble(g, nodes, times, 3, "random", 0, 4, 4)
    nodes[:] = 0
    out = T.sample_assemble(g, nodes[:1000], times[:1000], 3, "recent", 0, 4, 4)
    assert out["valid_len"].tolist() == [2] * 1000  # usable after a failure: 1 entry + self
    bad0 = np.array([5, 0], np.int64)  # query 0's node is checked before k (and before l)
    with pytest.raises(T.ValidationError, match="query node 5 out of range"):
        T.sample_assemble(g, bad0, [1.0, 1.0], 0, "recent", 0, 4, 4)
    with pytest.raises(T.ValidationError, match="k must be at least 1"):
        T.sample_assemble(g, [0, 9], [1.0, 1.0], 0, "recent", 0, 4, 4)
