"""Property-based parity (hypothesis): random small streams -- tied and out-of-order
timestamps, self-loops, hub-heavy or uniform endpoints, both reverse settings -- built and
sampled on the device, compared element by element with the oracle (bit-exact indices and
fp64 deltas)."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

pytestmark = pytest.mark.gpu


@st.composite
def streams(draw):
    V = draw(st.integers(1, 400))
    n = draw(st.integers(0, 3000))
    seed = draw(st.integers(0, 2**31 - 1))
    rng = np.random.default_rng(seed)
    skew = draw(st.sampled_from(["uniform", "hub", "two"]))
    if skew == "uniform":
        src, dst = rng.integers(0, V, n), rng.integers(0, V, n)
    elif skew == "hub":
        p = 1.0 / np.arange(1, V + 1) ** 1.2
        p /= p.sum()
        src, dst = rng.choice(V, n, p=p), rng.choice(V, n, p=p)
    else:
        src, dst = rng.integers(0, min(V, 2), n), rng.integers(0, V, n)
    tmax = draw(st.sampled_from([1, 5, 50, 10_000]))
    t = np.sort(rng.integers(0, tmax, n)).astype(np.float64)
    eid = np.arange(n)
    order = draw(st.sampled_from(["sorted", "shuffled", "eid_desc_in_ties"]))
    if order == "shuffled":
        perm = rng.permutation(n)
        src, dst, t, eid = src[perm], dst[perm], t[perm], eid[perm]
    elif order == "eid_desc_in_ties":
        eid = np.lexsort((-np.arange(n), t))  # eids decrease inside equal-time runs
    ev = np.zeros(n, dtype=[("edge_id", "<i8"), ("src", "<i8"), ("dst", "<i8"),
                            ("timestamp", "<f8")])
    ev["edge_id"], ev["src"], ev["dst"], ev["timestamp"] = eid, src, dst, t
    return ev, V, seed, tmax


@settings(max_examples=80, deadline=None, suppress_health_check=list(HealthCheck))
@given(streams(), st.booleans(), st.integers(1, 40), st.sampled_from(["recent", "random"]))
def test_random_streams_build_and_sample(oracle_mod, s, reverse, k, strategy):
    from paper_2409_05477_b200 import tgformer as T
    ev, V, seed, tmax = s
    want = oracle_mod.build(ev, V, reverse)
    g = T.build_parallel(T.EventStream(ev, V), reverse, 8)
    assert np.array_equal(g.indptr, want["indptr"])
    assert np.array_equal(g.neighbor_ids, want["nbr"])
    assert np.array_equal(g.edge_ids, want["eid"])
    assert np.array_equal(g.timestamps, want["ts"])
    rng = np.random.default_rng(seed + 1)
    q = 500
    nodes = rng.integers(0, V, q)
    times = np.concatenate([rng.integers(0, tmax + 1, q - 20).astype(np.float64),
                            [np.nan, -1.0, 0.0, -0.0, np.inf, -np.inf] + [tmax / 2] * 14])
    l = max(2, min(k + 1, 41))
    got = T.sample_assemble(g, nodes, times, k, strategy, seed, l, len(ev) + 1, dt64=True)
    ref = oracle_mod.sample_assemble(want, nodes, times, k, strategy, seed, l, len(ev) + 1)
    assert np.array_equal(got["node_index"].astype(np.int64), ref["node_index"])
    assert np.array_equal(got["edge_index"].astype(np.int64), ref["edge_index"])
    assert np.array_equal(got["valid_len"].astype(np.int64), ref["valid_len"])
    assert np.array_equal(got["time_delta64"], ref["time_delta"])
