"""GPU parity: build_sequence_batch / build_mask kernels (C ABI tgfx_assemble / tgfx_build_mask)
and the device stream/query generators vs the reference's golden vectors."""
import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    from paper_2409_05477_b200 import tgformer
    return tgformer


def test_sequences_and_masks_match_reference_golden(T):
    g = golden("sequence")
    for l in (2, 4, 11, 33):
        sb = T.assemble_arrays(g["counts"], g["nbr"], g["eid"], g["ts"], g["qn"], g["qt"], l, 5001)
        for kk in ("node_index", "edge_index", "valid_len", "target_row"):
            assert np.array_equal(getattr(sb, kk), g[f"l{l}_{kk}"]), (l, kk)
        assert sb.time_delta.tobytes() == g[f"l{l}_time_delta"].tobytes()
        for kind in ("causal", "tgat", "self_loop"):
            assert np.array_equal(T.build_mask(sb, kind), g[f"l{l}_mask_{kind}"]), (l, kind)


def test_reference_sequence_known_answers(T):
    """proj/tests/test_sequence.cpp:19-88"""
    E = T.NeighborEntry
    s = T.NeighborSample(7, 10.0, [E(1, 0, 2.0), E(2, 1, 4.0), E(5, 2, 7.0)])
    b = T.build_sequence(s, 8, 100)
    assert b.node_index[0].tolist() == [2, 3, 6, 8, 0, 0, 0, 0]
    assert b.edge_index[0].tolist() == [1, 2, 3, 100, 0, 0, 0, 0]
    assert b.valid_len[0] == 4 and b.target_row[0] == 3
    assert b.time_delta[0, :4].tolist() == [8.0, 6.0, 3.0, 0.0]
    b = T.build_sequence(T.NeighborSample(7, 3.0, []), 4, 9)
    assert b.node_index[0].tolist() == [8, 0, 0, 0] and b.edge_index[0].tolist() == [9, 0, 0, 0]
    ents = [E(i, i, float(i)) for i in range(10)]
    b = T.build_sequence(T.NeighborSample(0, 20.0, ents), 5, 50)
    assert b.valid_len[0] == 5 and b.node_index[0].tolist() == [7, 8, 9, 10, 1]
    assert b.time_delta[0, :4].tolist() == [14.0, 13.0, 12.0, 11.0]
    with pytest.raises(T.ValidationError, match="sequence length must be at least 2"):
        T.build_sequence(T.NeighborSample(3, 9.0, [E(1, 4, 2.5)]), 1, 11)
    m = T.build_mask(T.build_sequence(T.NeighborSample(1, 10.0, [E(2, 0, 1.0), E(3, 1, 2.0)]), 3, 5),
                     "causal")
    assert np.array_equal(m == 0.0, np.tril(np.ones((3, 3), bool)))
    with pytest.raises(T.ValidationError):
        T.parse_mask_kind("full")


def test_device_generator_matches_reference_streams(T):
    g = golden("streams")
    for key, raw in g.items():
        e, v, seed, z = key.split("_")
        st = T.make_random_stream(int(e), int(v), int(seed), float(z))
        assert st.events.view(np.uint8).tobytes() == raw.tobytes(), key


def test_device_generator_large_prefix(oracle_mod):
    """GDELT-shaped generator: the first 3M events of make_random_stream(3M) bit-identical."""
    from paper_2409_05477_b200 import device as D
    want = oracle_mod.make_random_stream(3_000_000, 16682, 42)
    got = D.random_stream(3_000_000, 16682, 42).cpu().numpy()
    assert got.tobytes() == want.view(np.uint8).tobytes()


def test_record_layout_calls_match_column_calls(T):
    """tgfx_sample_batch_records / tgfx_assemble_records (the C++ layer's forward_concat route,
    tgfx_neighbor records = NeighborEntry) equal the column calls, from pinned and pageable
    host buffers, on the reference golden sequences and on a sampled batch."""
    import ctypes as C

    from paper_2409_05477_b200._lib import check, lib
    L = lib()
    rec_t = np.dtype([("neighbor", np.int64), ("edge", np.int64), ("timestamp", np.float64)])
    g = golden("sequence")
    q, kp = g["nbr"].shape
    rec = np.zeros((q, kp), rec_t)
    rec["neighbor"], rec["edge"], rec["timestamp"] = g["nbr"], g["eid"], g["ts"]
    for l in (2, 4, 11, 33):
        outs = [np.zeros(q * l, np.int64), np.zeros(q * l, np.int64), np.zeros(q * l, np.float64),
                np.zeros(q, np.int64), np.zeros(q, np.int64)]
        args = [np.ascontiguousarray(x) for x in (g["counts"], rec, g["qn"], g["qt"])]
        check(L.tgfx_assemble_records(q, kp, *(a.ctypes.data for a in args), l, 5001,
                                      *(o.ctypes.data for o in outs)))
        for o, kk in zip(outs, ("node_index", "edge_index", "time_delta", "valid_len",
                                "target_row")):
            assert o.tobytes() == np.ascontiguousarray(g[f"l{l}_{kk}"]).tobytes(), (l, kk)

    ev = T.make_random_stream(30_000, 250, 3)
    gr = T.build_parallel(ev, True, 4)
    rng = np.random.default_rng(1)
    nq = 5000
    nodes = rng.integers(0, 250, nq).astype(np.int64)
    times = rng.uniform(0, 30_000, nq)
    # the same call from page-locked buffers
    p = C.c_void_p()
    check(L.tgfx_host_alloc(16 * nq, C.byref(p)))
    try:
        pin = np.ctypeslib.as_array((C.c_char * (16 * nq)).from_address(p.value))
        pn = pin[:8 * nq].view(np.int64)
        pt = pin[8 * nq:].view(np.float64)
        pn[:], pt[:] = nodes, times
        for strat, code, k in (("recent", 0, 10), ("random", 1, 20), ("random", 1, 300)):
            counts, nb, ed, ts = T.sample_batch_arrays(gr, nodes, times, k, strat, 9)
            for src_n, src_t in ((nodes, times), (pn, pt)):
                c2 = np.zeros(nq, np.int64)
                r2 = np.zeros((nq, k), rec_t)
                check(L.tgfx_sample_batch_records(gr.handle, src_n.ctypes.data, src_t.ctypes.data,
                                                  nq, k, code, 9, 0, c2.ctypes.data,
                                                  r2.ctypes.data))
                assert np.array_equal(c2, counts), strat
                assert np.array_equal(r2["neighbor"], nb), strat
                assert np.array_equal(r2["edge"], ed), strat
                assert r2["timestamp"].tobytes() == ts.tobytes(), strat
        bad = nodes.copy()
        bad[77] = 250
        with pytest.raises(T.ValidationError, match="query node 250 out of range"):
            check(L.tgfx_sample_batch_records(gr.handle, bad.ctypes.data, times.ctypes.data, nq, 5,
                                              0, 0, 0, np.zeros(nq, np.int64).ctypes.data,
                                              np.zeros((nq, 5), rec_t).ctypes.data))
    finally:
        check(L.tgfx_host_free(p))
