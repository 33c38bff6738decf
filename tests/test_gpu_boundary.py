"""The drop-in boundary where it used to differ from the reference:

* TCsr::validate (tcsr.cpp:54-81): message text and precedence on corrupted graphs, checked
  against the reference's own validate (oracle/_ref) on the very same columns;
* uniform sampling with k > 256 (the reference has no limit, sampler.cpp:54-82), entries and
  assembled rows, against the oracle;
* batched uniform launches whose Q is a multiple of the batch size but not of 32 (the tail
  lanes of the last warp must not read past the per-batch seed array)."""
import numpy as np
import pytest

from test_gpu_sample import check_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    from paper_2409_05477_b200 import tgformer
    return tgformer


def _device_validate(T, V, E, rev, ip, nb, ed, ts):
    g = T.TCsr.from_host(V, E, rev, ip, nb, ed, ts)
    try:
        g.validate()
        return ""
    except T.ValidationError as e:
        return str(e)


def _corruptions(og, rng):
    ip, nb, ed, ts = (og[k].copy() for k in ("indptr", "nbr", "eid", "ts"))
    V, E = og["num_nodes"], og["num_edges"]
    big = [u for u in range(V) if ip[u + 1] - ip[u] > 8]
    u1, u2 = big[3], big[9]

    cases = {}
    t = ts.copy()
    t[ip[u2] + 1] = t[ip[u2] + 2] + 5.0
    cases["unsorted_u2"] = (ip, nb, ed, t)
    t2 = t.copy()
    t2[ip[u1] + 1] = t2[ip[u1] + 2] + 5.0
    n2 = nb.copy()
    n2[0] = V
    cases["two_unsorted_and_bad_nbr"] = (ip, n2, ed, t2)
    n3, e3 = nb.copy(), ed.copy()
    n3[100] = -1
    e3[50] = E
    cases["eid_first"] = (ip, n3, e3, ts)
    n4, e4 = nb.copy(), ed.copy()
    n4[70], e4[70] = V + 5, -3
    cases["same_entry_nbr_first"] = (ip, n4, e4, ts)
    # equal timestamps with decreasing edge ids (entry_less ties)
    e5, t5 = ed.copy(), ts.copy()
    i = ip[u1] + 3
    t5[i] = t5[i + 1]
    e5[i], e5[i + 1] = max(e5[i], e5[i + 1]) , min(e5[i], e5[i + 1])
    if e5[i] == e5[i + 1]:
        e5[i + 1] -= 1
    cases["tie_eid_desc"] = (ip, nb, e5, t5)
    # NaN timestamps compare false: not flagged by the reference
    t6 = ts.copy()
    t6[ip[u1] + 1] = np.nan
    cases["nan_inside"] = (ip, nb, ed, t6)
    # indptr not monotone at a node after an unsorted slice, and before one
    ip7 = ip.copy()
    k = (u1 + u2) // 2
    ip7[k + 1] = ip7[k] - 1 if ip7[k] > 0 else 0
    if ip7[k] > ip7[k + 1]:
        t7 = ts.copy()
        t7[ip[u1] + 1] = t7[ip[u1] + 2] + 5.0      # u1 < k: slice error first
        cases["mono_after_unsorted"] = (ip7, nb, ed, t7)
        t8 = ts.copy()
        t8[ip[u2] + 1] = t8[ip[u2] + 2] + 5.0      # u2 > k: monotone error first
        cases["mono_before_unsorted"] = (ip7, nb, ed, t8)
    ip9 = ip.copy()
    ip9[-1] -= 1
    cases["endpoints"] = (ip9, nb, ed, ts)
    cases["clean"] = (ip, nb, ed, ts)
    return cases


def test_validate_text_and_precedence_match_reference(T, oracle_mod):
    rng = np.random.default_rng(5)
    for E, V, rev in ((40_000, 300, True), (30_000, 90, False)):
        ev = oracle_mod.make_random_stream(E, V, 11)
        og = oracle_mod.build(ev, V, rev)
        for name, (ip, nb, ed, ts) in _corruptions(og, rng).items():
            want = oracle_mod.ref_validate_columns(V, E, rev, ip, nb, ed, ts)
            got = _device_validate(T, V, E, rev, ip, nb, ed, ts)
            assert got == want, (name, got, want)
            if name == "clean":
                assert want == ""
            elif name != "nan_inside":
                assert want != "", name


def test_corrupt_indptr_is_refused_by_the_sampler(T, oracle_mod):
    ev = oracle_mod.make_random_stream(5000, 50, 3)
    og = oracle_mod.build(ev, 50, True)
    ip = og["indptr"].copy()
    ip[10] = 10**12   # inside a CRC-valid container this would index far outside ts
    g = T.TCsr.from_host(50, 5000, True, ip, og["nbr"], og["eid"], og["ts"])
    # the reference's walk of node 9's oversized slice meets node 10's entries first
    want = oracle_mod.ref_validate_columns(50, 5000, True, ip, og["nbr"], og["eid"], og["ts"])
    assert want
    with pytest.raises(T.ValidationError) as ei:
        g.validate()
    assert str(ei.value) == want
    with pytest.raises(T.ValidationError, match="indptr not monotone"):
        T.sample_batch_arrays(g, np.array([1]), np.array([5.0]), 5, "recent", 0)


@pytest.mark.parametrize("k", [257, 300, 1000, 4096])
def test_uniform_k_above_256(T, oracle_mod, k):
    E, V = 400_000, 60
    ev = oracle_mod.make_random_stream(E, V, 21)
    og = oracle_mod.build(ev, V, True)
    g = T.build_sequential(T.EventStream(ev, V), True)
    rng = np.random.default_rng(k)
    idx = rng.integers(0, E, 700)
    nodes = np.concatenate([ev["src"][idx], ev["dst"][idx[:300]]])
    times = np.concatenate([ev["timestamp"][idx], ev["timestamp"][idx[:300]]])
    c, nb, ed, ts = T.sample_batch_arrays(g, nodes, times, k, "random", 9, stream_base=5)
    wc, wn, we, wt = oracle_mod.sample_batch(og, nodes, times, k, "random", 9, stream_base=5)
    assert np.array_equal(c, wc)
    for q in range(len(nodes)):
        n = int(wc[q])
        assert np.array_equal(nb[q, :n], wn[q, :n]), q
        assert np.array_equal(ed[q, :n], we[q, :n]), q
        assert np.array_equal(ts[q, :n], wt[q, :n]), q
    for l in (11, 300):
        got = T.sample_assemble(g, nodes, times, k, "random", 9, l, E + 1, dt64=True)
        want = oracle_mod.sample_assemble(og, nodes, times, k, "random", 9, l, E + 1)
        check_rows(got, want, (k, l))


def test_batched_uniform_tail_lanes(T, oracle_mod):
    """Q % batch_q == 0 and Q % 32 != 0: the last warp's dead lanes must clamp their batch
    index (they used to read seeds[Q / batch_q], one past the array)."""
    import torch
    from paper_2409_05477_b200 import device as D
    E, V, bq = 50_000, 500, 600
    ev = D.random_stream(E, V, 4)
    g = D.build(ev, V, True)
    nodes, times = D.make_queries(ev, 0, 1000, 200, V)   # 3000 queries = 5 batches of 600
    q = nodes.numel()
    assert q % bq == 0 and q % 32 != 0
    seeds = torch.tensor([9 + b for b in range(q // bq)], dtype=torch.int64, device="cuda")
    for k, l in ((20, 21), (10, 11), (40, 11)):
        out = D.sample_assemble_batched(g, nodes, times, bq, k, "random", seeds, l, E + 1)
        og = oracle_mod.build(ev.cpu().numpy().view(oracle_mod.EVENT_DTYPE), V, True)
        hn, ht = nodes.cpu().numpy(), times.cpu().numpy()
        for b in range(q // bq):
            sl = slice(b * bq, (b + 1) * bq)
            want = oracle_mod.sample_assemble(og, hn[sl], ht[sl], k, "random", 9 + b, l, E + 1)
            got = {kk: v[sl].cpu().numpy() for kk, v in out.items()}
            check_rows(got, want, (k, l, b))


def test_fused_query_check():
    """check_query (sampler.cpp:22-27) fused into the sampler kernel: rows equal the
    validating path's, the first failing query over several calls sharing one word is
    reported with the reference's text, failing rows come out absent, and a trusted call with
    a bad node neither faults nor writes a bogus row."""
    import torch
    from paper_2409_05477_b200 import device as D
    from paper_2409_05477_b200._lib import ValidationError
    E, V = 60_000, 500
    ev = D.random_stream(E, V, 5)
    g = D.build(ev, V, True)
    nodes, times = D.make_queries(ev, 0, 6000, 600, V)
    for strat, k, l in (("recent", 10, 11), ("random", 20, 21)):
        want = D.sample_assemble(g, nodes, times, k, strat, 9, l, E + 1)
        w = D.first_bad_word()
        got = D.sample_assemble(g, nodes, times, k, strat, 9, l, E + 1, first_bad=w)
        D.query_error(nodes, w)  # no failure
        for key in want:
            assert torch.equal(want[key], got[key]), (strat, key)
    # two calls (stream_base 0 and 9000) sharing a word; failures at global 9000+17 and 9000+40
    bad = nodes.clone()
    bad[17] = V
    bad[40] = -2
    w = D.first_bad_word()
    D.sample_assemble(g, nodes[:9000], times[:9000], 10, "recent", 9, 11, E + 1, first_bad=w)
    rows = D.sample_assemble(g, bad[:9000], times[:9000], 10, "recent", 9, 11, E + 1,
                             stream_base=9000, first_bad=w)
    with pytest.raises(ValidationError, match=f"query node {V} out of range"):
        D.query_error(bad[:9000], w, stream_base=9000)
    assert int(rows["valid_len"][17]) == 0 and int(rows["valid_len"][40]) == 0
    assert int(rows["node_index"][17].abs().sum()) == 0
    ref = D.sample_assemble(g, nodes[:9000], times[:9000], 10, "recent", 9, 11, E + 1)
    keep = torch.ones(9000, dtype=torch.bool, device="cuda")
    keep[[17, 40]] = False
    assert torch.equal(rows["node_index"][keep], ref["node_index"][keep])
    # the validating path raises the same error, and trusted sampling of a bad node is absent
    with pytest.raises(ValidationError, match=f"query node {V} out of range"):
        D.sample_assemble(g, bad[:9000], times[:9000], 10, "recent", 9, 11, E + 1)
    tr = D.sample_assemble(g, bad[:9000], times[:9000], 10, "recent", 9, 11, E + 1, trusted=True)
    torch.cuda.synchronize()
    assert int(tr["valid_len"][40]) == 0


def test_host_buffer_sample_assemble_sub_chunks(T):
    """tgfx_sample_assemble with host buffers over several sub-chunks (a short head sub-chunk,
    then full ones, alternating between two lanes): rows equal the device-buffer call on the
    same queries (uniform-k included, so every sub-chunk's RNG stream offset is checked), and a
    bad node in a late sub-chunk raises the reference's error with the caller's buffers left
    untouched (sampler.cpp:88-93 validates every query before anything is returned)."""
    import torch
    from paper_2409_05477_b200 import device as D
    E, V = 400_000, 3000
    ev = D.random_stream(E, V, 21)
    g = D.build(ev, V, True)
    nodes, times = D.make_queries(ev, 0, E, 600, V)  # 1.2 M queries: head + 1 full sub-chunk
    hn, ht = nodes.cpu().numpy(), times.cpu().numpy()
    th = g
    for strat, k, l in (("recent", 10, 11), ("random", 20, 21)):
        want = D.sample_assemble(g, nodes, times, k, strat, 9, l, E + 1, stream_base=77)
        got = T.sample_assemble(th, hn, ht, k, strat, 9, l, E + 1, stream_base=77)
        for key in ("node_index", "edge_index", "time_delta", "valid_len"):
            assert np.array_equal(got[key], want[key].cpu().numpy()), (strat, key)
    from paper_2409_05477_b200._lib import ValidationError, check, lib
    bad = hn.copy()
    bad[1_000_003] = V + 5
    q, l = len(bad), 11
    outs = [np.full(q * l, 7, np.int32), np.full(q * l, 7, np.int32),
            np.full(q * l, 7.0, np.float32), np.full(q, 7, np.int32)]
    with pytest.raises(ValidationError, match=f"query node {V + 5} out of range"):
        check(lib().tgfx_sample_assemble(th.handle, bad.ctypes.data, ht.ctypes.data, q, 10, 0, 9,
                                         0, l, E + 1, outs[0].ctypes.data, outs[1].ctypes.data,
                                         outs[2].ctypes.data, None, outs[3].ctypes.data))
    assert all((o == 7).all() for o in outs)
