"""CPU: pin the C restatement (oracle/oracle.c) against golden vectors produced by the reference
itself (tests/golden/gen_golden.py).  Bit-exact everywhere."""
import glob
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, events_of, golden


def test_streams_match_reference_generator(oracle_mod):
    g = golden("streams")
    for key, raw in g.items():
        e, v, seed, z = key.split("_")
        ev = oracle_mod.make_random_stream(int(e), int(v), int(seed), float(z))
        assert ev.view(np.uint8).tobytes() == raw.tobytes(), key


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "build_*.npz"))))
def test_build_matches_reference(oracle_mod, path):
    g = dict(np.load(path))
    ev = events_of(g["events"])
    for rev in (0, 1):
        got = oracle_mod.build(ev, int(g["num_nodes"]), bool(rev))
        for k in ("indptr", "nbr", "eid"):
            assert np.array_equal(got[k], g[f"rev{rev}_{k}"]), (path, rev, k)
        # bit-level equality of the float column (keeps -0.0 vs +0.0 payloads)
        assert got["ts"].view(np.uint64).tobytes() == g[f"rev{rev}_ts"].view(np.uint64).tobytes()
        assert oracle_mod.validate(got)


@pytest.mark.parametrize("name", ["sample_4000_150_31", "sample_3000_40_32"])
def test_sampler_and_assembler_match_reference(oracle_mod, name):
    g = golden(name)
    e, v, seed = (int(x) for x in name.split("_")[1:])
    ev = oracle_mod.make_random_stream(e, v, seed)
    graph = oracle_mod.build(ev, v, True)
    for strat in ("recent", "random"):
        for k in (1, 6, 20, 40):
            for tag, nn, tt in (("rand", g["qn"], g["qt"]), ("event", g["en"], g["et"])):
                c, nb, ed, ts = oracle_mod.sample_batch(graph, nn, tt, k, strat, 9)
                p = f"{strat}_k{k}_{tag}"
                assert np.array_equal(c, g[p + "_counts"]), p
                assert np.array_equal(nb, g[p + "_nbr"]), p
                assert np.array_equal(ed, g[p + "_eid"]), p
                assert np.array_equal(ts, g[p + "_ts"]), p
    for strat, k, l in (("recent", 10, 11), ("random", 20, 21), ("random", 10, 5),
                        ("recent", 40, 33)):
        sb = oracle_mod.sample_assemble(graph, g["en"], g["et"], k, strat, 9, l, e + 1)
        for kk in ("node_index", "edge_index", "time_delta", "valid_len"):
            assert np.array_equal(sb[kk], g[f"asm_{strat}_k{k}_l{l}_{kk}"]), (strat, k, l, kk)


def test_two_hop_composition_matches_reference(oracle_mod):
    g = golden("two_hop_6000_200_51")
    ev = oracle_mod.make_random_stream(6000, 200, 51)
    graph = oracle_mod.build(ev, 200, True)
    for strat in ("recent", "random"):
        h1, h2 = oracle_mod.two_hop(graph, g["roots"], g["rtimes"], 10, 10, strat, 9, 11, 6001,
                                    seed2=0x5eed2)
        for kk in ("node_index", "edge_index", "time_delta", "valid_len"):
            assert np.array_equal(h1[kk], g[f"{strat}_hop1_{kk}"]), (strat, kk)
            assert np.array_equal(h2[kk], g[f"{strat}_hop2_{kk}"]), (strat, kk)


def test_sequences_and_masks_match_reference(oracle_mod):
    g = golden("sequence")
    for l in (2, 4, 11, 33):
        sb = oracle_mod.build_sequence_batch(g["counts"], g["nbr"], g["eid"], g["ts"], g["qn"],
                                             g["qt"], l, 5001)
        for kk in ("node_index", "edge_index", "time_delta", "valid_len", "target_row"):
            assert np.array_equal(sb[kk], g[f"l{l}_{kk}"]), (l, kk)
        for kind in ("causal", "tgat", "self_loop"):
            m = oracle_mod.build_mask(sb["valid_len"], sb["target_row"], l, kind)
            assert np.array_equal(m, g[f"l{l}_mask_{kind}"]), (l, kind)


def test_error_texts(oracle_mod):
    with open(os.path.join(GOLDEN, "errors.json")) as f:
        errs = json.load(f)
    with pytest.raises(oracle_mod.OracleError, match=errs["bad_endpoint"]):
        oracle_mod.build(oracle_mod.events_from([0], [7], [1.0]), 2, False)
    g = oracle_mod.build(oracle_mod.events_from([0, 1, 0], [2, 2, 1], [3.0, 4.0, 5.0]), 3, False)
    with pytest.raises(oracle_mod.OracleError, match=errs["bad_node"]):
        oracle_mod.sample_batch(g, [99], [1.0], 3)
    with pytest.raises(oracle_mod.OracleError, match=errs["bad_k"]):
        oracle_mod.sample_batch(g, [0], [1.0], 0)


def test_reference_unit_known_answers(oracle_mod):
    """Inline constants of proj/tests/test_tcsr.cpp:50-97, test_sampler.cpp:32-87,
    test_sequence.cpp:19-31."""
    O = oracle_mod
    three = O.events_from([0, 1, 0], [2, 2, 1], [3.0, 4.0, 5.0], eid=[1, 2, 0])
    g = O.build(three, 3, False)
    assert g["indptr"].tolist() == [0, 2, 3, 3]
    assert g["ts"][:2].tolist() == [3.0, 5.0] and g["nbr"][:2].tolist() == [2, 1]
    g = O.build(three, 3, True)
    assert g["indptr"].tolist() == [0, 2, 4, 6]
    assert g["nbr"][4:6].tolist() == [0, 1] and g["ts"][4:6].tolist() == [3.0, 4.0]
    g = O.build(O.events_from([1], [1], [4.0]), 2, True)
    assert g["indptr"].tolist() == [0, 0, 2] and g["eid"].tolist() == [0, 0]
    assert O.build(O.events_from([], [], []), 4, True)["indptr"].tolist() == [0] * 5
    small = O.build(O.events_from([0, 1, 0], [2, 2, 1], [3.0, 4.0, 5.0], eid=[1, 2, 0]), 3, False)
    c, nb, ed, ts = O.sample_batch(small, [0, 0, 0, 0], [4.0, 3.0, 5.0, 99.0], 5)
    assert c.tolist() == [1, 0, 1, 2]
    assert ts[3, :2].tolist() == [3.0, 5.0]
    sb = O.build_sequence_batch(np.array([3]), np.array([[1, 2, 5]]), np.array([[0, 1, 2]]),
                                np.array([[2.0, 4.0, 7.0]]), [7], [10.0], 8, 100)
    assert sb["node_index"][0].tolist() == [2, 3, 6, 8, 0, 0, 0, 0]
    assert sb["edge_index"][0].tolist() == [1, 2, 3, 100, 0, 0, 0, 0]
    assert sb["time_delta"][0, :4].tolist() == [8.0, 6.0, 3.0, 0.0]


def test_assemble_inputs_restatement_vs_reference(oracle_mod):
    """oracle.assemble_inputs (numpy restatement of attention.cpp:414-451) against the
    reference's own assemble_inputs compiled from its sources (oracle/_ref)."""
    import os
    if not os.path.exists(oracle_mod.REF_SO):
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(11)
    q, l = 64, 11
    vl = rng.integers(1, l + 1, q)
    ni = rng.integers(0, 40, (q, l))
    ei = rng.integers(0, 90, (q, l))
    dt = rng.uniform(0, 1e6, (q, l))
    for concat, (dv, de, dtt) in ((False, (16, 16, 16)), (True, (8, 12, 20))):
        nt = rng.normal(size=(40, dv))
        et = rng.normal(size=(90, de))
        om, ph = rng.normal(size=dtt), rng.normal(size=dtt)
        a = oracle_mod.assemble_inputs(ni, ei, dt, vl, nt, et, om, ph, concat)
        b = oracle_mod.ref_assemble_inputs(ni, ei, dt, vl, nt, et, om, ph, concat)
        # one fma-rounded argument of size <= 1e6 away: 4 ulp(1e6)
        assert np.abs(a - b).max() <= 4 * np.spacing(1e6 * 5)
    bad = ni.copy()
    bad[0, 0] = 40
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.assemble_inputs(bad, ei, dt, vl, nt, et, om, ph, True)


def test_train_queries_restatement_vs_reference(oracle_mod):
    """make_batches + train_epoch's shard split + forward_concat layout (training.cpp:157-209,
    425-440): the restatement against the reference's own make_batches (oracle/_ref)."""
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built")
    ev = oracle_mod.make_random_stream(7_000, 400, 5)
    for npp, workers, B in ((1, 1, 200), (3, 1, 333), (2, 3, 250), (1, 8, 64)):
        seed = oracle_mod.mix_streams(17, 0x6e67, 4)
        got = oracle_mod.make_train_queries(ev, B, npp, workers, 400, seed)
        want = oracle_mod.ref_train_queries(ev, 400, B, npp, workers, seed)
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_mix_streams_device_library_matches_restatement(oracle_mod):
    from paper_2409_05477_b200 import device as D
    for a, b, c in ((0, 0x6e67, 0), (17, 3 * 0x10001 + 5, 2), (2**64 - 1, 2**63, 7)):
        assert D.mix_streams(a, b, c) == oracle_mod.mix_streams(a, b, c)
