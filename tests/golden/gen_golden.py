"""Generate golden vectors by running the REFERENCE itself (oracle/_ref/libtgf_ref.so, compiled
from /root/reference/proj/src by oracle/Makefile).  Run here (where /root/reference exists):

    make -C oracle && python tests/golden/gen_golden.py

Every array in tests/golden/*.npz is an output of the unmodified reference functions
(make_random_stream, build_sequential/build_parallel, sample_batch, sample_random,
build_sequence_batch, build_mask).  These fixtures pin both the C restatement in oracle/
(tests/test_oracle_golden.py, CPU) and the CUDA path (tests/test_gpu_*.py).
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402


def save(name, **arrs):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrs)


def graph_arrays(rg):
    g = rg.export()
    return dict(indptr=g["indptr"], nbr=g["nbr"], eid=g["eid"], ts=g["ts"],
                num_nodes=np.int64(g["num_nodes"]), num_edges=np.int64(g["num_edges"]),
                reverse=np.int64(g["reverse"]))


def build_case(name, events, num_nodes):
    """Reference build_sequential (and build_parallel(4) equality) for both reverse flags."""
    out = dict(events=events.view(np.uint8).reshape(-1, 32) if len(events) else
               np.zeros((0, 32), np.uint8), num_nodes=np.int64(num_nodes))
    rs = O.RefStream(events, num_nodes)
    for rev in (0, 1):
        rg, _ = rs.build(bool(rev), 0)
        rp, _ = rs.build(bool(rev), 4)
        a, b = rg.export(), rp.export()
        for k in ("indptr", "nbr", "eid", "ts"):
            assert np.array_equal(a[k], b[k]), (name, k)
        for k, v in graph_arrays(rg).items():
            out[f"rev{rev}_{k}"] = v
    save("build_" + name, **out)


def main():
    cases = {}
    # 1. synthetic generator (synthetic.cpp:12-43)
    streams = {}
    for (e, v, seed, z) in [(1000, 50, 1, 1.2), (5000, 300, 21, 1.2), (4000, 150, 31, 1.2),
                            (3000, 40, 32, 1.2), (2000, 25, 33, 1.2), (6000, 500, 5, 0.6),
                            (1, 1, 3, 1.2), (0, 5, 4, 1.2)]:
        ev = O.ref_make_random_stream(e, v, seed, z)
        streams[f"{e}_{v}_{seed}_{z}"] = ev.view(np.uint8).reshape(-1, 32) if e else \
            np.zeros((0, 32), np.uint8)
    save("streams", **streams)

    # 2. builds (tcsr.cpp:83-151) incl. the reference's unit-test shapes (test_tcsr.cpp)
    three = O.events_from([0, 1, 0], [2, 2, 1], [3.0, 4.0, 5.0], eid=[1, 2, 0])
    build_case("three_edge", three, 3)
    build_case("self_loop", O.events_from([1], [1], [4.0]), 2)
    build_case("empty", O.events_from([], [], []), 4)
    for seed in (11, 12, 13):
        build_case(f"rand20000_{seed}", O.ref_make_random_stream(20000, 700, seed), 700)
    # unsorted inputs (never exercised by the reference's own tests)
    rng = np.random.default_rng(7)
    ev = O.ref_make_random_stream(5000, 120, 41)
    build_case("shuffled", ev[rng.permutation(len(ev))].copy(), 120)
    ev2 = O.ref_make_random_stream(5000, 120, 42)
    ev2["edge_id"] = len(ev2) - 1 - ev2["edge_id"]  # eids descend inside equal-t runs
    build_case("eid_desc", ev2, 120)
    ev3 = O.ref_make_random_stream(3000, 60, 43)
    zero = ev3["timestamp"] == 0.0
    ev3["timestamp"][zero & (ev3["edge_id"] % 2 == 1)] = -0.0  # -0.0 keys compare equal
    build_case("neg_zero", ev3, 60)
    ev4 = O.events_from(rng.integers(0, 9, 4000), rng.integers(0, 9, 4000),
                        rng.uniform(0, 1e6, 4000))  # fractional, unsorted, dense hubs
    build_case("float_unsorted", ev4, 9)

    # 3. sampler (sampler.cpp:16-104) on reference graphs
    for (e, v, seed) in [(4000, 150, 31), (3000, 40, 32)]:
        ev = O.ref_make_random_stream(e, v, seed)
        rs = O.RefStream(ev, v)
        rg, _ = rs.build(True, 0)
        crng = np.random.default_rng(seed)
        qn = crng.integers(0, v, 1500).astype(np.int64)
        qt = crng.uniform(-5, e * 0.55, 1500)
        qt[:50] = ev["timestamp"][crng.integers(0, e, 50)]  # exact event times (strict <)
        ea, ta = O.make_queries(ev, 0, 600, 600, v)  # earliest and latest batches
        eb, tb = O.make_queries(ev, e - 600, e, 600, v)
        en, et = np.concatenate([ea, eb]), np.concatenate([ta, tb])
        out = dict(qn=qn, qt=qt, en=en, et=et)
        for strat in ("recent", "random"):
            for k in (1, 6, 20, 40):
                for tag, (nn, tt) in (("rand", (qn, qt)), ("event", (en, et))):
                    (c, nb, ed, ts), _ = O.ref_sample_batch(rg, nn, tt, k, strat, 9)
                    out[f"{strat}_k{k}_{tag}_counts"] = c
                    out[f"{strat}_k{k}_{tag}_nbr"] = nb
                    out[f"{strat}_k{k}_{tag}_eid"] = ed
                    out[f"{strat}_k{k}_{tag}_ts"] = ts
        # fused sample + assemble, as forward_concat (training.cpp:211-214)
        for strat, k, l in (("recent", 10, 11), ("random", 20, 21), ("random", 10, 5),
                            ("recent", 40, 33)):
            sb, _ = O.ref_sample_assemble(rg, en, et, k, strat, 9, l, e + 1)
            for kk, vv in sb.items():
                out[f"asm_{strat}_k{k}_l{l}_{kk}"] = vv
        save(f"sample_{e}_{v}_{seed}", **out)

    # 4. 2-hop composition from reference calls
    ev = O.ref_make_random_stream(6000, 200, 51)
    rs = O.RefStream(ev, 200)
    rg, _ = rs.build(True, 0)
    roots, rtimes = O.make_queries(ev, 0, 600, 600, 200)
    out = dict(roots=roots, rtimes=rtimes)
    for strat in ("recent", "random"):
        k1, k2, l = 10, 10, 11
        (c1, n1, e1, t1), _ = O.ref_sample_batch(rg, roots, rtimes, k1, strat, 9)
        h1 = O.ref_build_sequence_batch(c1, n1, e1, t1, roots, rtimes, l, 6001)
        q = len(roots)
        ni = np.zeros((q, k1, l), np.int64)
        ei = np.zeros((q, k1, l), np.int64)
        dt = np.zeros((q, k1, l), np.float64)
        vl = np.zeros((q, k1), np.int64)
        for i in range(q):
            for j in range(int(c1[i])):
                if strat == "recent":
                    (c2, a, b, cc), _ = O.ref_sample_batch(rg, n1[i, j:j + 1], t1[i, j:j + 1], k2,
                                                           "recent", 0)
                    cnt, a, b, cc = c2, a, b, cc
                else:
                    a0, b0, c0 = O.ref_sample_random(rg, int(n1[i, j]), float(t1[i, j]), k2,
                                                     0x5eed2, i * k1 + j)
                    cnt = np.array([len(a0)], np.int64)
                    a = np.zeros((1, k2), np.int64)
                    b = np.zeros((1, k2), np.int64)
                    cc = np.zeros((1, k2), np.float64)
                    a[0, :len(a0)], b[0, :len(a0)], cc[0, :len(a0)] = a0, b0, c0
                h2 = O.ref_build_sequence_batch(cnt, a, b, cc, n1[i, j:j + 1], t1[i, j:j + 1], l,
                                                6001)
                ni[i, j], ei[i, j] = h2["node_index"][0], h2["edge_index"][0]
                dt[i, j], vl[i, j] = h2["time_delta"][0], h2["valid_len"][0]
        for kk, vv in h1.items():
            out[f"{strat}_hop1_{kk}"] = vv
        out[f"{strat}_hop2_node_index"], out[f"{strat}_hop2_edge_index"] = ni, ei
        out[f"{strat}_hop2_time_delta"], out[f"{strat}_hop2_valid_len"] = dt, vl
    save("two_hop_6000_200_51", **out)

    # 5. sequences + masks (sequence.cpp:55-111), incl. test_sequence.cpp's shapes
    crng = np.random.default_rng(3)
    q, kp = 500, 24
    counts = crng.integers(0, kp + 1, q).astype(np.int64)
    nbr = crng.integers(0, 1000, (q, kp)).astype(np.int64)
    eid = crng.integers(0, 5000, (q, kp)).astype(np.int64)
    ts = np.sort(crng.uniform(0, 100, (q, kp)), axis=1)
    qn = crng.integers(0, 1000, q).astype(np.int64)
    qt = np.full(q, 150.0)
    out = dict(counts=counts, nbr=nbr, eid=eid, ts=ts, qn=qn, qt=qt)
    for l in (2, 4, 11, 33):
        sb = O.ref_build_sequence_batch(counts, nbr, eid, ts, qn, qt, l, 5001)
        for kk, vv in sb.items():
            out[f"l{l}_{kk}"] = vv
        for kind in ("causal", "tgat", "self_loop"):
            out[f"l{l}_mask_{kind}"] = O.ref_build_mask(sb["valid_len"], sb["target_row"], l, kind)
    save("sequence", **out)

    # 6. error texts (common.hpp ValidationError messages)
    errs = {}
    bad = O.events_from([0], [7], [1.0])
    try:
        O.RefStream(bad, 2).build(False, 0)
    except O.OracleError as ex:
        errs["bad_endpoint"] = str(ex)
    try:
        O.RefStream(three, 3).build_parallel_raw(True, 0)
    except O.OracleError as ex:
        errs["bad_threads"] = str(ex)
    rg, _ = O.RefStream(three, 3).build(False, 0)
    for key, args in (("bad_node", ([99], [1.0], 3)), ("bad_k", ([0], [1.0], 0))):
        try:
            O.ref_sample_batch(rg, np.array(args[0]), np.array(args[1]), args[2])
        except O.OracleError as ex:
            errs[key] = str(ex)
    try:
        O.ref_build_sequence_batch(np.zeros(1, np.int64), np.zeros((1, 1), np.int64),
                                   np.zeros((1, 1), np.int64), np.zeros((1, 1)),
                                   np.zeros(1, np.int64), np.zeros(1), 1, 11)
    except O.OracleError as ex:
        errs["bad_l"] = str(ex)
    with open(os.path.join(HERE, "errors.json"), "w") as f:
        json.dump(errs, f, indent=1, sort_keys=True)
    print("golden vectors written:", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
