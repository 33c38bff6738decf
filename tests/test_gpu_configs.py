"""GPU parity on the five north-star configurations at (or, for MAG, 1/16 of) their full shapes.

  G  GDELT-shaped, 191,290,882 events: the whole device T-CSR equal, element by element, to
     the oracle's build_sequential (tcsr.cpp:83-105) of the oracle's own stream; the device
     stream itself equal to the oracle's make_random_stream (synthetic.cpp:12-43); sampling
     checked against the ORACLE's graph (not the device export), so a build bug at full size
     cannot hide behind the sampler test.
  R  Reddit-shaped, 672,447 events / 10,984 nodes: 2-hop recent 10x10 over every
     forward_concat batch (1,121 batches of 600 events, roots [src, dst, neg]), hop-1 and hop-2
     rows against the oracle's composition of sample_batch + build_sequence_batch
     (sampler.cpp:84-104, sequence.cpp:55-86).
  M  MAG-shaped at 1/16 scale (7,562,500 nodes, 81,250,000 events, Zipf 1.2): the single-GPU
     large-V build and a 2-rank node-range-partitioned build (two processes on this GPU, gloo
     host-staged exchange) both equal to the oracle; recent-10 rows on a stream-spread sample.
  W, L are in test_gpu_sample.py (full streams).

Index outputs are compared bit for bit; fp32 time deltas must equal the fp64 reference rounded
to nearest (relative error <= 2^-24, inside north_star's 1e-6)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from test_gpu_sample import check_rows

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CHUNK = 1 << 26


def _eq_chunks(dev, host, tag):
    """dev: 1-D cuda tensor; host: numpy array of the same length / dtype: chunked equality
    on the device (bitwise for floats, via an int64 view)."""
    assert dev.numel() == len(host), (tag, dev.numel(), len(host))
    if dev.dtype == torch.float64:
        dev = dev.view(torch.int64)
        host = host.view(np.int64)
    for a in range(0, len(host), CHUNK):
        b = min(len(host), a + CHUNK)
        h = torch.from_numpy(np.ascontiguousarray(host[a:b])).to(dev.device)
        if not torch.equal(dev[a:b], h):
            bad = int(torch.nonzero(dev[a:b] != h)[0, 0]) + a
            raise AssertionError(f"{tag}: first mismatch at {bad}")


def _spread_batches(E, B, nb):
    """nb batch indices spread over the stream, first and last included."""
    last = (E - 1) // B
    return sorted(set(np.linspace(0, last, nb).astype(np.int64).tolist()))


def test_gdelt_full_build_bit_exact_vs_oracle(oracle_mod):
    from paper_2409_05477_b200 import device as D
    E, V = 191_290_882, 16682
    host_ev = oracle_mod.make_random_stream(E, V, 42)
    ev = D.random_stream(E, V, 42)
    _eq_chunks(D.event_view(ev).reshape(-1), host_ev.view(np.int64).reshape(-1), "stream")
    want = oracle_mod.build(host_ev, V, True)
    g = D.build(ev, V, True)
    ip, nb, ed, ts = D.graph_tensors(g)
    _eq_chunks(ip, want["indptr"], "indptr")
    _eq_chunks(nb, want["nbr"], "nbr")
    _eq_chunks(ed, want["eid"], "eid")
    _eq_chunks(ts, want["ts"], "ts")
    g.validate()
    # sampling at full size against the oracle's own graph: 40 forward_concat batches spread
    # over the stream (recent-10) and 12 of them uniform-20, global stream index per query
    B = 600
    for i, b in enumerate(_spread_batches(E, B, 40)):
        e0, e1 = b * B, min(E, (b + 1) * B)
        nodes, times = D.make_queries(ev, e0, e1, B, V)
        hn, ht = oracle_mod.make_queries(host_ev, e0, e1, B, V)
        assert np.array_equal(nodes.cpu().numpy(), hn) and np.array_equal(times.cpu().numpy(), ht)
        out = D.sample_assemble(g, nodes, times, 10, "recent", 9 + b, 11, E + 1, dt64=True)
        got = {k: v.cpu().numpy() for k, v in out.items()}
        check_rows(got, oracle_mod.sample_assemble(want, hn, ht, 10, "recent", 9 + b, 11, E + 1),
                   ("recent", b))
        if i % 3 == 0:
            out = D.sample_assemble(g, nodes, times, 20, "random", 9 + b, 21, E + 1, dt64=True)
            got = {k: v.cpu().numpy() for k, v in out.items()}
            check_rows(got, oracle_mod.sample_assemble(want, hn, ht, 20, "random", 9 + b, 21,
                                                       E + 1), ("random", b))
    del want, host_ev, ip, nb, ed, ts
    torch.cuda.synchronize()


def test_reddit_two_hop_full_shape(oracle_mod):
    from paper_2409_05477_b200 import device as D
    E, V, B, k1, k2, l = 672_447, 10_984, 600, 10, 10, 11
    ev = D.random_stream(E, V, 42)
    host_ev = oracle_mod.make_random_stream(E, V, 42)
    assert np.array_equal(D.event_view(ev).cpu().numpy().reshape(-1),
                          host_ev.view(np.int64).reshape(-1))
    og = oracle_mod.build(host_ev, V, True)
    g = D.build(ev, V, True)
    roots, rtimes = D.make_queries(ev, 0, E, B, V)     # all 1,121 batches: 2,017,341 roots
    hn, ht = oracle_mod.make_queries(host_ev, 0, E, B, V)
    assert np.array_equal(roots.cpu().numpy(), hn) and np.array_equal(rtimes.cpu().numpy(), ht)
    out = D.two_hop(g, roots, rtimes, k1, k2, "recent", 0, l, E + 1)
    h1, h2 = oracle_mod.two_hop(og, hn, ht, k1, k2, "recent", 0, l, E + 1)
    q = len(hn)
    got1 = {k: v.cpu().numpy() for k, v in out["h1"].items()}
    check_rows(got1, h1, "hop1")
    got2 = {k: v.cpu().numpy().reshape((q, k1) + v.shape[1:]) for k, v in out["h2"].items()}
    for key in ("node_index", "edge_index", "valid_len"):
        assert np.array_equal(got2[key].astype(np.int64), h2[key]), key
    ref = h2["time_delta"]
    assert np.array_equal(got2["time_delta"], ref.astype(np.float32))
    n_hop2 = int((h2["valid_len"] > 0).sum())
    assert n_hop2 > 15_000_000, n_hop2   # ~16.4 M hop-2 rows at this shape
    torch.cuda.synchronize()


MAG16 = (81_250_000, 7_562_500)


def test_mag_sixteenth_large_v_build_and_sampling(oracle_mod):
    from paper_2409_05477_b200 import device as D
    E, V = MAG16
    ev = D.random_stream(E, V, 42)
    host_ev = oracle_mod.make_random_stream(E, V, 42)
    _eq_chunks(D.event_view(ev).reshape(-1), host_ev.view(np.int64).reshape(-1), "stream")
    want = oracle_mod.build(host_ev, V, True)
    g = D.build(ev, V, True)
    assert g.build_path == 2  # large-V path
    ip, nb, ed, ts = D.graph_tensors(g)
    _eq_chunks(ip, want["indptr"], "indptr")
    _eq_chunks(nb, want["nbr"], "nbr")
    _eq_chunks(ed, want["eid"], "eid")
    _eq_chunks(ts, want["ts"], "ts")
    g.validate()
    B = 600
    for b in _spread_batches(E, B, 30):
        e0, e1 = b * B, min(E, (b + 1) * B)
        nodes, times = D.make_queries(ev, e0, e1, B, V)
        hn, ht = nodes.cpu().numpy(), times.cpu().numpy()
        out = D.sample_assemble(g, nodes, times, 10, "recent", 9 + b, 11, E + 1, dt64=True)
        got = {k: v.cpu().numpy() for k, v in out.items()}
        check_rows(got, oracle_mod.sample_assemble(want, hn, ht, 10, "recent", 9 + b, 11, E + 1),
                   ("mag recent", b))
    torch.cuda.synchronize()


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _mag_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2409_05477_b200 import device as D, partition as P
        E, V = MAG16
        ev = D.random_stream(E, V, 42)
        per = -(-E // world)
        chunk = ev[rank * per * 32:min(E, (rank + 1) * per) * 32].clone()
        del ev
        res = P.build_partitioned(chunk, V, True, E, replicate=True, exchange_on_host=True)
        ip, nb, ed, ts = D.graph_tensors(res["local"])
        fip, fnb, fed, fts = D.graph_tensors(res["full"])
        np.savez(os.path.join(out_dir, f"mag_r{rank}.npz"), bounds=res["bounds"].cpu().numpy(),
                 P=res["positions"].cpu().numpy(), rng=np.array(res["range"]),
                 nrecv=res["received_records"], ip=ip.cpu().numpy(), nb=nb.cpu().numpy(), ed=ed.cpu().numpy(),
                 ts=ts.cpu().numpy(), fip=fip.cpu().numpy(), fnb=fnb.cpu().numpy(),
                 fed=fed.cpu().numpy(), fts=fts.cpu().numpy())
        del res
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()


def test_mag_sixteenth_partitioned_two_ranks(tmp_path, oracle_mod):
    from paper_2409_05477_b200 import device as D
    world = 2
    mp.spawn(_mag_worker, args=(world, _port(), str(tmp_path)), nprocs=world, join=True)
    E, V = MAG16
    ev = D.random_stream(E, V, 42)
    want = oracle_mod.build(ev.cpu().numpy().view(oracle_mod.EVENT_DTYPE), V, True)
    del ev
    for r in range(world):
        got = np.load(os.path.join(tmp_path, f"mag_r{r}.npz"))
        lo, hi = (int(x) for x in got["rng"])
        a0, a1 = int(got["P"][r]), int(got["P"][r + 1])
        m = int(want["indptr"][-1])
        assert a0 == m * r // world and a1 == m * (r + 1) // world  # balanced by entries
        assert int(got["nrecv"]) == a1 - a0
        assert np.array_equal(got["ip"], np.clip(want["indptr"][lo:hi + 1], a0, a1) - a0), r
        for k, w in (("nb", "nbr"), ("ed", "eid"), ("ts", "ts")):
            assert np.array_equal(got[k], want[w][a0:a1]), (r, k)
        assert np.array_equal(got["fip"], want["indptr"]), r
        for k, w in (("fnb", "nbr"), ("fed", "eid"), ("fts", "ts")):
            assert np.array_equal(got[k], want[w]), (r, k)
