"""SURVEY 8(f) rank 2, training side: train_epoch's sample_batch queries generated on the device
(make_batches negatives, proj/src/training.cpp:157-182; min(workers, b) shards, :425-440;
forward_concat's [src | dst | neg] layout per call, :193-209), against the reference's own
make_batches (oracle/_ref), and an epoch of per-call-seeded sampling (mix_streams seeds,
:445-446) in one batched launch against the reference's sample_batch + build_sequence_batch."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def O():
    from oracle import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    return oracle


@pytest.mark.parametrize("B,npp,workers", [(200, 1, 1), (333, 3, 1), (250, 2, 3), (64, 1, 8),
                                           (1000, 5, 4), (5, 2, 8), (7, 1, 3)])
def test_train_queries_match_reference_make_batches(O, B, npp, workers):
    import torch
    from paper_2409_05477_b200 import device as D
    E, V = 20_000, 700
    ev = D.random_stream(E, V, 21)
    host = ev.cpu().numpy().view(O.EVENT_DTYPE)
    seed = D.mix_streams(123, 0x6e67, 3)
    want_n, want_t = O.ref_train_queries(host, V, B, npp, workers, seed)
    nodes, times = D.make_train_queries(ev, E, 0, -(-E // B), B, npp, workers, V, seed)
    assert np.array_equal(nodes.cpu().numpy(), want_n)
    assert np.array_equal(times.cpu().numpy(), want_t)
    # a batch range [b0, b1) is the matching slice of the whole epoch's queries
    nb = -(-E // B)
    b0, b1 = nb // 3, nb - 1
    part_n, _ = D.make_train_queries(ev, E, b0, b1, B, npp, workers, V, seed)
    q0 = b0 * B * (2 + npp)
    assert torch.equal(part_n, nodes[q0:q0 + part_n.numel()])


def test_train_epoch_sampling_one_launch(O):
    """workers = 1: every step is one sample_batch call of B*(2+npp) queries (the last one
    shorter) with seed mix_streams(cfg.seed, epoch*0x10001 + step, 0): one batched launch
    with per-call seeds equals the reference call by call (uniform-k, so the seeds matter)."""
    import torch
    from paper_2409_05477_b200 import device as D
    E, V, B, npp, k, l = 12_000, 300, 500, 2, 12, 13
    cfg_seed, epoch = 99, 5
    ev = D.random_stream(E, V, 8)
    host = ev.cpu().numpy().view(O.EVENT_DTYPE)
    g = D.build(ev, V, True)
    rg = O.RefStream(host, V).build(True, 0)[0]
    bseed = D.mix_streams(cfg_seed, 0x6e67, epoch)
    nodes, times = D.make_train_queries(ev, E, 0, -(-E // B), B, npp, 1, V, bseed)
    calls = D.train_calls(E, B, npp, 1, cfg_seed, epoch)
    seeds = torch.tensor([c[2] - (1 << 64) if c[2] >= 1 << 63 else c[2] for c in calls],
                         dtype=torch.int64, device="cuda")
    rows = D.sample_assemble_batched(g, nodes, times, B * (2 + npp), k, "random", seeds, l, E + 1,
                                     dt64=True)
    hn, ht = nodes.cpu().numpy(), times.cpu().numpy()
    for off, size, seed in calls[:6] + calls[-2:]:
        want, _ = O.ref_sample_assemble(rg, hn[off:off + size], ht[off:off + size], k, "random",
                                        seed, l, E + 1)
        got_ni = rows["node_index"][off:off + size].cpu().numpy()
        got_dt = rows["time_delta64"][off:off + size].cpu().numpy()
        assert np.array_equal(got_ni, want["node_index"])
        assert np.array_equal(got_dt, want["time_delta"])
