"""assemble_inputs (proj/src/attention.cpp:414-451) on the device,
fed by the sampler's rows, vs the reference's own assemble_inputs (oracle/_ref) and the
numpy restatement.  fp64 path: equal up to the rounding of cos and of omega*dt+phi (the
reference's compiler and nvcc both contract it to one fma): |dz| <= 1e-12 + 4 ulp(|arg|).
fp32 / bf16 outputs: the fp64 value rounded once."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _tol(dt, omega, phi):
    arg = np.abs(np.asarray(omega)).max() * np.abs(dt).max() + np.abs(np.asarray(phi)).max()
    return 1e-12 + 4 * np.spacing(arg)


@pytest.mark.parametrize("concat,dims", [(False, (32, 32, 32)), (True, (16, 24, 40))])
def test_assemble_inputs_matches_reference(oracle_mod, concat, dims):
    from paper_2409_05477_b200 import device as D
    E, V = 150_000, 3000
    d_v, d_e, d_t = dims
    ev = D.random_stream(E, V, 17)
    g = D.build(ev, V, True)
    nodes, times = D.make_queries(ev, 0, 20_000, 600, V)
    rows = D.sample_assemble(g, nodes, times, 10, "recent", 0, 11, E + 1, dt64=True)
    rng = np.random.default_rng(5)
    nt = rng.normal(size=(V + 1, d_v))
    et = rng.normal(size=(E + 2, d_e))
    om = rng.normal(size=d_t) * 1e-3
    ph = rng.normal(size=d_t)
    h = {k: v.cpu().numpy() for k, v in rows.items()}
    want = oracle_mod.ref_assemble_inputs(h["node_index"], h["edge_index"], h["time_delta64"],
                                          h["valid_len"], nt, et, om, ph, concat)
    restated = oracle_mod.assemble_inputs(h["node_index"], h["edge_index"], h["time_delta64"],
                                          h["valid_len"], nt, et, om, ph, concat)
    tol = _tol(h["time_delta64"], om, ph)
    assert np.abs(restated - want).max() <= tol
    dev = lambda a: torch.as_tensor(a, device="cuda")  # noqa: E731
    z64 = D.assemble_inputs({k: rows[k] for k in ("node_index", "edge_index", "valid_len",
                                                  "time_delta64")},
                            dev(nt), dev(et), dev(om), dev(ph), concat, torch.float64)
    assert np.abs(z64.cpu().numpy() - want).max() <= tol
    # compact pipeline: int32 indices + fp32 deltas + fp32 tables -> fp32 / bf16 z
    z32 = D.assemble_inputs({k: rows[k] for k in ("node_index", "edge_index", "valid_len",
                                                  "time_delta")},
                            dev(nt), dev(et), dev(om), dev(ph), concat, torch.float32)
    want32 = oracle_mod.ref_assemble_inputs(h["node_index"], h["edge_index"],
                                            h["time_delta"].astype(np.float64), h["valid_len"],
                                            nt, et, om, ph, concat)
    assert np.allclose(z32.cpu().numpy(), want32, rtol=2e-7, atol=2e-7)
    zb = D.assemble_inputs({k: rows[k] for k in ("node_index", "edge_index", "valid_len",
                                                 "time_delta")},
                           dev(nt).float(), dev(et).float(), dev(om), dev(ph), concat,
                           torch.bfloat16)
    assert np.allclose(zb.float().cpu().numpy(), want32, rtol=1e-2, atol=2e-2)


def test_assemble_inputs_rejects_out_of_table_index():
    from paper_2409_05477_b200 import ValidationError, device as D
    rows = dict(node_index=torch.tensor([[1, 9, 0]], dtype=torch.int32, device="cuda"),
                edge_index=torch.tensor([[1, 2, 0]], dtype=torch.int32, device="cuda"),
                valid_len=torch.tensor([2], dtype=torch.int32, device="cuda"),
                time_delta=torch.zeros((1, 3), dtype=torch.float32, device="cuda"))
    t = torch.zeros((5, 4), dtype=torch.float64, device="cuda")
    w = torch.zeros(4, dtype=torch.float64, device="cuda")
    with pytest.raises(ValidationError, match="outside embedding tables"):
        D.assemble_inputs(rows, t, t, w, w)


@pytest.mark.parametrize("strategy,concat,dims,tab,out", [
    ("recent", False, (32, 32, 32), torch.float64, torch.float64),
    ("recent", True, (16, 24, 40), torch.float32, torch.float32),
    ("recent", True, (8, 8, 48), torch.float32, torch.bfloat16),
    ("random", False, (32, 32, 32), torch.float64, torch.float64),  # composed path
])
def test_fused_sample_inputs_equals_composition(oracle_mod, strategy, concat, dims, tab, out):
    """tgfx_sample_inputs_device (sampler + assemble_inputs in one kernel for recent-k) equals
    assemble_inputs of the sampler's rows bit for bit (same fp64 deltas, same cos), and the
    reference's own assemble_inputs within the cos/fma tolerance."""
    from paper_2409_05477_b200 import device as D
    E, V, k, l = 120_000, 2500, 10, 11
    d_v, d_e, d_t = dims
    ev = D.random_stream(E, V, 23)
    g = D.build(ev, V, True)
    nodes, times = D.make_queries(ev, 1_000, 9_000, 600, V)
    rng = np.random.default_rng(6)
    dev = lambda a: torch.as_tensor(a, device="cuda")  # noqa: E731
    nt, et = dev(rng.normal(size=(V + 1, d_v))).to(tab), dev(rng.normal(size=(E + 2, d_e))).to(tab)
    om, ph = dev(rng.normal(size=d_t) * 1e-3), dev(rng.normal(size=d_t))
    z, vl = D.sample_inputs(g, nodes, times, k, strategy, 3, l, E + 1, nt, et, om, ph, concat,
                            out)
    rows = D.sample_assemble(g, nodes, times, k, strategy, 3, l, E + 1, dt64=True)
    want = D.assemble_inputs({kk: rows[kk] for kk in ("node_index", "edge_index", "valid_len",
                                                      "time_delta64")},
                             nt, et, om, ph, concat, out)
    assert torch.equal(vl, rows["valid_len"])
    assert torch.equal(z.view(torch.int16 if out == torch.bfloat16 else
                              (torch.int32 if out == torch.float32 else torch.int64)),
                       want.view(torch.int16 if out == torch.bfloat16 else
                                 (torch.int32 if out == torch.float32 else torch.int64)))
    if tab == torch.float64 and out == torch.float64:
        h = {kk: vv.cpu().numpy() for kk, vv in rows.items()}
        ref = oracle_mod.ref_assemble_inputs(h["node_index"], h["edge_index"], h["time_delta64"],
                                             h["valid_len"], nt.cpu().numpy(), et.cpu().numpy(),
                                             om.cpu().numpy(), ph.cpu().numpy(), concat)
        assert np.abs(z.cpu().numpy() - ref).max() <= _tol(h["time_delta64"], om.cpu().numpy(),
                                                           ph.cpu().numpy())


def test_fused_sample_inputs_rejects_small_tables():
    from paper_2409_05477_b200 import ValidationError, device as D
    E, V = 20_000, 300
    ev = D.random_stream(E, V, 2)
    g = D.build(ev, V, True)
    nodes, times = D.make_queries(ev, 0, 600, 600, V)
    t = torch.zeros((V + 1, 4), dtype=torch.float64, device="cuda")
    small_e = torch.zeros((10, 4), dtype=torch.float64, device="cuda")
    w = torch.zeros(4, dtype=torch.float64, device="cuda")
    with pytest.raises(ValidationError, match="outside embedding tables"):
        D.sample_inputs(g, nodes, times, 10, "recent", 0, 11, E + 1, t, small_e, w, w)


def test_fused_sample_inputs_edge_shapes():
    """l = 2 (only the self-loop token and one neighbour), k larger than l - 1, an empty query
    list, and queries before any event (empty prefixes: self token only)."""
    from paper_2409_05477_b200 import device as D
    E, V = 30_000, 400
    ev = D.random_stream(E, V, 12)
    g = D.build(ev, V, True)
    nodes, times = D.make_queries(ev, 0, 1200, 600, V)
    times = times.clone()
    times[:50] = -1.0  # before every event
    nt = torch.randn((V + 1, 16), device="cuda", dtype=torch.float64)
    et = torch.randn((E + 2, 16), device="cuda", dtype=torch.float64)
    om = torch.randn(16, device="cuda", dtype=torch.float64) * 1e-3
    ph = torch.randn(16, device="cuda", dtype=torch.float64)
    for k, l in ((10, 2), (3, 11), (30, 5)):
        z, vl = D.sample_inputs(g, nodes, times, k, "recent", 0, l, E + 1, nt, et, om, ph, False,
                                torch.float64)
        rows = D.sample_assemble(g, nodes, times, k, "recent", 0, l, E + 1, dt64=True)
        want = D.assemble_inputs({kk: rows[kk] for kk in ("node_index", "edge_index",
                                                          "valid_len", "time_delta64")},
                                 nt, et, om, ph, False, torch.float64)
        assert torch.equal(z, want) and torch.equal(vl, rows["valid_len"]), (k, l)
        assert int(vl[:50].max()) == 1  # self token only
    z0, v0 = D.sample_inputs(g, nodes[:0], times[:0], 10, "recent", 0, 11, E + 1, nt, et, om, ph)
    assert z0.numel() == 0 and v0.numel() == 0
