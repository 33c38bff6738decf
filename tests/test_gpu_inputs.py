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
