"""Fused sampler + assemble_inputs (tgfx_sample_inputs_device) against the two-launch composition
(sample_assemble rows -> assemble_inputs), device time per call, on the Wikipedia and GDELT
shapes: forward_concat batches of 1,800 queries and one large call, d_model 32 (sum) and
32+32+32 (concat), f32 tables and z."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_05477_b200 import device as D  # noqa: E402


def timeit(fn, reps=20):
    st = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    out = []
    for name, E, V in (("W", 157_474, 9227), ("G-prefix", 20_000_000, 16682)):
        ev = D.random_stream(E, V, 42)
        g = D.build(ev, V, True)
        for q_ev in (600, 200_000):
            nodes, times = D.make_queries(ev, E // 2, E // 2 + q_ev, 600, V)
            gen = torch.Generator(device="cuda").manual_seed(1)
            for concat, dims in ((False, (32, 32, 32)), (True, (32, 32, 32))):
                d_v, d_e, d_t = dims
                nt = torch.randn((V + 1, d_v), device="cuda", generator=gen)
                et = torch.randn((E + 2, d_e), device="cuda", generator=gen)
                om = torch.randn(d_t, device="cuda", dtype=torch.float64, generator=gen) * 1e-3
                ph = torch.randn(d_t, device="cuda", dtype=torch.float64, generator=gen)

                def comp():
                    rows = D.sample_assemble(g, nodes, times, 10, "recent", 0, 11, E + 1,
                                             trusted=True)
                    return D.assemble_inputs(rows, nt, et, om, ph, concat, torch.float32,
                                             trusted=True)

                def fused():
                    return D.sample_inputs(g, nodes, times, 10, "recent", 0, 11, E + 1, nt, et,
                                           om, ph, concat, torch.float32, trusted=True)
                tc, tf = timeit(comp), timeit(fused)
                out.append(dict(graph=name, queries=nodes.numel(), concat=concat,
                                composed_ms=round(tc, 4), fused_ms=round(tf, 4),
                                speedup=round(tc / tf, 2)))
                print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
