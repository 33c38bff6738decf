"""Per-config device timings for BASELINE.json's W / R / L shapes (and uniform-k on G) --
the parity-test configs, measured for DESIGN.md; the headline line is bench.py's.

    python profiles/bench_configs.py > profiles/r01/configs.txt

Each config: device-generated make_random_stream(E, V, 42), rev = 1 build (median of 5), then
every forward_concat batch [src | dst | neg] of B events sampled + packed, one launch per
batch as forward_concat calls it (seed 9 + batch), CUDA events around the whole sweep; and
the same batches (same per-batch seeds) as one tgfx_sample_assemble_batched_device launch.  W and R are launch-latency-bound (a batch is ~1,800
queries), so µs/batch is the figure of merit there."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_05477_b200 import device as D  # noqa: E402

CFG = {
    "W": dict(E=157_474, V=9227, strat="recent", k=10, l=11, B=600, hops=1),
    "R": dict(E=672_447, V=10_984, strat="recent", k=10, l=11, B=600, hops=2),
    "L": dict(E=1_293_103, V=1980, strat="random", k=20, l=21, B=4000, hops=1),
    "G-uniform20": dict(E=191_290_882, V=16682, strat="random", k=20, l=21, B=600, hops=1,
                        max_queries=48_000_000),
}


def timed(fn, reps=5):
    ts = []
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts[1:])


def run(name, c):
    E, V, k, l, B = c["E"], c["V"], c["k"], c["l"], c["B"]
    ev = D.random_stream(E, V, 42)
    g = D.build(ev, V, True)
    build_ms = timed(lambda: D.rebuild(g, ev, trusted=True))
    nodes, times = D.make_queries(ev, 0, E, B, V)
    qmax = c.get("max_queries", nodes.numel())
    nodes, times = nodes[:qmax], times[:qmax]
    Q, qb = nodes.numel(), 3 * B
    batches = [(s, min(Q, s + qb)) for s in range(0, Q, qb)]
    if c["hops"] == 1:
        out = D.alloc_rows(qb, l)

        def per_batch():
            for i, (s, e) in enumerate(batches):
                sub = {kk: vv[:e - s] for kk, vv in out.items()}
                D.sample_assemble(g, nodes[s:e], times[s:e], k, c["strat"], 9 + i, l, E + 1,
                                  out=sub, trusted=True)
        big = D.alloc_rows(Q, l)
        seeds = torch.arange(9, 9 + len(batches), dtype=torch.int64, device="cuda")
        # the same per-batch seeds (9 + b) as the per-batch loop, in one launch
        one = lambda: D.sample_assemble_batched(g, nodes, times, qb, k, c["strat"], seeds, l,  # noqa: E731
                                                E + 1, out=big, trusted=True)
    else:
        out = dict(h1=D.alloc_rows(qb, l), h2=D.alloc_rows(qb * k, l))

        def per_batch():
            for i, (s, e) in enumerate(batches):
                D.two_hop(g, nodes[s:e], times[s:e], k, k, c["strat"], 9 + i, l, E + 1,
                          out=dict(h1={kk: vv[:e - s] for kk, vv in out["h1"].items()},
                                   h2={kk: vv[:(e - s) * k] for kk, vv in out["h2"].items()}),
                          trusted=True)
        big = dict(h1=D.alloc_rows(Q, l), h2=D.alloc_rows(Q * k, l))
        one = lambda: D.two_hop(g, nodes, times, k, k, c["strat"], 9, l, E + 1, out=big,  # noqa: E731
                                trusted=True)
    pb = timed(per_batch, 3)
    ob = timed(one, 3)
    hop2 = ""
    if c["hops"] == 2:
        rows = int((big["h2"]["valid_len"] > 0).sum().item())
        hop2 = f", {rows:,} hop-2 rows ({rows / (ob * 1e-3) / 1e6:,.1f} M rows/s in one launch)"
    print(f"{name}: E={E:,} V={V:,} {c['strat']}-{k} l={l} B={B}: build {build_ms:.3f} ms "
          f"({E / (build_ms * 1e-3) / 1e9:.2f} G edges/s); {Q:,} queries in {len(batches)} "
          f"batches: {pb:.2f} ms = {1e3 * pb / len(batches):.1f} us/batch "
          f"({Q / (pb * 1e-3) / 1e6:,.0f} M q/s); one launch {ob:.2f} ms "
          f"({Q / (ob * 1e-3) / 1e6:,.0f} M q/s){hop2}", flush=True)
    del g, ev, nodes, times, out, big
    torch.cuda.empty_cache()


if __name__ == "__main__":
    for name in (sys.argv[1:] or CFG):
        run(name, CFG[name])
