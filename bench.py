#!/usr/bin/env python
"""bench.py -- TF-TGN hot path on B200: T-CSR build + most-recent-k sampling + sequence packing.

Workload (BASELINE.json configs[3], GDELT-shaped; the metric's 1/2/4/8-GPU config):
  make_random_stream(E=191,290,882, V=16,682, seed=42, zipf=1.2) generated on the device
  (bit-identical to the reference generator), reverse=1 T-CSR build, then recent-10
  sampling + suffix-infill packing (l=11) of every query of every event in the
  forward_concat layout [src | dst | neg] per batch of B=600 events (573,872,646 queries),
  processed in chunks.  One step = one full rebuild of the T-CSR from the resident event
  stream + sampling/packing of all queries.  value = events through the path per second
  (edges/s); the build and sampler rates are reported beside it.

Timing: CUDA events on the launching stream, W untimed warm-up steps, K timed steps bracketed
by barrier + synchronize, max over ranks.  Inputs (6.1 GB events, 9.2 GB queries) exceed the
126 MB L2.  `e2e` repeats the step through the C ABI's host-buffer calls (tgfx_build_parallel
+ tgfx_sample_assemble with pinned host inputs/outputs; H2D/D2H inside the timed region).
`cpu_baseline` / --impl reference time the reference's own CPU code (oracle/_ref, compiled
from /root/reference) on a bounded prefix sample of the same workload.

Multi-GPU (torchrun, one process per GPU): default plan "strong": one pass, whole-batch query
shards (each rank generates only its shard's queries; stream_base keeps rows identical to 1 GPU),
every rank rebuilding its T-CSR replica from the stream; value = E / max-over-ranks step time.
The line adds `build_partitioned`: the node-range / entry-position partitioned build (one
all-to-all) and its replication, timed separately.  --config M / M16 make that partitioned build
+ replication the step's build.  --plan weak: every rank a full data-parallel pass with its own
negatives (neg_seed + rank).  No collective touches the sampling path; only the timing max over
ranks and the partitioned build's exchange.
"""
import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (E, V, strategy, k, l, B, two_hop)
    "G": dict(E=191_290_882, V=16682, strategy="recent", k=10, l=11, B=600,
              name="GDELT-shaped synthetic (V=16,682, E=191,290,882, Zipf 1.2)"),
    "W": dict(E=157_474, V=9227, strategy="recent", k=10, l=11, B=600,
              name="Wikipedia-shaped synthetic (V=9,227, E=157,474)"),
    "L": dict(E=1_293_103, V=1980, strategy="random", k=20, l=21, B=4000,
              name="LastFM-shaped synthetic (V=1,980, E=1,293,103)"),
    # Reddit-shaped (BASELINE configs[1]): 2-hop recent 10x10 of every root;
    # hop-2 rows [Q, k1, l] beside the hop-1 rows (device path only: no e2e / CPU legs)
    "R": dict(E=672_447, V=10_984, strategy="recent", k=10, l=11, B=600, two_hop=True,
              name="Reddit-shaped synthetic (V=10,984, E=672,447, Zipf 1.2), 2-hop recent 10x10"),
    # MAG-shaped (BASELINE configs[4]): at N > 1 the T-CSR comes from the node-range-partitioned
    # build (one NCCL all-to-all) + all-gather replication, then query-sharded sampling.  The
    # full shape needs N >= 4 (41.6 GB stream + 63 GB T-CSR + records per replica); M16 is the
    # 1/16 scale the parity tests use (fits one GPU).
    "M": dict(E=1_300_000_000, V=121_000_000, strategy="recent", k=10, l=11, B=600,
              partitioned=True, name="MAG-shaped synthetic (V=121,000,000, E=1,300,000,000, Zipf 1.2)"),
    "M16": dict(E=81_250_000, V=7_562_500, strategy="recent", k=10, l=11, B=600,
                partitioned=True,
                name="1/16-scale MAG-shaped synthetic (V=7,562,500, E=81,250,000, Zipf 1.2)"),
}
SEED, NEG_SEED, ZIPF = 42, 7, 1.2


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            time.sleep(0.25)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for line in (self.out or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------------------ CPU reference
def reference_full(cfg, threads, steps, warmup, ev_host=None, builds=("sequential", "parallel"),
                   batches_per_step=64):
    """The reference's own CPU path (oracle/_ref: /root/reference/proj/src compiled, loaded in
    the build for this host's CPU when it can run it) on the SAME workload as the GPU arm:

      * stream: the full make_random_stream(E, V, 42) -- generated by the reference's own
        generator unless ev_host is given;
      * build: one full reverse=1 build of all E events, timed once per run (build_sequential,
        and build_parallel(threads) -- the faster one counts);
      * sampling: forward_concat batches (3B queries: [src | dst | neg], seed 9 + batch index,
        sample_batch + build_sequence_batch as training.cpp:211-214 calls them) spread evenly
        over the WHOLE stream, `batches_per_step` per step, `warmup` untimed + `steps` timed;
        the per-query time of the timed steps is extrapolated to all 3E queries.

    value = E / (t_build + t_query * 3E): events through build + sampling per second."""
    import numpy as np
    from oracle import oracle as O
    O.ref(native=True)
    E, V, B = cfg["E"], cfg["V"], cfg["B"]
    t0 = time.perf_counter()
    if ev_host is None:
        ev_host = O.ref_make_random_stream(E, V, SEED)
    t_gen = time.perf_counter() - t0
    rs = O.RefStream(ev_host, V)
    bt = {}
    rg = None
    for kind in builds:
        g, secs = rs.build(True, 0 if kind == "sequential" else threads)
        bt[kind] = secs
        if rg is None:
            rg = g  # both builders return the same T-CSR
        del g
    t_build = min(bt.values())
    del rs
    nbatch = -(-E // B)
    per_step = []
    for s in range(warmup + steps):
        # batch indices spread over the stream; each step a different evenly spaced set
        frac = (s + 0.5) / (warmup + steps)
        bs = sorted({min(nbatch - 1, int((j + frac) * nbatch / batches_per_step))
                     for j in range(batches_per_step)})
        tq, nq = 0.0, 0
        for b in bs:
            e0, e1 = b * B, min(E, (b + 1) * B)
            nodes, times = O.make_queries(ev_host, e0, e1, B, V, NEG_SEED)
            _, secs = O.ref_sample_assemble(rg, nodes, times, cfg["k"], cfg["strategy"], 9 + b,
                                            cfg["l"], E + 1, threads=threads, want_outputs=False)
            tq += secs
            nq += len(nodes)
        if s >= warmup:
            per_step.append((tq, nq))
    tq = sum(t for t, _ in per_step)
    nq = sum(n for _, n in per_step)
    t_query = tq / max(nq, 1)
    Q = 3 * E
    total = t_build + t_query * Q
    return dict(value=E / total, total_s=total, build_s=t_build, builds=bt, gen_s=t_gen,
                t_query=t_query, queries_timed=nq, batches_timed=len(per_step) * batches_per_step,
                build_edges_per_s=E / t_build, sample_queries_per_s=1.0 / t_query,
                so=os.path.basename(O._ref_path or ""))


def _event_dtype():
    import numpy as np
    return np.dtype([("edge_id", "<i8"), ("src", "<i8"), ("dst", "<i8"), ("timestamp", "<f8")])


def reference_sample_text(cfg, r, threads):
    bt = ", ".join(f"{k} {v:.2f}s" for k, v in r["builds"].items())
    return (f"full {cfg['name']} stream ({cfg['E']:,} events): one reference build of all events "
            f"timed once ({bt}; the faster counts) + sample_batch+build_sequence_batch of "
            f"{r['queries_timed']:,} forward_concat queries from {r['batches_timed']} batches "
            f"spread over the whole stream ({threads} threads), per-query time extrapolated to "
            f"all {3 * cfg['E']:,} queries; reference compiled {r['so']}")


def run_reference(args, cfg):
    ws, rank, local = dist_setup()
    if rank != 0:
        return 0
    threads = len(os.sched_getaffinity(0))
    r = reference_full(cfg, threads, args.steps, args.warmup)
    value = r["value"]
    line = {
        "impl": "reference", "metric": metric_name(cfg), "value": value, "unit": "edges/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * r["total_s"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int64/f64", "data": "synthetic (reference generator)",
        "config": dict(config_obj(cfg, ws), parallelism=(
            f"reference CPU path (oracle/_ref, /root/reference/proj/src compiled -O3 "
            f"-march for this host), {threads} host threads on rank 0"
            + (f"; ranks 1..{ws - 1} idle" if ws > 1 else ""))),
        "cpu_baseline": {"value": value, "unit": "edges/s", "cores": threads, "kind": "reference",
                         "sample": reference_sample_text(cfg, r, threads)},
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "same_config": True,
        "extrapolation": "ms_per_step = build (timed once) + per-query sampling time x 3E",
        "build_s": r["build_s"], "builds_s": r["builds"],
        "build_edges_per_s": r["build_edges_per_s"],
        "sample_queries_per_s": r["sample_queries_per_s"],
    }
    print(json.dumps(line), flush=True)
    return 0


def metric_name(cfg):
    return ("T-CSR build edges/s + sampled queries/s (events through build + recent-k "
            "sampling/packing per second)")


def config_obj(cfg, ws, weak=True):
    E, V = cfg["E"], cfg["V"]
    if ws == 1:
        par = "1 GPU"
    elif weak:
        par = (f"dp{ws}: {ws} data-parallel workers, each a full pass (own T-CSR replica, "
               f"own negatives neg_seed+rank); no collective in the step")
    elif cfg.get("partitioned"):
        par = (f"node-range-partitioned build x{ws} (one all-to-all) + replication, then "
               f"query-sharded sampling x{ws} (whole batches, stream_base)")
    else:
        par = (f"query-sharded x{ws} (whole batches, stream_base), T-CSR replicated (each rank "
               f"builds it from the stream)")
    return {"workload": cfg["name"] + f"; reverse=1 T-CSR build + {cfg['strategy']}-{cfg['k']} "
                                      f"sampling, l={cfg['l']}, all 3E queries, batch {cfg['B']}",
            "events": E, "num_nodes": V, "queries": 3 * E, "k": cfg["k"],
            "seq_len": cfg["l"], "batch": cfg["B"], "reverse": 1,
            "parallelism": par,
            "l2_flush": (f"inputs larger than L2 ({32 * E / 1e9:.1f} GB events, "
                         f"{48 * E / 1e9:.1f} GB queries vs 126 MB L2)")}


# ------------------------------------------------------------------------------ our path
def run_ours(args, cfg):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2409_05477_b200 import _lib, device as D, shard as S

    ws, rank, local = dist_setup()
    # TGFX_BENCH_SHARE_GPU=1: test mode for the N>1 code path on a 1-GPU box -- all ranks on
    # device 0, gloo for the (timing-only) collectives
    share = os.environ.get("TGFX_BENCH_SHARE_GPU") == "1"
    torch.cuda.set_device(0 if share else local)
    red = "cpu" if share else "cuda"
    if ws > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    E, V, k, l, B = cfg["E"], cfg["V"], cfg["k"], cfg["l"], cfg["B"]
    strat = cfg["strategy"]
    Q = 3 * E
    stream = torch.cuda.current_stream()
    weak = args.plan == "weak"
    # weak: every rank is one data-parallel worker running a full pass (its own negatives);
    # strong: one pass, whole-batch query shards across ranks (shard.py)
    neg_seed = S.weak_neg_seed(NEG_SEED, rank) if weak else NEG_SEED

    # resident inputs: event stream (generated on device) and this rank's queries
    ev = D.random_stream(E, V, SEED)
    q_lo, q_hi = (0, Q) if weak else S.shard_range(Q, 3 * B, ws, rank)
    nodes = torch.empty(max(q_hi - q_lo, 1), dtype=torch.int64, device="cuda")
    times = torch.empty(max(q_hi - q_lo, 1), dtype=torch.float64, device="cuda")
    # whole batches per generation call keep the [src|dst|neg] batch layout (shards are whole
    # batches, so query q of the shard belongs to event (q_lo + q) // 3's batch)
    step_ev = (8_000_000 // B) * B
    for e0 in range(q_lo // 3, q_hi // 3, step_ev):
        e1 = min(q_hi // 3, e0 + step_ev)
        D.make_queries(ev, e0, e1, B, V, neg_seed, nodes=nodes[3 * e0 - q_lo:3 * e1 - q_lo],
                       times=times[3 * e0 - q_lo:3 * e1 - q_lo])
    chunk = args.chunk
    chunks = S.chunks(q_lo, q_hi, chunk)
    two = bool(cfg.get("two_hop"))
    if two:  # hop-1 rows + hop-2 rows [q, k, l] per chunk
        cq = min(chunk, max(q_hi - q_lo, 1))
        out = dict(h1=D.alloc_rows(cq, l), h2=D.alloc_rows(cq * k, l))
        args.no_e2e = args.no_cpu = True
    else:
        out = D.alloc_rows(min(chunk, max(q_hi - q_lo, 1)), l)
    # the T-CSR every rank samples: a local build of the whole stream (a replica), or for the
    # partitioned configs at N > 1 the node-range-partitioned build + all-gather replication
    part = bool(cfg.get("partitioned")) and ws > 1
    ev_part = None
    if part:
        from paper_2409_05477_b200 import partition as PT
        e_lo, e_hi = E * rank // ws, E * (rank + 1) // ws  # rank r holds the r-th stream chunk
        ev_part = ev[e_lo * 32:e_hi * 32].clone()
        del ev
        ev = None
        torch.cuda.empty_cache()
        g = PT.build_partitioned(ev_part, V, True, E, replicate=True, exchange_on_host=share)["full"]
    else:
        g = D.build(ev, V, True)
    torch.cuda.synchronize()

    # stratified row sample per chunk (64 rows) whose device-path result the e2e leg's host
    # rows are checked against on every e2e step
    rng = np.random.default_rng(1234)
    probe = [np.sort(np.unique(((np.arange(64) + rng.random(64)) * (e - s) / 64).astype(np.int64)))
             for s, e in chunks]
    expect = []

    # check_query (sampler.cpp:22-27) runs inside the sampler kernel for every query (fused
    # check): the kernels record the first failing global query index in `first_bad`, read
    # once per step (one 8-byte copy + sync inside the timed region) and raised like the
    # reference's ValidationError
    first_bad = D.first_bad_word()

    graph = [g]
    del g

    def one_step(record=None, taken=None):
        if record:
            record["b0"].record(stream)
        if part:  # partitioned build + all-gather replication (collectives inside)
            graph[0] = None
            graph[0] = PT.build_partitioned(ev_part, V, True, E, replicate=True,
                                            exchange_on_host=share)["full"]
        else:
            D.rebuild(graph[0], ev, trusted=True)
        g = graph[0]
        if record:
            record["b1"].record(stream)
        first_bad.fill_(-1)
        for i, (s, e) in enumerate(chunks):
            if record:
                record["c"][i][0].record(stream)
            if two:
                sub2 = dict(h1={kk: vv[: e - s] for kk, vv in out["h1"].items()},
                            h2={kk: vv[: (e - s) * k] for kk, vv in out["h2"].items()})
                D.two_hop(g, nodes[s - q_lo:e - q_lo], times[s - q_lo:e - q_lo], k, k, strat, 9,
                          l, E + 1, out=sub2)
                if record:
                    record["c"][i][1].record(stream)
                if taken is not None:
                    taken.append(int(sub2["h1"]["valid_len"].sum().item()) - (e - s))
                    taken2.append(int((sub2["h2"]["valid_len"].clamp(min=1) - 1).sum().item()))
                continue
            sub = {kk: vv[: e - s] for kk, vv in out.items()}
            D.sample_assemble(g, nodes[s - q_lo:e - q_lo], times[s - q_lo:e - q_lo], k, strat, 9,
                              l, E + 1, out=sub,
                              stream_base=s, first_bad=first_bad)
            if record:
                record["c"][i][1].record(stream)
            if taken is not None:  # warm-up only (the rows buffer is reused by every chunk)
                taken.append(int(sub["valid_len"].sum().item()) - (e - s))
                ix = torch.from_numpy(probe[i]).to(sub["valid_len"].device)
                expect.append({kk: vv[ix].cpu().numpy() for kk, vv in sub.items()})
        D.query_error(nodes, first_bad, stream_base=q_lo)

    taken, taken2 = [], []
    for w in range(args.warmup):
        one_step(taken=taken if w == 0 else None)
    if not taken:
        one_step(taken=taken)
    total_taken = sum(taken)

    ev_rec = [dict(b0=torch.cuda.Event(enable_timing=True), b1=torch.cuda.Event(enable_timing=True),
                   c=[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                      for _ in chunks]) for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _lib.launch_count()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(0 if share else local) as clk:
        start.record(stream)
        for s in range(args.steps):
            one_step(record=ev_rec[s])
        end.record(stream)
        torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    # build + int64 columns (untimed in the step): the step's build writes the sampler's 16-byte
    # gather records {u32 nbr, u32 eid, f64 ts} and ts; the reference's int64 neighbor_ids /
    # edge_ids columns are widened from the records on demand (k_widen).  Timed here as
    # rebuild + widening, the full reference-layout T-CSR.
    w_ms = []
    for _ in range(0 if part else 3):
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        D.rebuild(graph[0], ev, trusted=True)
        D.graph_tensors(graph[0])
        a1.record(stream)
        torch.cuda.synchronize()
        w_ms.append(a0.elapsed_time(a1))
    build_i64_ms = S.max_over_ranks([statistics.median(w_ms) if w_ms else 0.0], device=red)[0]
    # N > 1: the node-range-partitioned build (degree all-reduce, one all-to-all
    # of 32-byte records, local stable build of the owned range), timed on its own, and the
    # all-gather that replicates it for query-sharded sampling
    build_part = None
    if ws > 1:  # an auxiliary measurement: a failure here is reported, not fatal to the line
        try:
            build_part = measure_partitioned(ev_part if part else ev, E, V, ws, rank, share, red,
                                             stream, owned_chunk=part)
        except Exception as e:  # noqa: BLE001
            build_part = {"error": f"{type(e).__name__}: {e}"[:300]}
    total_ms = start.elapsed_time(end)
    build_ms = [r["b0"].elapsed_time(r["b1"]) for r in ev_rec]
    samp_launch_ms = [a.elapsed_time(b) for r in ev_rec for (a, b) in r["c"]]
    samp_ms = [sum(a.elapsed_time(b) for (a, b) in r["c"]) for r in ev_rec]
    # max over ranks (device-timed), sums of work
    total_ms, build_med, samp_med = S.max_over_ranks(
        [total_ms, statistics.median(build_ms), statistics.median(samp_ms)], device=red)
    q_local = q_hi - q_lo
    local_taken = total_taken
    q_all, taken_all = (int(x) for x in S.sum_over_ranks([q_local, local_taken], device=red))
    ms_per_step = total_ms / args.steps
    replicas = ws if weak else 1  # passes over the stream the job completes per step

    peak, peak_src = load_peaks()
    # algorithmic bytes, this rank's launches
    build_bytes = 32 * E + 24 * 2 * E + 8 * (V + 1)
    samp_bytes_local = 16 * q_local + 16 * q_local + 24 * local_taken + (12 * l + 4) * q_local
    if two:  # + hop-2: every hop-1 entry is a query (indptr pair + its window), k rows per root
        samp_bytes_local += 16 * local_taken + 24 * sum(taken2) + (12 * l + 4) * k * q_local
    avg_launch_ms = statistics.mean(samp_launch_ms)
    bytes_per_launch = samp_bytes_local / max(len(chunks), 1)
    achieved = bytes_per_launch / (avg_launch_ms * 1e-3) / 1e9
    traffic = load_traffic(cfg, bytes_per_launch)

    line = {
        "metric": metric_name(cfg), "value": replicas * E / (ms_per_step * 1e-3),
        "unit": "edges/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak" if weak else "strong", "vs_baseline": None,
        "dtype": "int64/f64 (T-CSR), int32/fp32 (sequence tensors)",
        "data": "synthetic (device generator, bit-identical to tgf::make_random_stream)",
        "config": config_obj(cfg, ws, weak),
        "build": {"ms": build_med, "edges_per_s": replicas * E / (build_med * 1e-3),
                  "alg_bytes": build_bytes,
                  "achieved_gbs": build_bytes / (build_med * 1e-3) / 1e9,
                  "frac": build_bytes / (build_med * 1e-3) / 1e9 / peak},
        "build_int64": None if part else {
                        "ms": build_i64_ms, "edges_per_s": E / (build_i64_ms * 1e-3),
                        "frac": build_bytes / (build_i64_ms * 1e-3) / 1e9 / peak,
                        "what": "rebuild + k_widen of the int64 neighbor_ids/edge_ids columns "
                                "(the reference TCsr layout); not part of the step"},
        "sample": {"ms": samp_med, "queries_per_s": q_all / (samp_med * 1e-3),
                   **({"hop2_rows_per_s": k * q_all / (samp_med * 1e-3),
                       "mean_taken_hop2": sum(taken2) / max(local_taken, 1)} if two else {}),
                   "launches_per_step": len(chunks), "mean_taken": taken_all / max(q_all, 1)},
        "roofline": {"kernel": ("k_recent_line x3 (2-hop: hop-1 rows, hop-1 entries, hop-2 rows)"
                                if two else
                                "k_recent_line (fused recent-k line-probe sampler + sequence packing)"),
                     "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "alg_bytes_per_launch": bytes_per_launch,
                     "avg_launch_ms": avg_launch_ms,
                     # SURVEY 8(d) algorithmic bytes count every window read as HBM traffic;
                     # most windows are L2 hits, so frac can exceed 1.  dram_frac is the ncu-
                     # measured DRAM traffic per launch (traffic) over the same launch time.
                     "dram_frac": (traffic / (avg_launch_ms * 1e-3) / 1e9 / peak
                                   if traffic else None)},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if build_part is not None:
        line["build_partitioned"] = build_part
    if part:
        line["build"]["what"] = ("partitioned build + all-gather replication per step "
                                 "(partition.build_partitioned, NCCL)")
    ev_host = None
    if rank == 0 and not args.no_cpu:
        ev_host = ev.cpu().numpy().view(_event_dtype())  # bit-identical to the reference's
    if not args.no_e2e:
        # the device-resident run's graph, rows and inputs are not part of the e2e path: the
        # e2e step starts from the device memory a fresh host-buffer caller would have
        graph.clear()
        del out
        dev_inputs = {"ev": ev, "nodes": nodes, "times": times}
        del ev, nodes, times
        import gc
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        e2e = run_e2e(args, cfg, dev_inputs, chunks, ws, rank, weak, red, probe, expect)
        if rank == 0:
            line["e2e"] = e2e
    if rank == 0 and not args.no_e2e:
        line["e2e_cpp"] = run_e2e_cpp(cfg)
    if rank == 0 and not args.no_cpu:
        threads = len(os.sched_getaffinity(0))
        r = reference_full(cfg, threads, steps=3, warmup=1, ev_host=ev_host,
                           builds=("sequential",), batches_per_step=48)
        line["cpu_baseline"] = {
            "value": r["value"], "unit": "edges/s", "cores": threads, "kind": "reference",
            "sample": reference_sample_text(cfg, r, threads),
            "build_edges_per_s": r["build_edges_per_s"],
            "sample_queries_per_s": r["sample_queries_per_s"]}
        del ev_host
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def measure_partitioned(ev_any, E, V, ws, rank, share, red, stream, owned_chunk=False, reps=3):
    """Device time (max over ranks) of partition.build_partitioned without replication, and of
    one replication all-gather.  ev_any: the whole stream (a rank takes its chunk) or, with
    owned_chunk, this rank's chunk already."""
    import torch
    import torch.distributed as dist
    from paper_2409_05477_b200 import partition as PT, shard as S
    if owned_chunk:
        ev_loc = ev_any
    else:
        e_lo, e_hi = E * rank // ws, E * (rank + 1) // ws
        ev_loc = ev_any[e_lo * 32:e_hi * 32]
    ms = []
    for i in range(reps + 1):
        dist.barrier()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        r = PT.build_partitioned(ev_loc, V, True, E, replicate=False, exchange_on_host=share)
        a1.record(stream)
        torch.cuda.synchronize()
        if i:
            ms.append(a0.elapsed_time(a1))
        del r
    dist.barrier()
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r = PT.build_partitioned(ev_loc, V, True, E, replicate=False, exchange_on_host=share)
    torch.cuda.synchronize()
    dist.barrier()
    a0.record(stream)
    full = PT.replicate(r, V, E, True, exchange_on_host=share)
    a1.record(stream)
    torch.cuda.synchronize()
    rep_ms = a0.elapsed_time(a1)
    sent = int(r.get("sent_records", 0))
    del full, r
    med = sorted(ms)[len(ms) // 2]
    med, rep_ms = S.max_over_ranks([med, rep_ms], device=red)
    sent_all = int(S.sum_over_ranks([sent], device=red)[0])
    return {"ms": med, "edges_per_s": E / (med * 1e-3), "ranks": ws,
            "exchange_bytes": 32 * sent_all, "replicate_ms": rep_ms,
            "what": "node-range-partitioned build: degree all-reduce, one all-to-all of 32-byte "
                    "records, local stable build of each owned range (aggregate events/s); "
                    "replicate_ms = the all-gather + import that gives every rank the full "
                    "T-CSR for query-sharded sampling",
            "collectives": "gloo, host-staged (1-GPU test mode)" if share else "NCCL"}


def load_traffic(cfg, bytes_per_launch):
    """DRAM bytes per k_recent launch from the committed ncu --set full summary, scaled from
    the profiled launch's query count to this launch (null if absent)."""
    if cfg is not CONFIGS["G"]:  # the committed capture is of the GDELT-shaped launch
        return None
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    try:
        with open(p) as f:
            d = json.load(f)
        t = d["k_recent_line"]
        return t["dram_bytes"] * bytes_per_launch / t["alg_bytes"]
    except Exception:
        return None


def run_e2e_cpp(cfg, batches=2000, warmup=50):
    """The drop-in C++ route (tools/forward_concat_bench.cpp, linked against libtgformer.so):
    tgf::build_parallel of the whole stream + forward_concat's per-batch pair
    tgf::sample_batch -> tgf::build_sequence_batch ("exact"), and the one-call
    tgf::sample_sequence_batch ("fused"), on forward_concat batches spread over the stream,
    per-query time extrapolated to all 3E queries.  Wall clock, host vectors in and out."""
    exe = os.path.join(ROOT, "paper_2409_05477_b200", "lib", "forward_concat_bench")
    out = {}
    for mode, name in ((0, "exact"), (1, "fused")):
        try:
            r = subprocess.run([exe, str(cfg["E"]), str(cfg["V"]), str(cfg["k"]), str(cfg["l"]),
                                str(cfg["B"]), cfg["strategy"], str(batches), str(warmup),
                                str(mode)], capture_output=True, text=True, timeout=600)
            d = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception as e:  # report, do not fail the bench line
            out[name] = {"error": f"{type(e).__name__}: {e}"}
            continue
        d["path"] = ("tgf::build_parallel + per batch tgf::sample_batch -> "
                     "tgf::build_sequence_batch (training.cpp:211-214)" if mode == 0 else
                     "tgf::build_parallel + per batch tgf::sample_sequence_batch")
        d["extrapolation"] = (f"{batches} forward_concat batches of {3 * cfg['B']} queries spread "
                              f"over the stream; per-query time x {3 * cfg['E']:,} queries")
        out[name] = d
    return out


def run_e2e(args, cfg, dev_inputs, chunks, ws, rank, weak, red="cuda", probe=None, expect=None):
    """Same step through the C ABI with HOST buffers (pinned): tgfx_build_parallel from host
    events, then tgfx_sample_assemble per chunk with host queries and host outputs.  At N > 1
    every rank runs it at once (PCIe and host memory are shared, as in a real job) when the
    host has the memory for N pinned copies; wall time is the max over ranks."""
    import numpy as np
    import torch
    from paper_2409_05477_b200 import _lib
    from paper_2409_05477_b200 import shard as S
    L = _lib.lib()
    E, V, k, l = cfg["E"], cfg["V"], cfg["k"], cfg["l"]
    need = 32 * E + 16 * (chunks[-1][1] - chunks[0][0]) + (12 * l + 4) * args.chunk
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = float("inf")
    # all ranks pin their own copies at once if every rank sees room for N copies (decided
    # collectively so every rank takes the same branch)
    short = S.max_over_ranks([0.0 if avail > 1.25 * ws * need else 1.0], device=red)[0]
    everyone = ws == 1 or short == 0.0
    active = everyone or rank == 0
    if not active:  # rank 0 alone measures; the others only join the collectives
        torch.distributed.barrier()
        S.max_over_ranks([0.0], device=red)
        S.sum_over_ranks([0], device=red)
        return None
    ev, nodes, times = dev_inputs["ev"], dev_inputs["nodes"], dev_inputs["times"]
    h_ev = torch.empty(ev.numel(), dtype=torch.uint8, pin_memory=True)
    h_ev.copy_(ev)
    lo, hi = chunks[0][0], chunks[-1][1]
    h_nodes = torch.empty(hi - lo, dtype=torch.int64, pin_memory=True)
    h_times = torch.empty(hi - lo, dtype=torch.float64, pin_memory=True)
    # the resident query arrays hold this rank's shard [q_lo, q_hi) = [lo, hi)
    h_nodes.copy_(nodes[:hi - lo])
    h_times.copy_(times[:hi - lo])
    del ev, nodes, times
    dev_inputs.clear()  # inputs now live in pinned host memory only
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    cmax = max(e - s for s, e in chunks)
    o_n = torch.empty(cmax * l, dtype=torch.int32, pin_memory=True)
    o_e = torch.empty(cmax * l, dtype=torch.int32, pin_memory=True)
    o_d = torch.empty(cmax * l, dtype=torch.float32, pin_memory=True)
    o_v = torch.empty(cmax, dtype=torch.int32, pin_memory=True)
    strat = 0 if cfg["strategy"] == "recent" else 1
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731

    # numpy views of the pinned outputs: the probe rows of each chunk are copied aside right
    # after its call (a few KB) and checked against the device path after the step
    v_n, v_e, v_d, v_v = (t.numpy() for t in (o_n, o_e, o_d, o_v))
    got = [None] * len(chunks)
    checked = [0, 0]  # rows, mismatching rows

    def step():
        h = C.c_void_p()
        _lib.check(L.tgfx_build_parallel(P(h_ev), E, V, 1, 1, C.byref(h)))
        for i, (s, e) in enumerate(chunks):
            _lib.check(L.tgfx_sample_assemble(
                h, C.c_void_p(h_nodes.data_ptr() + 8 * (s - lo)),
                C.c_void_p(h_times.data_ptr() + 8 * (s - lo)), e - s, k, strat, 9, s, l, E + 1,
                P(o_n), P(o_e), P(o_d), None, P(o_v)))
            if probe is not None:
                ix = probe[i]
                got[i] = (v_n.reshape(-1, l)[ix].copy(), v_e.reshape(-1, l)[ix].copy(),
                          v_d.reshape(-1, l)[ix].copy(), v_v[ix].copy())
        _lib.check(L.tgfx_graph_free(h))

    def verify():
        if probe is None or expect is None:
            return
        for i in range(len(chunks)):
            n_, e_, d_, v_ = got[i]
            want = expect[i]
            bad = ~((n_ == want["node_index"]).all(1) & (e_ == want["edge_index"]).all(1) &
                    (d_ == want["time_delta"]).all(1) & (v_ == want["valid_len"]))
            checked[0] += len(v_)
            checked[1] += int(bad.sum())

    step()  # warm-up
    n_steps = max(1, min(args.steps, args.e2e_steps))
    if ws > 1:
        torch.distributed.barrier()  # inactive ranks wait here too
    # per-step wall times; the median is reported (one step is a full graph allocation,
    # upload, build and 24 synchronous sampling calls -- host-side hiccups of the driver's
    # memory pool or of pinned-memory paging occasionally add 0.3-1 s to a single step)
    times_s = []
    for _ in range(n_steps):
        t0 = time.perf_counter()
        step()
        times_s.append(time.perf_counter() - t0)
        verify()  # outside the timed region
    if checked[1]:
        raise RuntimeError(f"e2e host rows differ from the device path: {checked[1]} of "
                           f"{checked[0]} probe rows")
    dt = statistics.median(times_s)
    from paper_2409_05477_b200 import shard as S
    dt = S.max_over_ranks([dt], device=red)[0]
    q_all = int(S.sum_over_ranks([hi - lo], device=red)[0])  # queries over all ranks
    nr = ws if everyone else 1
    passes = nr if weak else 1
    if not everyone:
        q_all = hi - lo
    return {"value": passes * E / dt, "unit": "edges/s", "ms_per_step": dt * 1e3,
            "steps": n_steps, "ranks": nr, "statistic": "median step",
            "step_ms": [round(x * 1e3, 1) for x in times_s],
            "h2d_bytes_per_step": nr * 32 * E + 16 * q_all,  # every rank uploads the stream
            "d2h_bytes_per_step": (12 * l + 4) * q_all,
            "path": "C ABI host-buffer calls tgfx_build_parallel + tgfx_sample_assemble "
                    "(pinned host memory), wall clock, max over ranks",
            "checked_rows": checked[0], "mismatched_rows": checked[1]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="G", choices=sorted(CONFIGS))
    ap.add_argument("--chunk", type=int, default=3 * 8_000_000)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--plan", default="strong", choices=["weak", "strong"],
                    help="N>1: strong = one pass, queries sharded across ranks (default); "
                         "weak = each rank a full data-parallel pass with its own negatives")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: W >= 3 required by the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
