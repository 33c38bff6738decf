"""Step pipelining experiment (GDELT shape): K steps of [rebuild + recent-10 sampling of all
queries], sequential on one stream vs pipelined on two streams (the build of step s+1 into a
second T-CSR overlaps the sampling of step s).  Prints ms per step for both."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_05477_b200 import device as D, shard as S  # noqa: E402


def main():
    E, V, B, K = 191_290_882, 16682, 600, int(os.environ.get("K", 6))
    Q = 3 * E
    ev = D.random_stream(E, V, 42)
    nodes = torch.empty(Q, dtype=torch.int64, device="cuda")
    times = torch.empty(Q, dtype=torch.float64, device="cuda")
    step_ev = (8_000_000 // B) * B
    for e0 in range(0, E, step_ev):
        e1 = min(E, e0 + step_ev)
        D.make_queries(ev, e0, e1, B, V, 7, nodes=nodes[3 * e0:3 * e1], times=times[3 * e0:3 * e1])
    chunks = S.chunks(0, Q, 24_000_000)
    out = D.alloc_rows(24_000_000, 11)
    gs = [D.build(ev, V, True), D.build(ev, V, True)]
    sa, sb = torch.cuda.Stream(priority=-1), torch.cuda.Stream()
    fb = D.first_bad_word()

    def sample(g, st):
        for s, e in chunks:
            sub = {kk: vv[: e - s] for kk, vv in out.items()}
            D.sample_assemble(g, nodes[s:e], times[s:e], 10, "recent", 9, 11, E + 1, out=sub,
                              stream_base=s, first_bad=fb, stream=st)

    def sequential():
        st = torch.cuda.current_stream()
        for _ in range(K):
            D.rebuild(gs[0], ev, trusted=True, stream=st)
            sample(gs[0], st)

    def pipelined():
        built = [torch.cuda.Event(), torch.cuda.Event()]
        used = [torch.cuda.Event(), torch.cuda.Event()]
        D.rebuild(gs[0], ev, trusted=True, stream=sa)
        built[0].record(sa)
        for s in range(K):
            cur, nxt = s % 2, (s + 1) % 2
            sb.wait_event(built[cur])
            sample(gs[cur], sb)
            used[cur].record(sb)
            if s + 1 < K:
                if s >= 1:
                    sa.wait_event(used[nxt])
                D.rebuild(gs[nxt], ev, trusted=True, stream=sa)
                built[nxt].record(sa)
        torch.cuda.current_stream().wait_stream(sb)
        torch.cuda.current_stream().wait_stream(sa)

    res = {}
    for name, fn in (("sequential", sequential), ("pipelined", pipelined), ("sequential2", sequential),
                     ("pipelined2", pipelined)):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        res[name] = a.elapsed_time(b) / K
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
