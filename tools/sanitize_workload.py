"""Small build + sample workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): python tools/sanitize_workload.py under `compute-sanitizer --tool X`.
Results: profiles/r01/compute_sanitizer.txt."""
import sys, numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from oracle import oracle as O
from paper_2409_05477_b200 import tgformer as T
for E, V, rev in ((20000, 300, True), (30000, 5000, False), (5000, 1, True)):
    ev = O.make_random_stream(E, V, 3)
    g = T.build_parallel(T.EventStream(ev, V), rev, 4)
    want = O.build(ev, V, rev)
    assert np.array_equal(g.neighbor_ids, want["nbr"])
    nodes, times = O.make_queries(ev, 0, min(E, 3000), 600, V)
    for strat, k, l in (("recent", 10, 11), ("random", 20, 21), ("random", 40, 21)):
        got = T.sample_assemble(g, nodes, times, k, strat, 9, l, E + 1)
        ref = O.sample_assemble(want, nodes, times, k, strat, 9, l, E + 1)
        assert np.array_equal(got["node_index"].astype(np.int64), ref["node_index"])
# unsorted stream (general path)
ev = O.make_random_stream(20000, 300, 5)[::-1].copy()
g = T.build_parallel(T.EventStream(ev, 300), True, 4)
assert np.array_equal(g.neighbor_ids, O.build(ev, 300, True)["nbr"])
print("sanitize workload ok")
# round 2 paths: large-V onesweep build, uniform k > 256, fused query check, sampler fused with
# assemble_inputs, training queries, 2-hop
import torch  # noqa: E402
from paper_2409_05477_b200 import device as D  # noqa: E402
ev = D.random_stream(40000, 60000, 4)  # V > 45 K: the large-V path
g = D.build(ev, 60000, True)
want = O.build(ev.cpu().numpy().view(O.EVENT_DTYPE), 60000, True)
assert np.array_equal(D.graph_tensors(g)[1].cpu().numpy(), want["nbr"])
ev = D.random_stream(30000, 200, 6)
g = D.build(ev, 200, True)
nodes, times = D.make_queries(ev, 0, 2000, 600, 200)
fb = D.first_bad_word()
D.sample_assemble(g, nodes, times, 10, "recent", 9, 11, 30001, first_bad=fb)
D.query_error(nodes, fb)
D.sample_batch(g, nodes[:300], times[:300], 600, "random", 3)  # k > 256
nt = torch.randn((201, 8), device="cuda")
et = torch.randn((30002, 8), device="cuda")
w = torch.randn(8, dtype=torch.float64, device="cuda")
D.sample_inputs(g, nodes, times, 10, "recent", 0, 11, 30001, nt, et, w, w, True)
D.make_train_queries(ev, 30000, 0, 10, 500, 2, 3, 200, 77)
D.two_hop(g, nodes[:600], times[:600], 5, 5, "recent", 0, 6, 30001)
torch.cuda.synchronize()
print("sanitize workload (round 2 paths) ok")
