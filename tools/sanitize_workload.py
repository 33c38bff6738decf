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
