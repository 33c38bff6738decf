"""Device allocator under the host-buffer calls.

Buffers of >= 256 MB are recycled by exact size through a cache keyed by pointer
(csrc/api.cu dmalloc/dfree).  Every such buffer must be released through dfree: a direct
cudaFreeAsync leaves a stale registry entry, and a later small buffer handed the same address
by the pool would then be cached as a multi-GB block and handed out over live memory.  This
test alternates >= 256 MB host-buffer builds and sampling calls (upload staging, graph columns,
gather records, per-lane row buffers) with small builds and samples, and checks every result
bit for bit against the oracle."""
import numpy as np
import pytest

from test_gpu_sample import check_rows

pytestmark = pytest.mark.gpu


def test_big_and_small_allocations_alternate(oracle_mod):
    from paper_2409_05477_b200 import tgformer as T
    cases = [(9_000_000, 16682, 5), (1000, 40, 6), (9_500_000, 3000, 7), (2000, 7, 8)]
    for it in range(2):
        for E, V, seed in cases:
            ev = oracle_mod.make_random_stream(E, V, seed + it)
            want = oracle_mod.build(ev, V, True)
            g = T.build_parallel(T.EventStream(ev, V), True, 4)     # host-buffer build
            assert np.array_equal(g.indptr, want["indptr"]), (E, it)
            assert np.array_equal(g.neighbor_ids, want["nbr"]), (E, it)
            assert np.array_equal(g.edge_ids, want["eid"]), (E, it)
            assert np.array_equal(g.timestamps, want["ts"]), (E, it)
            e1 = min(E, 2_000_000)
            nodes, times = oracle_mod.make_queries(ev, 0, e1, 600, V)
            # l = 21: each 4 M-query lane buffer is >= 256 MB (big-block path)
            got = T.sample_assemble(g, nodes, times, 20, "random", 9 + it, 21, E + 1)
            exp = oracle_mod.sample_assemble(want, nodes, times, 20, "random", 9 + it, 21, E + 1)
            check_rows(got, exp, (E, it, "random"))
            got = T.sample_assemble(g, nodes[:5000], times[:5000], 10, "recent", 0, 11, E + 1)
            exp = oracle_mod.sample_assemble(want, nodes[:5000], times[:5000], 10, "recent", 0,
                                             11, E + 1)
            check_rows(got, exp, (E, it, "recent"))
            del g
