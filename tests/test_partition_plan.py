"""CPU checks of the partitioned build's ownership plan (paper_2409_05477_b200/partition.py):
rank d owns global entry positions [d*m/N, (d+1)*m/N); nodes whose slice a cut falls inside
are split by position; per-warp split-node entries are apportioned to ranks by overlap."""
import numpy as np
import torch

from paper_2409_05477_b200 import partition as PT


def _brute(deg, world):
    indptr = np.concatenate([[0], np.cumsum(deg)])
    m = int(indptr[-1])
    P = [m * d // world for d in range(world + 1)]
    owner_pos = np.zeros(m, np.int64)
    for d in range(world):
        owner_pos[P[d]:P[d + 1]] = d
    node_of = np.repeat(np.arange(len(deg)), deg)
    split = sorted({int(node_of[p]) for p in P[1:world]
                    if 0 < p < m and indptr[node_of[p]] < p})
    return P, indptr, owner_pos, node_of, split


def test_plan_entry_ranges_matches_brute_force():
    rng = np.random.default_rng(3)
    for world in (1, 2, 3, 5, 8):
        for trial in range(20):
            V = int(rng.integers(1, 60))
            w = np.minimum(rng.zipf(1.3, size=V), 300).astype(np.int64)
            deg = np.where(rng.random(V) < 0.2, 0, w)  # empty slices too
            if deg.sum() == 0:
                deg[0] = 5
            P, bounds, split, indptr = PT.plan_entry_ranges(torch.tensor(deg), world)
            bP, bind, owner_pos, node_of, bsplit = _brute(deg, world)
            assert P.tolist() == bP
            assert indptr.tolist() == bind.tolist()
            assert sorted(split.tolist()) == bsplit
            b = bounds.tolist()
            assert b[0] == 0 and b[-1] == V and all(x <= y for x, y in zip(b, b[1:]))
            # every entry of a non-split node goes to its node range's rank, and that rank is
            # the owner of the entry's global position
            for p in range(int(indptr[-1])):
                u = int(node_of[p])
                if u in bsplit:
                    continue
                d = max(k for k in range(world) if b[k] <= u)
                assert d == owner_pos[p], (world, trial, p)


def test_split_counts_per_rank_overlap():
    rng = np.random.default_rng(4)
    world, nw = 4, 6
    scounts = torch.tensor(rng.integers(0, 50, size=(nw, 7)), dtype=torch.int64)
    gp = torch.tensor(rng.integers(0, 400, size=7), dtype=torch.int64)
    P = torch.tensor([0, 150, 300, 450, 2000], dtype=torch.int64)
    occ, per_rank = PT.split_counts_per_rank(scounts, gp, P, world)
    for w in range(nw):
        for d in range(world):
            want = 0
            for i in range(7):
                s0 = int(gp[i]) + int(scounts[:w, i].sum())
                for p in range(s0, s0 + int(scounts[w, i])):
                    want += int(P[d]) <= p < int(P[d + 1])
            assert int(per_rank[w, d]) == want
    assert torch.equal(occ[0], torch.zeros(7, dtype=torch.int64))
