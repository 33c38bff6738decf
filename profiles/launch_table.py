"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel:
   python profiles/launch_table.py launches.csv"""
import collections
import csv
import sys


def table(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    agg = collections.defaultdict(list)
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    for r in rows[hi + 1:]:
        if len(r) <= vi or (mi is not None and r[mi] != "gpu__time_duration.sum"):
            continue
        agg[r[ki].split("(")[0][-40:]].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6))
    return agg


if __name__ == "__main__":
    agg = table(sys.argv[1])
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':40s} {'n':>5s} {'total ms':>10s} {'mean ms':>9s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{k:40s} {len(v):5d} {sum(v):10.3f} {sum(v) / len(v):9.4f} {100 * sum(v) / tot:5.1f}%")
