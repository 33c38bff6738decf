"""Per-instruction stall summary from an ncu report's source page (SASS):
   python profiles/ncu_source.py <report.ncu-rep> [top_n]"""
import csv
import io
import subprocess
import sys

REASONS = ["stall_long_sb", "stall_short_sb", "stall_barrier", "stall_wait", "stall_lg",
           "stall_mio", "stall_branch_resolving", "stall_math", "stall_membar", "stall_selected",
           "stall_not_selected", "stall_no_inst", "stall_dispatch", "stall_drain", "stall_tex"]


def main(path, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    si, wi = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    idx = {r: h.index(r) for r in REASONS if r in h}
    data, totals = [], {r: 0 for r in idx}
    for r in rows[2:]:
        try:
            w = int(r[wi])
        except (ValueError, IndexError):
            continue
        why = {k: int(r[i] or 0) for k, i in idx.items()}
        for k in why:
            totals[k] += why[k]
        data.append((w, r[0][-5:], r[si].strip(), why))
    tot = sum(d[0] for d in data) or 1
    print("total samples", tot)
    print("by reason:", ", ".join(f"{k[6:]}={100 * v / tot:.1f}%" for k, v in
                                  sorted(totals.items(), key=lambda x: -x[1]) if v))
    for w, a, s, why in sorted(data, key=lambda d: -d[0])[:top]:
        top3 = sorted(why.items(), key=lambda x: -x[1])[:2]
        print(f"{w:7d} {100 * w / tot:5.1f}% {a} {s[:60]:60s} " +
              " ".join(f"{k[6:]}:{v}" for k, v in top3 if v))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
