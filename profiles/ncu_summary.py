"""Summarise an ncu report (raw page) into the metrics we track; usage:
   python profiles/ncu_summary.py <report.ncu-rep> [more metric substrings]"""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.per_cycle_active", "launch__shared_mem_per_block_dynamic",
        "lts__t_sector_hit_rate.pct"]


def summary(path, extra=()):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")]}
        for w in list(WANT) + [c for c in h if any(e in c for e in extra)]:
            if w in h:
                i = h.index(w)
                d[w] = (v[i], units[i])
        res.append(d)
    return res


if __name__ == "__main__":
    for d in summary(sys.argv[1], sys.argv[2:]):
        print("==", d.pop("kernel")[:100])
        for k, (v, u) in d.items():
            print(f"  {k:62s} {v:>22s} {u}")
