"""Per-kernel table from an ncu --csv launch list (gpu__time_duration / dram bytes metrics):
   python profiles/launch_csv.py <launches.csv> [first_id] [last_id]"""
import csv
import sys


def main(path, lo=0, hi=1 << 30):
    rows = list(csv.reader(open(path)))
    hdr, out = None, {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            out.setdefault((int(d["ID"]), d["Kernel Name"]), {})[d["Metric Name"]] = d["Metric Value"]
    for (i, k), m in sorted(out.items()):
        if lo <= i <= hi:
            t = float(m.get("gpu__time_duration.sum", "0").replace(",", ""))
            rd = float(m.get("dram__bytes_read.sum", "0").replace(",", ""))
            wr = float(m.get("dram__bytes_write.sum", "0").replace(",", ""))
            print(f"{i:4d} {t / 1e3:9.3f} us  rd {rd / 1e9:7.3f} GB  wr {wr / 1e9:7.3f} GB  {k[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], *(int(x) for x in sys.argv[2:4]))
