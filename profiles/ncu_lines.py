"""Per-CUDA-source-line stall samples of one kernel in an ncu report.

   python profiles/ncu_lines.py <report.ncu-rep> <lib.so> <mangled-kernel-substring> [top_n]

Maps the SASS-level samples of `ncu --page source` to source lines with `nvdisasm -g` of
the same binary (needs -lineinfo).  The .so must be the one that was profiled.
"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile


def sass_lines(lib, fun_sub):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
    for cub in glob.glob(os.path.join(d, "*.cubin")):
        txt = subprocess.run(["nvdisasm", "-g", cub], capture_output=True, text=True).stdout
        m = None
        cur_line, in_fun, mapping = None, False, {}
        for ln in txt.splitlines():
            if ln.lstrip().startswith(".section") and ".text." in ln:
                in_fun = fun_sub in ln
            h = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if h:
                cur_line = (os.path.basename(h.group(1)), int(h.group(2)))
            a = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+([A-Z@].*?);", ln)
            if in_fun and a and cur_line:
                mapping[int(a.group(1), 16)] = (cur_line, a.group(2).strip())
        if mapping:
            return mapping
    return {}


def main(rep, lib, fun_sub, top=30):
    mapping = sass_lines(lib, fun_sub)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    col = os.environ.get("NCU_COLUMN", "Warp Stall Sampling (All Samples)")
    wi = h.index(col)
    addrs = []
    for r in rows[2:]:
        try:
            addrs.append((int(r[0], 16), int(r[wi] or 0)))
        except ValueError:
            pass
    base = min(a for a, _ in addrs)
    per = collections.Counter()
    for a, w in addrs:
        key = mapping.get(a - base, (("?", 0), ""))[0]
        per[key] += w
    tot = sum(per.values()) or 1
    src = {}
    for (f, ln), w in per.most_common(top):
        print(f"{w:8d} {100 * w / tot:5.1f}%  {f}:{ln}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 30)
