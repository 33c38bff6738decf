"""Build-only timing on the GDELT shape (A/B of TGFX_SCATTER_VARIANT etc., one process per
setting): median device time of a full reverse=1 rebuild from the resident stream, plus a
positional checksum of the columns so settings can be compared bit for bit."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_05477_b200 import device as D  # noqa: E402


def main():
    E = int(os.environ.get("E", 191_290_882))
    V = int(os.environ.get("V", 16682))
    reps = int(os.environ.get("REPS", 10))
    ev = D.random_stream(E, V, 42)
    g = D.build(ev, V, True)
    st = torch.cuda.current_stream()
    ts = []
    for i in range(reps + 3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        D.rebuild(g, ev, trusted=True)
        b.record(st)
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    ip, nb, ed, tt = D.graph_tensors(g)
    w = torch.arange(1, nb.numel() + 1, device="cuda", dtype=torch.int64)
    ck = [int((x.view(torch.int64) * w).sum()) for x in (nb, ed, tt)] + [int(ip.sum())]
    print(json.dumps({"variant": os.environ.get("TGFX_SCATTER_VARIANT", "10"), "E": E, "V": V,
                      "build_ms_median": statistics.median(ts), "build_ms": ts,
                      "checksum": ck}), flush=True)


if __name__ == "__main__":
    main()
