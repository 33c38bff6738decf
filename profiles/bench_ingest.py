"""CSV ingestion throughput: the reference's load_csv (oracle/_ref, one host thread: it is a
sequential getline loop + stable_sort) vs tgfx_load_csv (file read + upload + device parse)
and tgfx_csv_parse_device (bytes already on the device), on a GDELT-like prefix written as
"src,dst,timestamp" with integer timestamps, rows in file order = time order.

    python profiles/bench_ingest.py [rows]"""
import ctypes as C
import os
import sys
import tempfile
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2409_05477_b200 import _lib  # noqa: E402


def main(rows):
    ev = O.make_random_stream(rows, 16682, 42)
    path = os.path.join(tempfile.mkdtemp(), "g.csv")
    body = np.char.add(np.char.add(np.char.add(np.char.add(ev["src"].astype(str), ","),
                                               ev["dst"].astype(str)), ","),
                       ev["timestamp"].astype(np.int64).astype(str))
    with open(path, "w") as f:
        f.write("src,dst,timestamp\n")
        f.write("\n".join(body.tolist()))
        f.write("\n")
    nbytes = os.path.getsize(path)
    t0 = time.perf_counter()
    ref_ev, _, _ = O.ref_load_csv(path)
    t_ref = time.perf_counter() - t0
    L = _lib.lib()
    h = C.c_void_p()
    _lib.check(L.tgfx_load_csv(path.encode(), 0, C.byref(h)))  # warm-up
    L.tgfx_csv_free(h)
    t0 = time.perf_counter()
    _lib.check(L.tgfx_load_csv(path.encode(), 0, C.byref(h)))
    t_file = time.perf_counter() - t0
    n = C.c_int64()
    _lib.check(L.tgfx_csv_info(h, C.byref(n), None, None))
    got = np.zeros(n.value, dtype=O.EVENT_DTYPE)
    _lib.check(L.tgfx_csv_export(h, got.ctypes.data_as(C.c_void_p), None))
    L.tgfx_csv_free(h)
    assert got.tobytes() == ref_ev.tobytes()
    raw = np.fromfile(path, dtype=np.uint8)
    d = torch.tensor(raw, device="cuda")
    ts = []
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.check(L.tgfx_csv_parse_device(C.c_void_p(d.data_ptr()), nbytes, 0, None, C.byref(h)))
        ts.append(time.perf_counter() - t0)
        L.tgfx_csv_free(h)
    t_dev = min(ts[1:])
    print(f"load_csv {rows:,} rows, {nbytes / 1e6:.1f} MB: reference {t_ref:.2f} s "
          f"({rows / t_ref / 1e6:.2f} M rows/s); tgfx_load_csv (read+upload+parse) {t_file:.3f} s "
          f"({rows / t_file / 1e6:.1f} M rows/s); device parse of resident bytes {t_dev * 1e3:.1f} ms "
          f"({rows / t_dev / 1e6:.0f} M rows/s, {nbytes / t_dev / 1e9:.1f} GB/s); bit-exact: yes")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000)
