"""load_csv on the device (proj/src/event_stream.cpp:85-154) vs the
reference's own load_csv (oracle/_ref) and std::from_chars (the reference's number parser,
oracle/fromchars.cpp): events, ordering, ids, features bit-exact; errors with the
reference's exception types and texts."""
import os
import random
import struct

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _device_parse(strings, kind):
    from paper_2409_05477_b200 import _lib
    blob = b"".join(strings)
    off = np.zeros(len(strings) + 1, np.int64)
    off[1:] = np.cumsum([len(s) for s in strings])
    d_buf = torch.tensor(np.frombuffer(blob, np.uint8).copy(), device="cuda")
    d_off = torch.tensor(off, device="cuda")
    n = len(strings)
    ii = torch.zeros(n, dtype=torch.int64, device="cuda")
    dd = torch.zeros(n, dtype=torch.float64, device="cuda")
    st = torch.zeros(n, dtype=torch.int32, device="cuda")
    import ctypes as C
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    _lib.check(_lib.lib().tgfx_parse_numbers_device(P(d_buf), P(d_off), n, 0 if kind == "int" else 1,
                                                    P(ii), P(dd), P(st), None))
    return st.cpu().numpy(), (ii if kind == "int" else dd).cpu().numpy()


def _random_reals(rng, n):
    out, tags = [], []
    for _ in range(n):
        k = rng.randrange(12)
        tags.append(k)
        if k == 0:  # repr of a random double (up to 17 significant digits)
            x = struct.unpack("<d", struct.pack("<Q", rng.getrandbits(64)))[0]
            out.append(repr(x).encode())
        elif k == 1:  # uniform in [0, 1e9) with a few digits
            out.append(("%.*f" % (rng.randrange(0, 8), rng.uniform(0, 1e9))).encode())
        elif k == 2:  # scientific with wide exponents
            out.append(("%se%d" % (rng.choice(["1", "9.99", "2.2250738585072014", "4.9", "1.7976931348623157"]),
                                   rng.randrange(-340, 320))).encode())
        elif k == 3:  # long digit strings (> 19 significant digits)
            out.append((str(rng.randrange(1, 10**rng.randrange(18, 40))) + "." +
                        str(rng.randrange(0, 10**rng.randrange(1, 20)))).encode())
        elif k == 4:  # specials and malformed
            out.append(rng.choice([b"inf", b"-Infinity", b"INF", b"nan", b"-NaN", b"nan(123)",
                                   b"nan(", b"infx", b"1e", b"1e+", b"+1", b"-", b".", b"e5",
                                   b"0x10", b"1.", b".5", b"-0", b"00012", b"1_", b"", b"- 1",
                                   b"1e-999", b"2.4e-324", b"2.5e-324", b"1.7976931348623159e308",
                                   b"1e309", b"4.9406564584124654e-324", b"1.5E+3", b"  7  "]))
        elif k == 5:  # integers as reals
            out.append(str(rng.randrange(-10**18, 10**18)).encode())
        elif k == 6:  # halfway-ish: exact decimal of a double midpoint (many digits)
            m = rng.getrandbits(53) | 1
            e = rng.randrange(-60, 10)
            from decimal import Decimal, getcontext
            getcontext().prec = 200
            out.append(str(Decimal(m) * (Decimal(2) ** e) + (Decimal(2) ** (e - 1))).encode())
        elif k == 7:  # timestamps with ties / small decimals
            out.append(("%d.%d" % (rng.randrange(0, 100000), rng.randrange(0, 10))).encode())
        elif k == 8:  # denormal / tiny
            out.append(("%.17g" % (rng.uniform(0, 1) * 1e-310)).encode())
        elif k == 9:
            out.append(("%.*e" % (rng.randrange(0, 25), rng.uniform(-1e6, 1e6))).encode())
        elif k == 10:
            out.append(("0." + "0" * rng.randrange(0, 30) + str(rng.randrange(1, 10**9))).encode())
        else:
            out.append(str(rng.randrange(0, 2**53)).encode() + b"e" + str(rng.randrange(-30, 40)).encode())
    return out, tags


def test_real_parser_matches_from_chars(oracle_mod):
    rng = random.Random(7)
    strings, tags = _random_reals(rng, 60_000)
    st, got = _device_parse(strings, "real")
    ok, want = oracle_mod.from_chars([s.strip(b" \t\r") for s in strings], "real")
    unsupported = 0
    for i, s in enumerate(strings):
        if st[i] == 2:  # only > 19 significant digits may need the big-integer path
            digits = sum(c in b"0123456789" for c in s.split(b"e")[0].split(b"E")[0].lstrip(b"-0."))
            assert digits > 19, s
            unsupported += tags[i] != 6  # category 6 builds exact midpoints on purpose
            continue
        assert (st[i] == 0) == bool(ok[i]), (s, st[i], ok[i])
        if ok[i]:
            a, b = got[i], want[i]
            assert (a == b and np.signbit(a) == np.signbit(b)) or (np.isnan(a) and np.isnan(b)), (s, a, b)
    assert unsupported < 0.002 * len(strings)


def test_int_parser_matches_from_chars(oracle_mod):
    rng = random.Random(3)
    strings = [rng.choice([str(rng.randrange(-2**63, 2**63)), str(rng.randrange(0, 10**25)),
                           "-" + str(rng.randrange(0, 10**20)), "+5", "007", "-0", "1.5", "",
                           "9223372036854775807", "9223372036854775808", "-9223372036854775808",
                           "-9223372036854775809", " 12 ", "1e3", "--1"]).encode()
               for _ in range(20_000)]
    st, got = _device_parse(strings, "int")
    ok, want = oracle_mod.from_chars([s.strip(b" \t\r") for s in strings], "int")
    assert np.array_equal(st == 0, ok)
    assert np.array_equal(got[ok], want[ok])


def _write(path, header, rows, crlf=False, trailing_newline=True, blank_every=0):
    nl = "\r\n" if crlf else "\n"
    lines = [header] + rows
    out = []
    for i, r in enumerate(lines):
        out.append(r)
        if blank_every and i % blank_every == blank_every - 1:
            out.append("   ")
    txt = nl.join(out) + (nl if trailing_newline else "")
    with open(path, "w", newline="") as f:
        f.write(txt)


def _check_same(T, oracle_mod, path, has_features):
    s, feats = T.load_csv(path, has_features)
    ev, v, wf = oracle_mod.ref_load_csv(path, has_features)
    assert s.num_nodes == v
    assert s.events.tobytes() == ev.tobytes()
    assert feats.shape == wf.shape
    assert feats.tobytes() == wf.tobytes()
    return s


def test_load_csv_matches_reference(tmp_path, oracle_mod):
    from paper_2409_05477_b200 import tgformer as T
    rng = np.random.default_rng(11)
    # (a) a Zipf stream written in shuffled order, integer timestamps with many ties
    ev = oracle_mod.make_random_stream(60_000, 700, 5)
    perm = rng.permutation(len(ev))
    rows = ["%d,%d,%d" % (ev["src"][i], ev["dst"][i], ev["timestamp"][i]) for i in perm]
    _write(tmp_path / "a.csv", "src,dst,timestamp", rows)
    s = _check_same(T, oracle_mod, str(tmp_path / "a.csv"), False)
    g = T.build_sequential(s, True)  # the parsed stream feeds the builder directly
    assert g.num_entries() == 2 * len(ev)
    # (b) decimal timestamps, repr-printed features, CRLF, blank lines, spaces, no final newline
    n = 20_000
    t = np.round(rng.uniform(0, 5000, n), rng.integers(0, 4))
    f = rng.normal(size=(n, 3))
    rows = [" %d , %d,%r,%r,%r,%r" % (rng.integers(0, 90), rng.integers(0, 90), float(t[i]),
                                      float(f[i, 0]), float(f[i, 1]), float(f[i, 2]))
            for i in range(n)]
    _write(tmp_path / "b.csv", "src,dst,timestamp,f1,f2,f3", rows, crlf=True,
           trailing_newline=False, blank_every=97)
    _check_same(T, oracle_mod, str(tmp_path / "b.csv"), True)
    _check_same(T, oracle_mod, str(tmp_path / "b.csv"), False)  # extra columns ignored
    # (c) exponent / special formats, -0.0 and inf timestamps
    rows = ["1,2,1e3", "2,3,-0", "3,4,1000.0", "4,5,inf", "5,6,1.5e2", "6,7,150", "0,0,0.0"]
    _write(tmp_path / "c.csv", "src,dst,timestamp", rows)
    _check_same(T, oracle_mod, str(tmp_path / "c.csv"), False)
    # (d) header only
    _write(tmp_path / "d.csv", "src,dst,timestamp", [])
    s = _check_same(T, oracle_mod, str(tmp_path / "d.csv"), False)
    assert s.num_nodes == 0 and len(s.events) == 0


@pytest.mark.parametrize("header,rows,has_features", [
    ("src,dst", ["1,2"], False),                       # header needs 3 fields
    ("src,dst,timestamp", ["1,2,3", "4,5"], False),    # field count
    ("src,dst,timestamp", ["1,2,3", "x,5,6"], False),  # bad src
    ("src,dst,timestamp", ["1,2,3", "4, 5.5 ,6"], False),  # bad dst
    ("src,dst,timestamp", ["1,2,3", "4,5,1e"], False),  # bad timestamp (not consumed)
    ("src,dst,timestamp", ["1,2,3", "4,5,1e999"], False),  # out of range
    ("src,dst,timestamp", ["1,2,3", "-4,5,6"], False),  # negative node id (ValidationError)
    ("src,dst,timestamp", ["1,2,3", "4,5,-6"], False),  # negative timestamp
    ("src,dst,timestamp,f", ["1,2,3,0.5", "4,5,6,zz"], True),  # bad feature
    ("src,dst,timestamp", ["1,2,3", "4,5,x", "-1,2,3"], False),  # first failing line wins
])
def test_load_csv_errors_match_reference(tmp_path, oracle_mod, header, rows, has_features):
    from paper_2409_05477_b200 import tgformer as T
    p = str(tmp_path / "e.csv")
    _write(p, header, rows)
    with pytest.raises(oracle_mod.OracleError) as want:
        oracle_mod.ref_load_csv(p, has_features)
    kind = {1: T.ValidationError, 6: T.ParseError}[want.value.code]
    with pytest.raises(kind) as got:
        T.load_csv(p, has_features)
    assert str(got.value) == str(want.value)


def test_load_csv_file_errors(tmp_path, oracle_mod):
    from paper_2409_05477_b200 import tgformer as T
    missing = str(tmp_path / "nope.csv")
    with pytest.raises(T.ValidationError, match="cannot open"):
        T.load_csv(missing)
    empty = tmp_path / "empty.csv"
    empty.write_bytes(b"")
    with pytest.raises(oracle_mod.OracleError) as want:
        oracle_mod.ref_load_csv(str(empty))
    with pytest.raises(T.ParseError) as got:
        T.load_csv(str(empty))
    assert str(got.value) == str(want.value)
