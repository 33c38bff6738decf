"""CPU: the C-ABI library builds for sm_100a, loads, and exports every symbol include/tgfx.h
declares (no compute calls: there is no GPU here).  Also checks the product never links the
oracle."""
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "tgfx.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(tgfx_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def built():
    from paper_2409_05477_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        _lib.build_library()
    return _lib


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("tgfx_build_sequential", "tgfx_build_parallel", "tgfx_sample_batch",
              "tgfx_sample_assemble", "tgfx_assemble", "tgfx_build_mask", "tgfx_graph_export",
              "tgfx_make_random_stream", "tgfx_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(built):
    L = built.lib()
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    # the ctypes signature table covers the whole header
    assert sorted(built.SIGNATURES) == declared_symbols()


def test_library_is_sm100a_only(built):
    out = subprocess.run(["cuobjdump", "--list-elf", built.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out), out


def test_no_oracle_in_product(built):
    out = subprocess.run(["ldd", built.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in out and "tgf_ref" not in out
    pkg = os.path.join(ROOT, "paper_2409_05477_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f


def test_abi_version_and_error_plumbing(built):
    L = built.lib()
    assert L.tgfx_abi_version() == 2
    # num_threads validation happens before any device work (tcsr.cpp:108)
    import ctypes as C
    h = C.c_void_p()
    rc = L.tgfx_build_parallel(None, 0, 3, 1, 0, C.byref(h))
    assert rc == built.TGFX_EVALIDATION
    assert L.tgfx_last_error().decode() == "num_threads must be at least 1"
