"""ctypes binding of libtgfx.so (include/tgfx.h).

The library is the product: every call runs hand-written sm_100a kernels.  There is no
fallback -- if the shared object is missing or no sm_100 device is present, calls fail
loudly (TgfxError / OSError).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
# TGFX_LIB: another build of the same library (A/B timing of two builds in one session)
LIB_PATH = os.environ.get("TGFX_LIB") or os.path.join(HERE, "lib", "libtgfx.so")

TGFX_OK, TGFX_EVALIDATION, TGFX_EFORMAT, TGFX_ECUDA, TGFX_ENOMEM, TGFX_EUNSUPPORTED = range(6)
TGFX_RECENT, TGFX_RANDOM = 0, 1
TGFX_TRUSTED, TGFX_INDEX64 = 1, 2


class TgfxError(RuntimeError):
    """Base of all errors raised by the library (mirrors std::runtime_error)."""

    code = TGFX_ECUDA


class ValidationError(TgfxError):
    """proj/include/tgformer/common.hpp:15-17"""

    code = TGFX_EVALIDATION


class FormatError(TgfxError):
    """proj/include/tgformer/common.hpp:25-27"""

    code = TGFX_EFORMAT


class ParseError(TgfxError):
    """proj/include/tgformer/common.hpp:20-22"""

    code = 6


class CudaError(TgfxError):
    code = TGFX_ECUDA


class OutOfMemory(TgfxError):
    code = TGFX_ENOMEM


class Unsupported(TgfxError):
    code = TGFX_EUNSUPPORTED


_ERRORS = {1: ValidationError, 2: FormatError, 3: CudaError, 4: OutOfMemory, 5: Unsupported,
           6: ParseError}

_P = C.c_void_p
_I64 = C.c_int64
_U64 = C.c_uint64
_I = C.c_int
_U = C.c_uint

# name -> argtypes (all return int status unless listed in _RESTYPE)
SIGNATURES = {
    "tgfx_last_error": [],
    "tgfx_abi_version": [],
    "tgfx_launch_count": [],
    "tgfx_device_bytes": [],
    "tgfx_build_sequential": [_P, _I64, _I64, _I, C.POINTER(_P)],
    "tgfx_build_parallel": [_P, _I64, _I64, _I, _I, C.POINTER(_P)],
    "tgfx_build_device": [_P, _I64, _I64, _I, _P, _U, C.POINTER(_P)],
    "tgfx_rebuild_device": [_P, _P, _P, _U],
    "tgfx_graph_from_host": [_I64, _I64, _I, _I64, _P, _P, _P, _P, C.POINTER(_P)],
    "tgfx_graph_from_device": [_I64, _I64, _I, _I64, _P, _P, _P, _P, _P, _U, C.POINTER(_P)],
    "tgfx_build_range_device": [_P, _I64, _I64, _I64, _I64, _P, _U, C.POINTER(_P)],
    "tgfx_degree_hist_device": [_P, _I64, _I64, _I, _P, _P],
    "tgfx_partition_warps": [_I64],
    "tgfx_partition_count_device": [_P, _I64, _I, _P, _I, _I64, _P, _P, _P, _P],
    "tgfx_partition_scatter_device": [_P, _I64, _I, _P, _I, _I64, _P, _P, _P, _P, _P],
    "tgfx_graph_info": [_P, C.POINTER(_I64), C.POINTER(_I64), C.POINTER(_I64), C.POINTER(_I)],
    "tgfx_graph_export": [_P, _P, _P, _P, _P],
    "tgfx_graph_device_arrays": [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P),
                                 C.POINTER(_P)],
    "tgfx_graph_validate": [_P],
    "tgfx_graph_free": [_P],
    "tgfx_graph_build_path": [_P],
    "tgfx_sample_batch": [_P, _P, _P, _I64, _I64, _I, _U64, _U64, _P, _P, _P, _P],
    "tgfx_sample_batch_records": [_P, _P, _P, _I64, _I64, _I, _U64, _U64, _P, _P],
    "tgfx_host_alloc": [C.c_size_t, C.POINTER(_P)],
    "tgfx_host_free": [_P],
    "tgfx_sample_batch_device": [_P, _P, _P, _I64, _I64, _I, _U64, _U64, _P, _P, _P, _P, _P, _U],
    "tgfx_sample_assemble": [_P, _P, _P, _I64, _I64, _I, _U64, _U64, _I64, _I64, _P, _P, _P, _P,
                             _P],
    "tgfx_sample_sequence_batch": [_P, _P, _P, _I64, _I64, _I, _U64, _U64, _I64, _I64, _P, _P,
                                   _P, _P, _P],
    "tgfx_sample_assemble_checked_device": [_P, _P, _P, _I64, _I64, _I, _U64, _U64, _I64, _I64,
                                            _P, _P, _P, _P, _P, _P, _P, _U],
    "tgfx_query_error": [_P, _U64, _P, _P],
    "tgfx_make_train_queries_device": [_P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _U64, _P,
                                       _P, _P],
    "tgfx_mix_streams": [_U64, _U64, _U64],
    "tgfx_sample_inputs_device": [_P, _P, _P, _I64, _I64, _I, _U64, _U64, _I64, _I64, _P, _I64,
                                  _P, _I64, _I, _P, _P, _I64, _I64, _I64, _I, _P, _I, _P, _P,
                                  _U],
    "tgfx_sample_assemble_device": [_P, _P, _P, _I64, _I64, _I, _U64, _U64, _I64, _I64, _P, _P,
                                    _P, _P, _P, _P, _U],
    "tgfx_sample_assemble_batched_device": [_P, _P, _P, _I64, _I64, _I64, _I, _P, _I64, _I64,
                                            _P, _P, _P, _P, _P, _P, _U],
    "tgfx_assemble_inputs_device": [_I64, _I64, _P, _P, _P, _P, _I, _I, _P, _I64, _P, _I64, _I,
                                    _P, _P, _I64, _I64, _I64, _I, _P, _I, _P, _U],
    "tgfx_load_csv": [C.c_char_p, _I, C.POINTER(_P)],
    "tgfx_csv_parse_device": [_P, _I64, _I, _P, C.POINTER(_P)],
    "tgfx_csv_info": [_P, C.POINTER(_I64), C.POINTER(_I64), C.POINTER(_I64)],
    "tgfx_csv_device_arrays": [_P, C.POINTER(_P), C.POINTER(_P)],
    "tgfx_csv_export": [_P, _P, _P],
    "tgfx_csv_free": [_P],
    "tgfx_parse_numbers_device": [_P, _P, _I64, _I, _P, _P, _P, _P],
    "tgfx_sample_two_hop_device": [_P, _P, _P, _I64, _I64, _I64, _I, _U64, _U64, _I64, _I64, _P,
                                   _P, _P, _P, _P, _P, _P, _P, _P, _U],
    "tgfx_sample_two_hop": [_P, _P, _P, _I64, _I64, _I64, _I, _U64, _U64, _I64, _I64, _P, _P, _P,
                            _P, _P, _P, _P, _P],
    "tgfx_assemble": [_I64, _I64, _P, _P, _P, _P, _P, _P, _I64, _I64, _P, _P, _P, _P, _P],
    "tgfx_assemble_records": [_I64, _I64, _P, _P, _P, _P, _I64, _I64, _P, _P, _P, _P, _P],
    "tgfx_build_mask": [_I64, _I64, _P, _P, _I, _P],
    "tgfx_make_random_stream": [_I64, _I64, _U64, C.c_double, _P],
    "tgfx_make_random_stream_device": [_I64, _I64, _U64, C.c_double, _P, _P],
    "tgfx_make_queries_device": [_P, _I64, _I64, _I64, _I64, _U64, _P, _P, _P],
}
_RESTYPE = {"tgfx_last_error": C.c_char_p, "tgfx_launch_count": C.c_uint64,
            "tgfx_device_bytes": C.c_int64, "tgfx_partition_warps": C.c_int64,
            "tgfx_mix_streams": C.c_uint64}

_lib = None


def build_library(verbose=False):
    """Compile libtgfx.so for sm_100a (nvcc; no GPU needed)."""
    cmd = ["make", "-C", os.path.join(HERE, "csrc")]
    if not verbose:
        cmd.insert(1, "-s")
    subprocess.run(cmd, check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OSError(f"{LIB_PATH} is not built; run paper_2409_05477_b200._lib.build_library()"
                          " (or __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = _RESTYPE.get(name, C.c_int)
        _lib = L
    return _lib


def check(rc):
    if rc != TGFX_OK:
        msg = lib().tgfx_last_error().decode()
        raise _ERRORS.get(rc, TgfxError)(msg)


def launch_count():
    return int(lib().tgfx_launch_count())
