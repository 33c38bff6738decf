"""B200-native T-CSR builder + temporal sampler + sequence assembler (TF-TGN hot path).

The compute lives in libtgfx.so (hand-written sm_100a CUDA behind the C ABI in
include/tgfx.h).  `tgformer` mirrors the reference's C++ API names for Python callers;
`device` exposes the asynchronous device-pointer calls used by bench.py.
"""
from ._lib import (CudaError, FormatError, OutOfMemory, ParseError, TgfxError,  # noqa: F401
                   Unsupported, ValidationError, build_library, launch_count, lib)
from . import tgformer  # noqa: F401

__version__ = "0.1.0"
