"""ctypes binding of synth/synth.c: ``weight_bits`` in C, multi-threaded.

Same bits as :func:`synth.weight_bits` (pinned by tests/test_synth_cpu.py);
used to fill full-size trainer buffers on the host (tests' streamed parity,
bench.py's CPU legs).  No arithmetic of the method lives here.
"""
from __future__ import annotations

import concurrent.futures as cf
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "synth.c")
_LIB = os.path.join(_HERE, "libsynth.so")
_lib = None
_pool = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O3", "-std=gnu11", "-fPIC", "-shared", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.synth_fill.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
        _lib.synth_fill.restype = None
    return _lib


def threads() -> int:
    return max(1, os.cpu_count() or 1)


def _executor():
    global _pool
    if _pool is None:
        _pool = cf.ThreadPoolExecutor(threads())
    return _pool


def fill(out: np.ndarray, seed: int, param: int, is_norm: bool, dtype: str, r0: int, r1: int, c0: int, c1: int,
         parallel: bool = True) -> None:
    """Write rows [r0, r1) x cols [c0, c1) of source param `param` as bit patterns
    (uint32 for "f32", uint16 for "bf16"), row-major, into the contiguous buffer
    ``out`` (any dtype; at least rows*cols*esize bytes)."""
    if dtype not in ("f32", "bf16"):
        raise ValueError(f"unsupported source dtype {dtype!r}")
    es = 4 if dtype == "f32" else 2
    nr, nc = r1 - r0, c1 - c0
    if nr <= 0 or nc <= 0:
        return
    assert out.flags.c_contiguous and out.nbytes >= nr * nc * es
    base = out.ctypes.data
    L = lib()
    f32 = int(dtype == "f32")
    n = threads() if parallel else 1
    rows_per = max(1, -(-nr // (4 * n))) if nr * nc >= (1 << 20) else nr
    if rows_per >= nr:
        L.synth_fill(seed, param, int(is_norm), f32, r0, r1, c0, c1, base)
        return
    futs = []
    for a in range(r0, r1, rows_per):
        b = min(r1, a + rows_per)
        futs.append(_executor().submit(L.synth_fill, seed, param, int(is_norm), f32, a, b, c0, c1,
                                       base + (a - r0) * nc * es))
    for f in futs:
        f.result()


def weight_bits(seed: int, param: int, is_norm: bool, dtype: str, r0: int, r1: int, c0: int, c1: int) -> np.ndarray:
    """[r1-r0, c1-c0] array of bit patterns (the C twin of synth.weight_bits on a rectangle)."""
    out = np.empty((max(0, r1 - r0), max(0, c1 - c0)), np.uint32 if dtype == "f32" else np.uint16)
    fill(out, seed, param, is_norm, dtype, r0, r1, c0, c1)
    return out
