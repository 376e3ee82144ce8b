"""Seeded synthetic inputs shared by the oracle side and the CUDA side of the tests.

This module holds NO arithmetic of the method (no re-layout, no cast, no
quantisation).  It only defines

* the model shapes and layout configurations the paper's workloads use
  (``configs``; Llama-3.1 shapes, §8 P:580 names the models), and
* a counter-based generator that turns (seed, param id, global row, global col)
  into a trainer weight *bit pattern* using integer operations only, so the
  numpy version here and the CUDA version in the product's K0 kernel
  (``paper_2505_24034_b200/csrc/init.cu``) produce identical bits by
  construction.

Distribution: linear / embedding weights have a
random sign, a full random mantissa and an exponent drawn geometrically below
2^-6, i.e. |x| in [2^-6, 2^-5) with p=1/2, [2^-7, 2^-6) with p=1/4, ... -- the
scale of the Llama N(0, 0.02) init.  Norm weights lie in [1, 1.03) (fp32) or
[1, 1.023) (bf16): "1 + small".
"""
from __future__ import annotations

import numpy as np

from .configs import MODELS, CONFIGS, Model, LayoutConfig, placement  # noqa: F401

_M = np.uint64(0xFFFFFFFFFFFFFFFF)
_K_SEED = np.uint64(0x9E3779B97F4A7C15)
_K_PARAM = np.uint64(0xD1B54A32D192ED03)
_K_ROW = np.uint64(0xABC98388FB8FAC03)
_K_COL = np.uint64(0x8CB92BA72F3D8DD7)


def _mix(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser (wrapping uint64 arithmetic)."""
    with np.errstate(over="ignore"):
        x = x ^ (x >> np.uint64(30))
        x = x * np.uint64(0xBF58476D1CE4E5B9)
        x = x ^ (x >> np.uint64(27))
        x = x * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return x


def hash64(seed: int, param: int, rows, cols) -> np.ndarray:
    """64-bit hash of (seed, param, row, col); rows/cols broadcast."""
    r = np.asarray(rows, dtype=np.uint64)
    c = np.asarray(cols, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = (np.uint64(seed) * _K_SEED + np.uint64(param) * _K_PARAM
             + r * _K_ROW + c * _K_COL)
    return _mix(x)


def _ctz8(t: np.ndarray) -> np.ndarray:
    """Trailing zeros of (t | 0x100) for t in [0, 256): a geometric draw in [0, 8]."""
    t = (t | np.uint64(0x100)).astype(np.uint64)
    k = np.zeros(t.shape, dtype=np.uint64)
    for _ in range(8):
        z = (t & np.uint64(1)) == 0
        k = k + z.astype(np.uint64)
        t = np.where(z, t >> np.uint64(1), t)
    return k


def weight_bits(seed: int, param: int, is_norm: bool, dtype: str, rows, cols) -> np.ndarray:
    """Bit patterns of trainer weight elements at global coordinates (rows, cols).

    dtype "f32" -> uint32 patterns, "bf16" -> uint16 patterns.  ``param`` is the
    canonical source-parameter id.
    """
    h = hash64(seed, param, rows, cols)
    if dtype == "f32":
        if is_norm:
            return (np.uint64(0x3F800000) | ((h >> np.uint64(8)) & np.uint64(0x3FFFF))).astype(np.uint32)
        sign = h >> np.uint64(63)
        k = _ctz8(h & np.uint64(0xFF))
        exp = np.uint64(127 - 6) - k
        mant = (h >> np.uint64(8)) & np.uint64(0x7FFFFF)
        return ((sign << np.uint64(31)) | (exp << np.uint64(23)) | mant).astype(np.uint32)
    if dtype == "bf16":
        if is_norm:
            return (np.uint64(0x3F80) | ((h >> np.uint64(8)) & np.uint64(0x3))).astype(np.uint16)
        sign = h >> np.uint64(63)
        k = _ctz8(h & np.uint64(0xFF))
        exp = np.uint64(127 - 6) - k
        mant = (h >> np.uint64(8)) & np.uint64(0x7F)
        return ((sign << np.uint64(15)) | (exp << np.uint64(7)) | mant).astype(np.uint16)
    raise ValueError(f"unsupported source dtype {dtype!r}")


def full_param_bits(seed: int, param: int, is_norm: bool, dtype: str, rows: int, cols: int) -> np.ndarray:
    """The whole [rows, cols] parameter as bit patterns (test sizes only)."""
    r = np.arange(rows, dtype=np.uint64)[:, None]
    c = np.arange(cols, dtype=np.uint64)[None, :]
    return weight_bits(seed, param, is_norm, dtype, r, c)
