"""ctypes wrapper of the CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / ``--impl reference`` legs of bench.py -- never by the product
package ``paper_2505_24034_b200``.  See oracle.c's header for what it computes
and the passages it follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, E_INVALID, E_INDIVISIBLE, E_MISMATCH, E_UNSUPPORTED = 0, -1, -2, -3, -4
E_NOMEM, E_UNCOVERED, E_OVERLAP = -7, -8, -9
DTYPES = {"f32": 0, "bf16": 1, "fp8": 2, "mxfp8": 3, "mxfp4": 4, "nvfp4": 5}


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared",
                               "-fno-fast-math", "-ffp-contract=off",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


class Model(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("n_layers", "d_model", "n_heads", "n_kv_heads", "head_dim", "d_ffn", "vocab", "with_embed")]


class Cfg(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("fsdp", "tp_train", "tp_gen", "src_dtype", "dst_dtype", "fsdp_inner", "dp_gen", "pp_train",
                 "pp_gen")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        i64p = ctypes.POINTER(ctypes.c_int64)
        ip = ctypes.POINTER(ctypes.c_int)
        M, C = ctypes.POINTER(Model), ctypes.POINTER(Cfg)
        L.orc_bf16_rne.argtypes, L.orc_bf16_rne.restype = [ctypes.c_uint32], ctypes.c_uint16
        L.orc_e4m3_rn_satfinite.argtypes, L.orc_e4m3_rn_satfinite.restype = [ctypes.c_float], ctypes.c_uint8
        L.orc_bf16_rne_array.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        L.orc_e4m3_array.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        L.orc_fp8_block.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        L.orc_mx_block.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_mx4_block.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_e2m1_array.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        L.orc_nv_tensor_scales.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        L.orc_nv_tensor_scales.restype = ctypes.c_float
        L.orc_nv_group.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_dst_tensor_scale_off.argtypes = [M, C, ctypes.c_int, ctypes.c_int]
        L.orc_dst_tensor_scale_off.restype = ctypes.c_int64
        L.orc_num_src_params.argtypes, L.orc_num_src_params.restype = [M], ctypes.c_int
        L.orc_num_dst_params.argtypes, L.orc_num_dst_params.restype = [M], ctypes.c_int
        L.orc_src_param_info.argtypes = [M, ctypes.c_int, i64p, i64p, ip]
        L.orc_src_piece.argtypes = [M, C, ctypes.c_int, ctypes.c_int, i64p, i64p, i64p, i64p]
        L.orc_src_piece.restype = ctypes.c_int64
        L.orc_src_rank_bytes.argtypes, L.orc_src_rank_bytes.restype = [M, C, ctypes.c_int], ctypes.c_int64
        L.orc_dst_rank_bytes.argtypes, L.orc_dst_rank_bytes.restype = [M, C, ctypes.c_int], ctypes.c_int64
        L.orc_dst_param.argtypes = [M, C, ctypes.c_int, ctypes.c_int, i64p, i64p, ip, i64p, i64p]
        L.orc_dst_element_source.argtypes = [M, C, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                             ctypes.c_int64, ip, i64p, i64p]
        L.orc_dst_param_sources.argtypes = [M, C, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.c_void_p]
        L.orc_sync.argtypes = [M, C, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_sync_range.argtypes = [M, C, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
        L.orc_check.argtypes = [M, C]
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def bf16_rne(bits_u32: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(bits_u32, dtype=np.uint32)
    out = np.empty(a.shape, dtype=np.uint16)
    lib().orc_bf16_rne_array(_ptr(a), a.size, _ptr(out))
    return out


def e4m3(vals_f32: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(vals_f32, dtype=np.float32)
    out = np.empty(a.shape, dtype=np.uint8)
    lib().orc_e4m3_array(_ptr(a), a.size, _ptr(out))
    return out


def fp8_block(x: np.ndarray):
    """Quantise one block (rows, cols <= 128) -> (uint8 codes, fp32 scale)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    q = np.empty(x.shape, dtype=np.uint8)
    s = np.zeros(1, dtype=np.float32)
    lib().orc_fp8_block(_ptr(x), x.shape[0], x.shape[1], x.shape[1], _ptr(q), x.shape[1], _ptr(s))
    return q, s[0]


def mx_block(x: np.ndarray):
    """Quantise one MXFP8 block (<= 32 elements) -> (uint8 codes, E8M0 scale byte)."""
    x = np.ascontiguousarray(x, dtype=np.float32).reshape(-1)
    q = np.empty(x.shape, dtype=np.uint8)
    s = np.zeros(1, dtype=np.uint8)
    lib().orc_mx_block(_ptr(x), x.size, _ptr(q), _ptr(s))
    return q, int(s[0])


def e2m1(vals_f32: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(vals_f32, dtype=np.float32)
    out = np.empty(a.shape, dtype=np.uint8)
    lib().orc_e2m1_array(_ptr(a), a.size, _ptr(out))
    return out


def mx4_block(x: np.ndarray):
    """Quantise one MXFP4 block (<= 32 elements) -> (uint8 codes, one per element; E8M0 byte)."""
    x = np.ascontiguousarray(x, dtype=np.float32).reshape(-1)
    q = np.empty(x.shape, dtype=np.uint8)
    s = np.zeros(1, dtype=np.uint8)
    lib().orc_mx4_block(_ptr(x), x.size, _ptr(q), _ptr(s))
    return q, int(s[0])


def nv_tensor_scales(x: np.ndarray):
    """NVFP4 per-tensor scales -> (S_dec, S_enc)."""
    x = np.ascontiguousarray(x, dtype=np.float32).reshape(-1)
    enc = ctypes.c_float()
    dec = lib().orc_nv_tensor_scales(_ptr(x), x.size, ctypes.byref(enc))
    return np.float32(dec), np.float32(enc.value)


def nv_group(x: np.ndarray, s_enc):
    """One NVFP4 group (<= 16 elements) -> (codes one per element, E4M3 scale byte)."""
    x = np.ascontiguousarray(x, dtype=np.float32).reshape(-1)
    q = np.empty(x.shape, dtype=np.uint8)
    s = np.zeros(1, dtype=np.uint8)
    lib().orc_nv_group(_ptr(x), x.size, float(s_enc), _ptr(q), _ptr(s))
    return q, int(s[0])


class Layout:
    """The oracle's own view of both layouts for one configuration."""

    def __init__(self, model, fsdp, tp_train, tp_gen, src_dtype="f32", dst_dtype="bf16", fsdp_inner=False,
                 dp_gen=1, pp_train=1, pp_gen=1):
        m = model
        self.m = Model(m.n_layers, m.d_model, m.n_heads, m.n_kv_heads, m.head_dim, m.d_ffn, m.vocab, m.with_embed)
        self.c = Cfg(fsdp, tp_train, tp_gen, DTYPES[src_dtype], DTYPES[dst_dtype], int(fsdp_inner), dp_gen,
                     pp_train, pp_gen)
        self.src_dtype, self.dst_dtype = src_dtype, dst_dtype
        self.n_src, self.n_dst = fsdp * tp_train * pp_train, tp_gen * pp_gen * dp_gen
        L = lib()
        self.status = L.orc_check(ctypes.byref(self.m), ctypes.byref(self.c))
        self.n_src_params = L.orc_num_src_params(ctypes.byref(self.m))
        self.n_dst_params = L.orc_num_dst_params(ctypes.byref(self.m))

    def src_param_info(self, p):
        R, C, k = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
        lib().orc_src_param_info(ctypes.byref(self.m), p, ctypes.byref(R), ctypes.byref(C), ctypes.byref(k))
        return R.value, C.value, k.value

    def src_piece(self, rank, p):
        """-> (byte offset, r0, r1, c0, c1) of param p in trainer rank's buffer."""
        v = [ctypes.c_int64() for _ in range(4)]
        off = lib().orc_src_piece(ctypes.byref(self.m), ctypes.byref(self.c), rank, p, *[ctypes.byref(x) for x in v])
        return (off,) + tuple(x.value for x in v)

    def src_rank_bytes(self, rank):
        return lib().orc_src_rank_bytes(ctypes.byref(self.m), ctypes.byref(self.c), rank)

    def dst_rank_bytes(self, g):
        return lib().orc_dst_rank_bytes(ctypes.byref(self.m), ctypes.byref(self.c), g)

    def dst_param(self, g, gp):
        """-> (rows, cols, quant, byte offset, scale byte offset or -1)."""
        R, C, o, s = (ctypes.c_int64() for _ in range(4))
        q = ctypes.c_int()
        rc = lib().orc_dst_param(ctypes.byref(self.m), ctypes.byref(self.c), g, gp, ctypes.byref(R),
                                 ctypes.byref(C), ctypes.byref(q), ctypes.byref(o), ctypes.byref(s))
        assert rc == 0
        return R.value, C.value, q.value, o.value, s.value

    def dst_tensor_scale_off(self, g, gp):
        return lib().orc_dst_tensor_scale_off(ctypes.byref(self.m), ctypes.byref(self.c), g, gp)

    def dst_element_source(self, g, gp, lr, lc):
        p, r, c = ctypes.c_int(), ctypes.c_int64(), ctypes.c_int64()
        rc = lib().orc_dst_element_source(ctypes.byref(self.m), ctypes.byref(self.c), g, gp, lr, lc,
                                          ctypes.byref(p), ctypes.byref(r), ctypes.byref(c))
        assert rc == 0
        return p.value, r.value, c.value

    def dst_param_sources(self, g, gp):
        """-> (src_param [R,C] int32, row [R,C] int64, col [R,C] int64): the source
        element of every element of generator param gp on rank g."""
        R, C = self.dst_param(g, gp)[:2]
        p = np.empty((R, C), np.int32)
        r = np.empty((R, C), np.int64)
        c = np.empty((R, C), np.int64)
        rc = lib().orc_dst_param_sources(ctypes.byref(self.m), ctypes.byref(self.c), g, gp, _ptr(p), _ptr(r), _ptr(c))
        assert rc == 0, rc
        return p, r, c

    def sync_addrs(self, src_addrs, dst_addrs, gp_range):
        """orc_sync_range on raw host addresses: src_addrs[r] / dst_addrs[q] are the
        (virtual) bases of the rank buffers; only the bytes of the params in
        gp_range are read / written, so a caller may pass ``slice address -
        slice offset`` to stream one parameter at a time."""
        S = (ctypes.c_void_p * len(src_addrs))(*src_addrs)
        D = (ctypes.c_void_p * len(dst_addrs))(*dst_addrs)
        return lib().orc_sync_range(ctypes.byref(self.m), ctypes.byref(self.c), S, D, gp_range[0], gp_range[1])

    def sync(self, src_bufs, dst_bufs, gp_range=None):
        """Run the oracle on host numpy uint8 buffers (dst written in place)."""
        S = (ctypes.c_void_p * len(src_bufs))(*[_ptr(b) for b in src_bufs])
        D = (ctypes.c_void_p * len(dst_bufs))(*[_ptr(b) for b in dst_bufs])
        if gp_range is None:
            return lib().orc_sync(ctypes.byref(self.m), ctypes.byref(self.c), S, D)
        return lib().orc_sync_range(ctypes.byref(self.m), ctypes.byref(self.c), S, D, gp_range[0], gp_range[1])
