"""Thin ctypes binding of libllrl (include/llrl.h): argument marshalling only.

Every step of the path runs in the library's C++ planner and sm_100a kernels.
There is no Python or CPU fallback: if ``libllrl.so`` is missing, importing
this module raises.  PyTorch is used by callers for device memory, streams and
process groups only.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libllrl.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libllrl.so not built at {LIB_PATH}: run __graft_entry__.build() "
                      "(python paper_2505_24034_b200/build.py)")

_lib = ctypes.CDLL(LIB_PATH)

OK, E_INVALID, E_INDIVISIBLE, E_MISMATCH, E_UNSUPPORTED, E_CUDA, E_NOPEER, E_NOMEM = 0, -1, -2, -3, -4, -5, -6, -7
F32, BF16, FP8_E4M3, MXFP8, MXFP4, NVFP4 = 0, 1, 2, 3, 4, 5
DTYPES = {"f32": F32, "bf16": BF16, "fp8": FP8_E4M3, "mxfp8": MXFP8, "mxfp4": MXFP4, "nvfp4": NVFP4}
MESH_FSDP_INNER = 1
PLAN_MULTICAST = 1
PLAN_NCCL = 2
(P_ATTN_NORM, P_Q, P_K, P_V, P_O, P_MLP_NORM, P_GATE, P_UP, P_DOWN, P_EMBED, P_FINAL_NORM, P_LM_HEAD,
 P_QKV, P_GATE_UP) = range(14)

EXPORTS = [
    "llrl_layout_describe", "llrl_layout_describe_ex", "llrl_layout_num_ranks", "llrl_layout_num_params", "llrl_layout_rank_bytes",
    "llrl_layout_param_view", "llrl_layout_destroy", "llrl_plan_create", "llrl_plan_destroy",
    "llrl_plan_num_runs", "llrl_plan_get_runs", "llrl_plan_stats_get", "llrl_plan_traffic",
    "llrl_plan_device_bytes", "llrl_plan_device_info", "llrl_comm_create", "llrl_comm_export", "llrl_comm_import", "llrl_comm_flag_ptr",
    "llrl_comm_set_peer", "llrl_comm_timed_out", "llrl_comm_destroy", "llrl_ipc_handle", "llrl_ipc_open", "llrl_ipc_close",
    "llrl_sync", "llrl_sync_host", "llrl_plan_num_groups", "llrl_plan_group_range", "llrl_plan_set_max_ctas", "llrl_sync_group", "llrl_sync_num_launches", "llrl_fill_synthetic", "llrl_mc_create", "llrl_mc_import", "llrl_mc_join",
    "llrl_mc_destroy", "llrl_plan_set_multicast", "llrl_last_error", "llrl_plan_nv_num_tensors",
    "llrl_plan_nv_tensor", "llrl_plan_nv_tensor_sources", "llrl_sync_nv_amax", "llrl_nccl_unique_id",
    "llrl_nccl_attach", "llrl_plan_nccl_info", "llrl_debug_timeline", "llrl_mc_export_local", "llrl_mc_map_peer",
    "llrl_version",
]


class LlrlError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"llrl status {status}: {msg}")
        self.status = status


class ModelDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("n_layers", "d_model", "n_heads", "n_kv_heads", "head_dim", "d_ffn", "vocab", "with_embed")]


class LayoutOpts(ctypes.Structure):
    _fields_ = [("fsdp", ctypes.c_int32), ("tp_train", ctypes.c_int32), ("tp_gen", ctypes.c_int32),
                ("dp_gen", ctypes.c_int32), ("pp_train", ctypes.c_int32), ("pp_gen", ctypes.c_int32),
                ("src_dtype", ctypes.c_int32), ("dst_dtype", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("reserved", ctypes.c_int32)]


class ParamView(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("layer", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("quantised", ctypes.c_int32), ("rows", ctypes.c_int64), ("cols", ctypes.c_int64),
                ("byte_off", ctypes.c_int64), ("scale_off", ctypes.c_int64), ("full_r0", ctypes.c_int64),
                ("full_c0", ctypes.c_int64), ("src_param", ctypes.c_int32), ("is_norm", ctypes.c_int32),
                ("tensor_scale_off", ctypes.c_int64)]


class Run(ctypes.Structure):
    _fields_ = [("src_param", ctypes.c_int32), ("src_rank", ctypes.c_int32), ("dst_rank", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("src_off", ctypes.c_int64), ("dst_off", ctypes.c_int64),
                ("len", ctypes.c_int64)]


class PlanStats(ctypes.Structure):
    _fields_ = [("n_devices", ctypes.c_int32), ("n_src_ranks", ctypes.c_int32), ("n_dst_ranks", ctypes.c_int32),
                ("n_tiles", ctypes.c_int64), ("n_items", ctypes.c_int64), ("n_fp8_blocks", ctypes.c_int64),
                ("n_fp8_pull_blocks", ctypes.c_int64), ("src_bytes", ctypes.c_int64), ("dst_bytes", ctypes.c_int64)]


class DeviceInfo(ctypes.Structure):
    _fields_ = [("n_items", ctypes.c_int64), ("n_cast_items", ctypes.c_int64), ("n_fp8_items", ctypes.c_int64),
                ("n_fp8_pull_items", ctypes.c_int64), ("n_signal", ctypes.c_int32),
                ("n_senders_in", ctypes.c_int32), ("n_launches", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("nv_amax_read_bytes", ctypes.c_int64)]


class NcclInfo(ctypes.Structure):
    _fields_ = [("n_broadcasts", ctypes.c_int32), ("n_allgathers", ctypes.c_int32), ("bytes", ctypes.c_int64),
                ("mode", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class NvTensor(ctypes.Structure):
    _fields_ = [("dst_rank", ctypes.c_int32), ("dst_param", ctypes.c_int32), ("device", ctypes.c_int32),
                ("n_sources", ctypes.c_int32)]


class NvSource(ctypes.Structure):
    _fields_ = [("src_rank", ctypes.c_int32), ("src_param", ctypes.c_int32), ("src_off", ctypes.c_int64),
                ("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("src_ld", ctypes.c_int64)]


_vp, _i64, _int = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
_P = ctypes.POINTER


def _sig(name, args, res=ctypes.c_int):
    f = getattr(_lib, name)
    f.argtypes, f.restype = args, res


_sig("llrl_layout_describe", [_P(ModelDesc), _int, _int, _int, _int, _int, ctypes.c_uint32, _P(_vp), _P(_vp)])
_sig("llrl_layout_describe_ex", [_P(ModelDesc), _P(LayoutOpts), _P(_vp), _P(_vp)])
_sig("llrl_layout_num_ranks", [_vp, _P(_int)])
_sig("llrl_layout_num_params", [_vp, _P(_int)])
_sig("llrl_layout_rank_bytes", [_vp, _int, _P(_i64)])
_sig("llrl_layout_param_view", [_vp, _int, _int, _P(ParamView)])
_sig("llrl_layout_destroy", [_vp], None)
_sig("llrl_plan_create", [_vp, _vp, _P(_int), _P(_int), ctypes.c_uint32, _P(_vp)])
_sig("llrl_plan_destroy", [_vp], None)
_sig("llrl_plan_num_runs", [_vp, _P(_i64)])
_sig("llrl_plan_get_runs", [_vp, _i64, _i64, _P(Run)])
_sig("llrl_plan_stats_get", [_vp, _P(PlanStats)])
_sig("llrl_plan_traffic", [_vp, _P(_i64)])
_sig("llrl_plan_device_bytes", [_vp, _int, _P(_i64), _P(_i64), _P(_i64), _P(_i64)])
_sig("llrl_plan_device_info", [_vp, _int, _P(DeviceInfo)])
_sig("llrl_mc_create", [_int, _i64, _P(_int), _P(_i64), _P(_vp)])
_sig("llrl_mc_import", [_int, _int, _i64, _P(_vp)])
_sig("llrl_mc_join", [_vp, _int, _P(_vp), _P(_vp)])
_sig("llrl_mc_destroy", [_vp], None)
_sig("llrl_mc_export_local", [_vp, _P(_int)])
_sig("llrl_mc_map_peer", [_vp, _int, _int, _P(_vp)])
_sig("llrl_plan_set_multicast", [_vp, _int, _P(_vp)])
_sig("llrl_comm_create", [_int, _P(_vp)])
_sig("llrl_comm_export", [_vp, ctypes.c_char_p])
_sig("llrl_comm_import", [_vp, _int, ctypes.c_char_p])
_sig("llrl_comm_flag_ptr", [_vp, _P(_vp)])
_sig("llrl_comm_set_peer", [_vp, _int, _vp])
_sig("llrl_comm_timed_out", [_vp, _P(_int)])
_sig("llrl_comm_destroy", [_vp], None)
_sig("llrl_ipc_handle", [_vp, ctypes.c_char_p, _P(_i64)])
_sig("llrl_ipc_open", [ctypes.c_char_p, _i64, _P(_vp)])
_sig("llrl_ipc_close", [_vp, _i64])
_sig("llrl_sync", [_vp, _vp, _int, _P(_vp), _P(_vp), _vp])
_sig("llrl_plan_num_groups", [_vp, _P(_int)])
_sig("llrl_plan_set_max_ctas", [_vp, _int, _int])
_sig("llrl_plan_group_range", [_vp, _int, _int, _int, _P(_i64), _P(_i64)])
_sig("llrl_sync_group", [_vp, _vp, _int, _int, _P(_vp), _P(_vp), _vp])
_sig("llrl_sync_host", [_vp, _vp, _int, _P(_vp), _P(_vp), _P(_vp), _P(_vp), _vp])
_sig("llrl_sync_num_launches", [_vp, _int, _P(_int)])
_sig("llrl_plan_nv_num_tensors", [_vp, _P(_int)])
_sig("llrl_plan_nv_tensor", [_vp, _int, _P(NvTensor)])
_sig("llrl_plan_nv_tensor_sources", [_vp, _int, _int, _int, _P(NvSource)])
_sig("llrl_sync_nv_amax", [_vp, _vp, _int, _vp, _P(_vp), _P(_vp), _vp])
_sig("llrl_nccl_unique_id", [ctypes.c_char_p])
_sig("llrl_nccl_attach", [_vp, _int, ctypes.c_char_p, _int, _int])
_sig("llrl_plan_nccl_info", [_vp, _int, _P(NcclInfo)])
_sig("llrl_debug_timeline", [_vp, _int, _P(ctypes.c_uint64), _int, _P(_int)])
_sig("llrl_fill_synthetic", [_vp, _int, _vp, ctypes.c_uint64, _vp])
_sig("llrl_last_error", [], ctypes.c_char_p)
_sig("llrl_version", [], ctypes.c_char_p)


def lib():
    return _lib


def _check(st):
    if st != OK:
        raise LlrlError(st, _lib.llrl_last_error().decode())


def _ptrs(values):
    return (_vp * max(1, len(values)))(*[int(v) if v else None for v in values])


class Layout:
    """Owns one side's llrl_layout (created in pairs by ``describe``)."""
    _h = None

    def __init__(self, handle, is_src):
        self._h = _vp(handle)
        self.is_src = is_src
        n = _int()
        _check(_lib.llrl_layout_num_ranks(self._h, ctypes.byref(n)))
        self.n_ranks = n.value
        _check(_lib.llrl_layout_num_params(self._h, ctypes.byref(n)))
        self.n_params = n.value

    @property
    def handle(self):
        return self._h

    def rank_bytes(self, rank):
        b = _i64()
        _check(_lib.llrl_layout_rank_bytes(self._h, rank, ctypes.byref(b)))
        return b.value

    def param_view(self, rank, param) -> ParamView:
        v = ParamView()
        _check(_lib.llrl_layout_param_view(self._h, rank, param, ctypes.byref(v)))
        return v

    def close(self):
        if self._h and _lib is not None:     # (at interpreter exit the module may be torn down first)
            _lib.llrl_layout_destroy(self._h)
            self._h = None

    __del__ = close


def nccl_unique_id() -> bytes:
    """llrl_nccl_unique_id: 128 bytes to share with every process before llrl_nccl_attach."""
    buf = ctypes.create_string_buffer(128)
    _check(_lib.llrl_nccl_unique_id(buf))
    return buf.raw


def describe(model, fsdp, tp_train, tp_gen, src_dtype="f32", dst_dtype="bf16", fsdp_inner=False, dp_gen=1,
             pp_train=1, pp_gen=1):
    """llrl_layout_describe_ex -> (src Layout, dst Layout)."""
    m = ModelDesc(model.n_layers, model.d_model, model.n_heads, model.n_kv_heads, model.head_dim, model.d_ffn,
                  model.vocab, model.with_embed)
    o = LayoutOpts(fsdp, tp_train, tp_gen, dp_gen, pp_train, pp_gen, DTYPES[src_dtype], DTYPES[dst_dtype],
                   MESH_FSDP_INNER if fsdp_inner else 0, 0)
    s, d = _vp(), _vp()
    _check(_lib.llrl_layout_describe_ex(ctypes.byref(m), ctypes.byref(o), ctypes.byref(s), ctypes.byref(d)))
    return Layout(s.value, True), Layout(d.value, False)


class Plan:
    _h = None

    def __init__(self, src: Layout, dst: Layout, src_device, dst_device, multicast=False, nccl=False):
        assert len(src_device) == src.n_ranks and len(dst_device) == dst.n_ranks
        h = _vp()
        sd = (_int * len(src_device))(*src_device)
        dd = (_int * len(dst_device))(*dst_device)
        _check(_lib.llrl_plan_create(src.handle, dst.handle, sd, dd,
                                     (PLAN_MULTICAST if multicast else 0) | (PLAN_NCCL if nccl else 0),
                                     ctypes.byref(h)))
        self._h = h
        self.n_src, self.n_dst = src.n_ranks, dst.n_ranks
        self.src_device, self.dst_device = list(src_device), list(dst_device)

    @property
    def handle(self):
        return self._h

    def stats(self) -> PlanStats:
        s = PlanStats()
        _check(_lib.llrl_plan_stats_get(self._h, ctypes.byref(s)))
        return s

    def traffic(self):
        G = self.stats().n_devices
        buf = (_i64 * (G * G))()
        _check(_lib.llrl_plan_traffic(self._h, buf))
        return [[buf[i * G + j] for j in range(G)] for i in range(G)]

    def device_bytes(self, device):
        v = [_i64() for _ in range(4)]
        _check(_lib.llrl_plan_device_bytes(self._h, device, *[ctypes.byref(x) for x in v]))
        return dict(zip(("hbm_read", "hbm_write", "nvl_tx", "nvl_rx"), (x.value for x in v)))

    def device_info(self, device) -> DeviceInfo:
        v = DeviceInfo()
        _check(_lib.llrl_plan_device_info(self._h, device, ctypes.byref(v)))
        return v

    def set_multicast(self, device, dst_mc_ptrs):
        _check(_lib.llrl_plan_set_multicast(self._h, device, _ptrs(dst_mc_ptrs)))

    def num_runs(self):
        n = _i64()
        _check(_lib.llrl_plan_num_runs(self._h, ctypes.byref(n)))
        return n.value

    def runs(self, first=0, count=None):
        """Canonical 1-D runs as a numpy structured array."""
        import numpy as np
        if count is None:
            count = self.num_runs() - first
        dt = np.dtype([("src_param", np.int32), ("src_rank", np.int32), ("dst_rank", np.int32),
                       ("flags", np.int32), ("src_off", np.int64), ("dst_off", np.int64), ("len", np.int64)])
        out = np.zeros(count, dtype=dt)
        _check(_lib.llrl_plan_get_runs(self._h, first, count, out.ctypes.data_as(_P(Run))))
        return out

    def num_launches(self, device):
        n = _int()
        _check(_lib.llrl_sync_num_launches(self._h, device, ctypes.byref(n)))
        return n.value

    def sync(self, comm, device, src_ptrs, dst_ptrs, stream):
        """llrl_sync: enqueue this device's share of the sync on `stream` (int handle)."""
        _check(_lib.llrl_sync(self._h, comm.handle if comm else None, device, _ptrs(src_ptrs), _ptrs(dst_ptrs),
                              _vp(stream)))

    def num_groups(self):
        n = _int()
        _check(_lib.llrl_plan_num_groups(self._h, ctypes.byref(n)))
        return n.value

    def set_max_ctas(self, device, n):
        _check(_lib.llrl_plan_set_max_ctas(self._h, device, n))

    def group_range(self, side, rank, group):
        lo, hi = _i64(), _i64()
        _check(_lib.llrl_plan_group_range(self._h, side, rank, group, ctypes.byref(lo), ctypes.byref(hi)))
        return lo.value, hi.value

    def sync_group(self, comm, device, group, src_ptrs, dst_ptrs, stream):
        """llrl_sync_group: this device's share of one layer group."""
        _check(_lib.llrl_sync_group(self._h, comm.handle if comm else None, device, group, _ptrs(src_ptrs),
                                    _ptrs(dst_ptrs), _vp(stream)))

    def nv_num_tensors(self):
        n = _int()
        _check(_lib.llrl_plan_nv_num_tensors(self._h, ctypes.byref(n)))
        return n.value

    def nv_tensor(self, tid) -> NvTensor:
        t = NvTensor()
        _check(_lib.llrl_plan_nv_tensor(self._h, tid, ctypes.byref(t)))
        return t

    def nv_tensor_sources(self, tid):
        n = self.nv_tensor(tid).n_sources
        out = (NvSource * max(1, n))()
        _check(_lib.llrl_plan_nv_tensor_sources(self._h, tid, 0, n, out))
        return list(out[:n])

    def debug_timeline(self, device, max_ctas=4096):
        """llrl_debug_timeline: [(start_ns, end_ns)] per CTA of the last cast launch
        (needs LLRL_TIMELINE=1 before the first sync)."""
        buf = (ctypes.c_uint64 * (2 * max_ctas))()
        n = _int()
        _check(_lib.llrl_debug_timeline(self._h, device, buf, max_ctas, ctypes.byref(n)))
        return [(buf[2 * c], buf[2 * c + 1]) for c in range(n.value)]

    def nccl_info(self, device) -> NcclInfo:
        v = NcclInfo()
        _check(_lib.llrl_plan_nccl_info(self._h, device, ctypes.byref(v)))
        return v

    def nccl_attach(self, device, uid: bytes, rank, nranks):
        """llrl_nccl_attach (collective over every process of the job)."""
        _check(_lib.llrl_nccl_attach(self._h, device, uid, rank, nranks))

    def sync_nv_amax(self, comm, device, amax_ptr, src_ptrs, dst_ptrs, stream):
        """llrl_sync_nv_amax: NVFP4 in one pass with the caller's per-tensor amax."""
        _check(_lib.llrl_sync_nv_amax(self._h, comm.handle if comm else None, device, _vp(amax_ptr),
                                      _ptrs(src_ptrs), _ptrs(dst_ptrs), _vp(stream)))

    def sync_host(self, comm, device, host_src, host_dst, src_ptrs, dst_ptrs, stream):
        _check(_lib.llrl_sync_host(self._h, comm.handle if comm else None, device, _ptrs(host_src),
                                   _ptrs(host_dst), _ptrs(src_ptrs), _ptrs(dst_ptrs), _vp(stream)))

    def close(self):
        if self._h and _lib is not None:
            _lib.llrl_plan_destroy(self._h)
            self._h = None

    __del__ = close


class Comm:
    """Completion flags of one device (a6)."""
    _h = None

    def __init__(self, device):
        h = _vp()
        _check(_lib.llrl_comm_create(device, ctypes.byref(h)))
        self._h = h
        self.device = device

    @property
    def handle(self):
        return self._h

    def export(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        _check(_lib.llrl_comm_export(self._h, buf))
        return buf.raw

    def import_peer(self, peer_device, handle: bytes):
        _check(_lib.llrl_comm_import(self._h, peer_device, handle))

    def flag_ptr(self):
        p = _vp()
        _check(_lib.llrl_comm_flag_ptr(self._h, ctypes.byref(p)))
        return p.value

    def timed_out(self) -> bool:
        v = _int()
        _check(_lib.llrl_comm_timed_out(self._h, ctypes.byref(v)))
        return bool(v.value)

    def set_peer(self, peer_device, ptr):
        _check(_lib.llrl_comm_set_peer(self._h, peer_device, _vp(ptr)))

    def close(self):
        if self._h:
            _lib.llrl_comm_destroy(self._h)
            self._h = None

    __del__ = close


class McBuf:
    """One NVLS multicast object (llrl_mc_*)."""
    _h = None

    def __init__(self, handle, size):
        self._h = handle
        self.size = size

    @staticmethod
    def create(n_devices, nbytes):
        h, fd, size = _vp(), _int(), _i64()
        _check(_lib.llrl_mc_create(n_devices, nbytes, ctypes.byref(fd), ctypes.byref(size), ctypes.byref(h)))
        return McBuf(h, size.value), fd.value

    @staticmethod
    def import_fd(fd, n_devices, size):
        h = _vp()
        _check(_lib.llrl_mc_import(fd, n_devices, size, ctypes.byref(h)))
        return McBuf(h, size)

    def join(self, device):
        """-> (local unicast pointer, multicast pointer) on `device`."""
        a, b = _vp(), _vp()
        _check(_lib.llrl_mc_join(self._h, device, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def export_local(self):
        """POSIX fd of this process's memory bound to the object (after join)."""
        fd = _int()
        _check(_lib.llrl_mc_export_local(self._h, ctypes.byref(fd)))
        return fd.value

    def map_peer(self, fd, device):
        """Map a peer's bound memory (its exported fd) for `device` -> pointer."""
        p = _vp()
        _check(_lib.llrl_mc_map_peer(self._h, fd, device, ctypes.byref(p)))
        return p.value

    def close(self):
        if self._h:
            _lib.llrl_mc_destroy(self._h)
            self._h = None

    __del__ = close


def ipc_handle(ptr):
    buf = ctypes.create_string_buffer(64)
    off = _i64()
    _check(_lib.llrl_ipc_handle(_vp(ptr), buf, ctypes.byref(off)))
    return buf.raw, off.value


def ipc_open(handle: bytes, offset: int) -> int:
    p = _vp()
    _check(_lib.llrl_ipc_open(handle, offset, ctypes.byref(p)))
    return p.value


def ipc_close(ptr, offset):
    _check(_lib.llrl_ipc_close(_vp(ptr), offset))


def fill_synthetic(src_layout: Layout, rank, ptr, seed, stream):
    _check(_lib.llrl_fill_synthetic(src_layout.handle, rank, _vp(ptr), seed, _vp(stream)))


def version():
    return _lib.llrl_version().decode()
