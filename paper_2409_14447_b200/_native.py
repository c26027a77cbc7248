"""Loader of the sm_100a CUDA library and device-side containers.

There is no CPU implementation of the planner in this package: every
planning entry point calls into `_build/libparva_b200.so` through the C ABI
declared in include/parva_b200.h.  If the library or a CUDA device is
missing, `lib()` / `require_cuda()` raise NativeLibraryError.

PyTorch is used only as the device-memory and stream provider: tensors hold
the device buffers, `torch.cuda.current_stream()` orders the launches.
"""

from __future__ import annotations

import ctypes as C
import threading
from collections import OrderedDict

import numpy as np

from .errors import NativeLibraryError
from .records import CONFIG_DTYPE, PLAN_DTYPE

_LIB = None
_LOCK = threading.Lock()


class ParvaTables(C.Structure):
    _fields_ = [("d_pts", C.c_void_p), ("d_seg_start", C.c_void_p),
                ("d_seg_count", C.c_void_p), ("n_tables", C.c_int32), ("n_points", C.c_int64),
                ("max_seg_points", C.c_int32)]


class ParvaRawTables(C.Structure):
    _fields_ = [("d_tp", C.c_void_p), ("d_lat", C.c_void_p), ("d_mem", C.c_void_p), ("d_procs", C.c_void_p),
                ("d_seg_start", C.c_void_p), ("d_seg_count", C.c_void_p), ("n_tables", C.c_int32),
                ("n_points", C.c_int64)]


class ParvaIndex(C.Structure):
    _fields_ = [("d_lat_sorted", C.c_void_p), ("d_best", C.c_void_p), ("d_tp", C.c_void_p)]


class GeneralProblem(C.Structure):
    _fields_ = [("n_cat", C.c_int32), ("d_cat_size", C.c_void_p), ("d_cat_tp", C.c_void_p),
                ("d_cat_name", C.c_void_p), ("n_services", C.c_int32), ("n_names", C.c_int32),
                ("d_svc_t1", C.c_void_p), ("d_svc_t2", C.c_void_p), ("d_svc_opt", C.c_void_p),
                ("d_svc_count", C.c_void_p), ("d_svc_last", C.c_void_p), ("d_svc_rate", C.c_void_p),
                ("n_gpus", C.c_int32), ("d_gpu_id", C.c_void_p), ("d_pl_off", C.c_void_p),
                ("d_pl_cat", C.c_void_p), ("d_pl_slot", C.c_void_p), ("d_ledger_val", C.c_void_p),
                ("d_ledger_order", C.c_void_p), ("relocate", C.c_int32), ("optimize", C.c_int32),
                ("threshold", C.c_int32)]


class GeneralResult(C.Structure):
    _fields_ = [("gpu_cap", C.c_int32), ("place_cap", C.c_int32), ("diag_cap", C.c_int32),
                ("d_status", C.c_void_p), ("d_counts", C.c_void_p), ("d_gpu_id", C.c_void_p),
                ("d_pl_off", C.c_void_p), ("d_pl_cat", C.c_void_p), ("d_pl_slot", C.c_void_p),
                ("d_diag", C.c_void_p), ("d_ledger_val", C.c_void_p), ("d_ledger_order", C.c_void_p),
                ("d_fallback", C.c_void_p)]


class SimProblem(C.Structure):
    _fields_ = [("n_services", C.c_int32), ("d_kind", C.c_void_p), ("d_pcg", C.c_void_p), ("d_scale", C.c_void_p),
                ("d_count", C.c_void_p), ("d_horizon_s", C.c_void_p), ("d_buf_off", C.c_void_p),
                ("d_seg_off", C.c_void_p), ("d_seg_ms", C.c_void_p), ("d_seg_batch", C.c_void_p),
                ("d_seg_lanes", C.c_void_p), ("d_slo", C.c_void_p), ("d_horizon_ms", C.c_void_p)]


class SimResult(C.Structure):
    _fields_ = [("d_arrived", C.c_void_p), ("d_served", C.c_void_p), ("d_batches", C.c_void_p),
                ("d_violations", C.c_void_p), ("d_buf", C.c_void_p), ("d_busy_ms", C.c_void_p),
                ("d_status", C.c_void_p)]


EXPORTS = (
    "parva_abi_version", "parva_plan_batch_workspace", "parva_build_index", "parva_configure_sweep",
    "parva_plan_batch", "parva_plan_batch_overlapped", "parva_plan_batch_fused", "parva_gather_wait",
    "parva_gather_release", "parva_host_gate",
    "parva_ipc_alloc", "parva_ipc_free", "parva_ipc_handle_bytes", "parva_ipc_handle", "parva_ipc_open",
    "parva_ipc_close", "parva_plan_batch_preconfigured", "parva_plan_host_scratch", "parva_plan_host",
    "parva_plan_general_workspace", "parva_plan_general", "parva_select_optimal_lists",
    "parva_match_demand_lists", "parva_propose_small_batch", "parva_packed_layout",
    "parva_plan_host_packed_scratch", "parva_plan_host_packed", "parva_prepare_tables",
    "parva_mapped_layout", "parva_plan_host_mapped_scratch", "parva_plan_host_mapped", "parva_stream_bytes",
    "parva_stream_pack", "parva_stream_pack_arrays", "parva_forget_block", "parva_plan_host_mapped_submit", "parva_plan_host_mapped_wait",
    "parva_plan_host_arrays_submit",
    "parva_simulate", "parva_sim_seed_states", "parva_sim_log1p", "parva_sim_exponential",
)


class SlotTicket(C.Structure):
    """parva_slot_ticket (include/parva_b200.h): serializes overlapped launches
    that share an output slot."""
    _fields_ = [("d_count", C.c_void_p), ("wait_count", C.c_uint64), ("d_err", C.c_void_p)]


class Mirror(C.Structure):
    """parva_mirror (include/parva_b200.h): the fused all-gather's destinations."""
    _fields_ = [("n", C.c_int32), ("overlap", C.c_int32), ("plan", C.c_void_p * 8), ("cfg", C.c_void_p * 8),
                ("spill", C.c_void_p * 8), ("flag", C.c_void_p * 8), ("d_acks", C.c_void_p), ("d_done", C.c_void_p),
                ("d_spill", C.c_void_p), ("plan_capacity", C.c_int64), ("cfg_capacity", C.c_int64),
                ("spill_capacity", C.c_int64), ("plan_bytes", C.c_int32), ("epoch", C.c_uint32),
                ("prev_epoch", C.c_uint32), ("reserved", C.c_int32), ("ticket", SlotTicket)]


class GatherSlot(C.Structure):
    """parva_gather_slot (include/parva_b200.h): the consumer side of one slot."""
    _fields_ = [("n", C.c_int32), ("pdl", C.c_int32), ("d_flags", C.c_void_p), ("ack", C.c_void_p * 8)]


def lib_path():
    from .build import LIB
    return LIB


def load_library(build_if_missing: bool = True):
    """dlopen the library (no CUDA device needed to load it)."""
    global _LIB
    with _LOCK:
        if _LIB is None:
            from . import build as _build
            path = _build.LIB
            if build_if_missing and _build.stale():
                try:
                    _build.build()
                except Exception as exc:  # noqa: BLE001
                    raise NativeLibraryError(f"cannot build {path}: {exc}") from exc
            if not path.exists():
                raise NativeLibraryError(f"CUDA library {path} is missing; run __graft_entry__.build()")
            try:
                _LIB = C.CDLL(str(path))
            except OSError as exc:
                raise NativeLibraryError(f"cannot load {path}: {exc}") from exc
            _LIB.parva_plan_batch_workspace.restype = C.c_size_t
            _LIB.parva_plan_host_scratch.restype = C.c_size_t
            _LIB.parva_plan_general_workspace.restype = C.c_size_t
            _LIB.parva_plan_host_packed_scratch.restype = C.c_size_t
            _LIB.parva_plan_host_mapped_scratch.restype = C.c_size_t
            _LIB.parva_stream_bytes.restype = C.c_int64
            _LIB.parva_stream_pack.restype = C.c_int64
            _LIB.parva_stream_pack_arrays.restype = C.c_int64
            V, I32 = C.c_void_p, C.c_int32
            _LIB.parva_plan_host_arrays_submit.argtypes = [V, V, I32, V, V, V, V, I32, V, C.c_int64, V, I32, I32,
                                                           I32, I32, V, C.c_size_t, V, V]
        return _LIB


def lib():
    return load_library()


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise NativeLibraryError("no CUDA device: the planner runs only on the GPU (sm_100a); there is no CPU path")
    lib()
    return torch


def stream_handle(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def np_ptr(a: np.ndarray):
    """ctypes pointer to a C-contiguous numpy array (host memory)."""
    assert a.flags["C_CONTIGUOUS"]
    return C.c_void_p(a.ctypes.data)


def check(rc: int, what: str):
    if rc != 0:
        raise NativeLibraryError(f"{what} failed with parva status {rc}")


def ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def to_device(a: np.ndarray, pad: int = 0):
    torch = require_cuda()
    a = np.ascontiguousarray(a)
    if pad:
        a = np.concatenate([a, np.zeros(pad, dtype=a.dtype)])
    return torch.from_numpy(a).to("cuda", non_blocking=False)


def empty_records(n: int, dtype: np.dtype):
    torch = require_cuda()
    return torch.empty((max(n, 1), dtype.itemsize), dtype=torch.uint8, device="cuda")


def records_to_numpy(t, n: int, dtype: np.dtype) -> np.ndarray:
    return t[:n].cpu().numpy().view(dtype).reshape(n)


class DeviceTables:
    """Prepared tables resident in HBM + their prefix-argmax index.

    Layout: (tp, lat) f64 pairs [2P] (+2 pad), seg_start i64[T*5],
    seg_count i32[T*5];
    index: lat_sorted f64[P], best u16[P].  batch/procs stay on the host for
    decoding winners.
    """

    def __init__(self, packed, build_index: bool = True):
        require_cuda()
        self.packed = packed
        inter = np.empty(2 * packed.n_points, dtype=np.float64)
        inter[0::2] = packed.tp
        inter[1::2] = packed.lat
        self.pts = to_device(inter, pad=2)
        self.seg_start = to_device(packed.seg_start.astype(np.int64))
        self.seg_count = to_device(packed.seg_count.astype(np.int32))
        self._finish(build_index)

    @classmethod
    def prepare_on_device(cls, raw, memory_map=None, single_process: bool = False, build_index: bool = True):
        """prepare_tables (pipeline.py:70-80) on the GPU from raw packed tables
        (tables.pack_raw): memory filter + single-process restriction as kernel
        predicates (csrc/prepare.cu)."""
        from .profiles import check_memory_map
        from .tables import PackedTables
        torch = require_cuda()
        mm = check_memory_map(memory_map)
        caps = np.array([mm[s] for s in (1, 2, 3, 4, 7)], dtype=np.float64)
        P = raw.n_points
        d = [to_device(a) for a in (raw.tp, raw.lat, raw.mem, raw.procs.astype(np.int32),
                                    raw.seg_start.astype(np.int64), raw.seg_count.astype(np.int32))] \
            if P else None
        self = cls.__new__(cls)
        self.pts = torch.zeros(2 * max(P, 1) + 2, dtype=torch.float64, device="cuda")
        self.seg_start = torch.zeros(max(raw.n_tables * 5, 1), dtype=torch.int64, device="cuda")
        self.seg_count = torch.zeros(max(raw.n_tables * 5, 1), dtype=torch.int32, device="cuda")
        src = torch.zeros(max(P, 1), dtype=torch.int32, device="cuda")
        n_out = C.c_int64(0)
        if P:
            R = ParvaRawTables(*[t.data_ptr() for t in d], raw.n_tables, P)
            check(lib().parva_prepare_tables(C.byref(R), caps.ctypes.data_as(C.c_void_p), C.c_int32(int(single_process)),
                                             ptr(self.pts), ptr(self.seg_start), ptr(self.seg_count), ptr(src),
                                             C.byref(n_out), stream_handle()), "parva_prepare_tables")
        n = int(n_out.value)
        idx = src[:n].cpu().numpy()
        self.packed = PackedTables(names=list(raw.names), tp=raw.tp[idx], lat=raw.lat[idx], batch=raw.batch[idx],
                                   procs=raw.procs[idx], seg_start=self.seg_start[:raw.n_tables * 5].cpu().numpy(),
                                   seg_count=self.seg_count[:raw.n_tables * 5].cpu().numpy())
        self._finish(build_index)
        return self

    def _finish(self, build_index: bool):
        import torch
        packed = self.packed
        self.max_seg_points = int(packed.seg_count.max(initial=0))
        self.struct = ParvaTables(self.pts.data_ptr(), self.seg_start.data_ptr(),
                                  self.seg_count.data_ptr(), packed.n_tables, packed.n_points, self.max_seg_points)
        self.index = None
        self.index_struct = None
        if build_index and packed.n_points and int(packed.seg_count.max(initial=0)) <= 4096:
            self.lat_sorted = torch.empty(packed.n_points + 2, dtype=torch.float64, device="cuda")
            self.best = torch.empty(packed.n_points + 8, dtype=torch.int16, device="cuda")
            self.idx_tp = torch.empty(packed.n_points + 2, dtype=torch.float64, device="cuda")
            self.index_struct = ParvaIndex(self.lat_sorted.data_ptr(), self.best.data_ptr(), self.idx_tp.data_ptr())
            check(lib().parva_build_index(C.byref(self.struct), C.byref(self.index_struct), stream_handle()),
                  "parva_build_index")
            self.index = True

    @property
    def n_tables(self) -> int:
        return self.packed.n_tables


class _LRU:
    def __init__(self, n=8):
        self.n = n
        self.d: OrderedDict = OrderedDict()

    def get(self, key, make):
        if key in self.d:
            self.d.move_to_end(key)
            return self.d[key][1]
        val = make()
        self.d[key] = val
        if len(self.d) > self.n:
            self.d.popitem(last=False)
        return val[1]


_TABLE_CACHE = _LRU(8)


_RAW_CACHE = _LRU(8)


def device_tables_for(tables, memory_map=None, single_process=False, prepared=False) -> DeviceTables:
    """Cached DeviceTables for a {model: ProfileTable} mapping (or sequence).

    The raw points are packed once per table set; the preparation for given
    options (memory map, single process) runs on the GPU (csrc/prepare.cu)."""
    from .tables import pack_raw
    items = list(tables.items()) if hasattr(tables, "items") else [(t.model_id, t) for t in tables]
    mm = None if memory_map is None else tuple(sorted((int(k), float(v)) for k, v in dict(memory_map).items()))
    tkey = tuple((n, id(t)) for n, t in items)
    key = (tkey, mm, bool(single_process), bool(prepared))

    def make_raw():
        return ([t for _, t in items], pack_raw(dict(items) if hasattr(tables, "items") else [t for _, t in items]))

    def make():
        raw = _RAW_CACHE.get(tkey, make_raw)
        if prepared:
            return ([t for _, t in items], DeviceTables(raw))
        return ([t for _, t in items], DeviceTables.prepare_on_device(raw, memory_map, single_process))

    return _TABLE_CACHE.get(key, make)


__all__ = ["CONFIG_DTYPE", "PLAN_DTYPE", "DeviceTables", "device_tables_for", "lib", "load_library",
           "require_cuda", "EXPORTS"]
