"""ctypes declarations of libwmh.so (include/wmh.h).  Argument marshalling only."""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "libwmh_debug.so" if os.environ.get("WMH_LIB") == "debug" else "libwmh.so")
if os.environ.get("WMH_LIB_AB"):          # A/B experiments: another build of the library (scripts only)
    SO_PATH = os.path.join(_HERE, os.environ["WMH_LIB_AB"])

WMH_OK, WMH_EINVAL, WMH_EBOUND, WMH_EEMPTY, WMH_EOVERFLOW, WMH_ECUDA, WMH_ENOMEM = range(7)
WMH_DENSE, WMH_CSR = 0, 1
WMH_OPT_TIME_KERNEL = 1
WMH_OPT_TILE_BYTES = 2
WMH_OPT_TILE_BITPLANES = 4
WMH_OPT_TILE_BITSLICE = 8
WMH_OPT_VALIDATE = 16
WMH_OPT_ISGREEN_BINSEARCH = 32
ALGOS = {"auto": 0, "simple": 1, "tiled": 2, "index": 3}
STATUS_NAMES = {0: "WMH_OK", 1: "WMH_EINVAL", 2: "WMH_EBOUND", 3: "WMH_EEMPTY", 4: "WMH_EOVERFLOW",
                5: "WMH_ECUDA", 6: "WMH_ENOMEM"}

# Every symbol include/wmh.h declares (tests check the .so exports all of them).
EXPORTS = ["wmh_colmax", "wmh_prepare", "wmh_layout_info", "wmh_layout_digest", "wmh_layout_tables", "wmh_layout_free",
           "wmh_hash", "wmh_hash_ex", "wmh_hash_host", "wmh_collide", "wmh_last_error", "wmh_version",
           "wmh_kernel_launches", "wmh_last_kernel_ms", "wmh_quantize", "wmh_scale_objective", "wmh_lsh_build",
           "wmh_lsh_query", "wmh_lsh_free", "wmh_hasher_create", "wmh_hasher_run", "wmh_hasher_free",
           "wmh_check_rows", "wmh_collide2", "wmh_choose_scale", "wmh_empty_launch"]


class WmhRows(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("n_rows", ctypes.c_int64), ("dim", ctypes.c_int64),
                ("dense", ctypes.c_void_p), ("row_ptr", ctypes.c_void_p), ("col", ctypes.c_void_p),
                ("val", ctypes.c_void_p), ("nnz", ctypes.c_int64), ("weight_bytes", ctypes.c_int32)]


class WmhHashOpts(ctypes.Structure):
    _fields_ = [("algo", ctypes.c_int32), ("chunk", ctypes.c_int32), ("algo_used", ctypes.c_int32),
                ("horizon", ctypes.c_uint32), ("flags", ctypes.c_uint32), ("plan_out", ctypes.c_void_p),
                ("tile_used", ctypes.c_int32), ("reserved", ctypes.c_int32 * 3)]


class WmhError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    """Load the in-tree libwmh.so.  Raises (never falls back) when it is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(SO_PATH):
            raise RuntimeError(f"libwmh.so not built ({SO_PATH}); run __graft_entry__.build() "
                               "or python paper_1602_08393_b200/build.py")
        L = ctypes.CDLL(SO_PATH)
        vp, i64, u64, u32, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int32
        rows_p = ctypes.POINTER(WmhRows)
        st = ctypes.c_int
        proto = {
            "wmh_colmax": (st, [rows_p, vp, vp]),
            "wmh_prepare": (st, [vp, i64, rows_p, ctypes.POINTER(vp), vp]),
            "wmh_layout_info": (st, [vp, ctypes.POINTER(i64), ctypes.POINTER(u64), ctypes.POINTER(u32),
                                     ctypes.POINTER(u32)]),
            "wmh_layout_tables": (st, [vp, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp)]),
            "wmh_layout_digest": (st, [vp, ctypes.POINTER(u64)]),
            "wmh_layout_free": (None, [vp]),
            "wmh_hash": (st, [vp, rows_p, u64, u32, u32, i32, vp, vp, vp]),
            "wmh_hash_ex": (st, [vp, rows_p, u64, u32, u32, i32, vp, vp, ctypes.POINTER(WmhHashOpts), vp]),
            "wmh_hash_host": (st, [vp, rows_p, u64, u32, u32, i32, vp, vp]),
            "wmh_collide": (st, [vp, i32, u32, i64, vp, i64, vp, vp, i32, vp]),
            "wmh_collide2": (st, [vp, i64, vp, i64, i32, u32, vp, i64, vp, vp, i32, vp]),
            "wmh_check_rows": (st, [vp, rows_p, vp]),
            "wmh_empty_launch": (st, [vp]),
            "wmh_choose_scale": (st, [rows_p, ctypes.POINTER(ctypes.c_float), i32, ctypes.POINTER(i32), vp]),
            "wmh_last_error": (ctypes.c_char_p, []),
            "wmh_version": (ctypes.c_char_p, []),
            "wmh_kernel_launches": (ctypes.c_uint64, []),
            "wmh_last_kernel_ms": (st, [ctypes.POINTER(ctypes.c_float)]),
            "wmh_quantize": (st, [vp, i64, ctypes.c_float, vp, vp]),
            "wmh_lsh_build": (st, [vp, i32, u32, i64, u32, u32, ctypes.POINTER(vp), vp]),
            "wmh_lsh_query": (st, [vp, vp, i64, u32, vp, vp, vp]),
            "wmh_lsh_free": (None, [vp]),
            "wmh_hasher_create": (st, [vp, u64, u32, u32, u32, ctypes.POINTER(vp), vp]),
            "wmh_hasher_run": (st, [vp, rows_p, i32, vp, vp, vp]),
            "wmh_hasher_free": (None, [vp]),
            "wmh_scale_objective": (st, [rows_p, ctypes.POINTER(ctypes.c_float), i32, ctypes.POINTER(u64), vp]),
        }
        for name, (res, args) in proto.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
        return L


def check(status: int) -> None:
    if status != WMH_OK:
        raise WmhError(status, load().wmh_last_error().decode(errors="replace"))
