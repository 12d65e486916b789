"""ctypes binding of librobench_b200.so (the C ABI in include/robench_b200.h).

This is the reference-side binding a Python caller uses; INTEGRATION.md shows
the same binding for other hosts.  There is no fallback: if the native
library is missing or fails to load, importing the engine raises.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

from . import errors, pack

import os

LIB_PATH = Path(os.environ.get("RB_LIB") or Path(__file__).resolve().with_name("librobench_b200.so"))

RB_OK = 0
_STATUS = {
    1: errors.UnknownFunction,
    2: errors.DisabledFunction,
    3: errors.BatchTooLarge,
    4: errors.DimensionMismatch,
    5: errors.NonFiniteInput,
    6: errors.UseAfterDispose,
    7: ValueError,
    8: errors.DeviceError,
    9: errors.DeviceError,
}

EXPORTS = ("rb_initialize", "rb_dispose", "rb_func_evaluate", "rb_func_evaluatef",
           "rb_h_func_evaluate", "rb_h_func_evaluatef", "rb_last_error",
           "rb_abi_version", "rb_struct_sizes", "rb_launch_count", "rb_np_powf",
           "rb_debug_phases", "rb_uniform_population", "rb_func_evaluate_async",
           "rb_ticket_status", "rb_initialize_sharded", "rb_func_evaluate_sharded",
           "rb_sharded_ticket_status", "rb_dispose_sharded", "rb_h_func_evaluate_x64",
           "rb_func_evaluate_many", "rb_h_func_evaluate_many", "rb_graph_capture",
           "rb_graph_launch", "rb_graph_status", "rb_graph_destroy")
RB_DOUBLE, RB_SINGLE = 0, 1


class RbPack(ctypes.Structure):
    _fields_ = [
        ("dim", ctypes.c_int32), ("n_functions", ctypes.c_int32), ("functions", ctypes.c_void_p),
        ("n_members", ctypes.c_int32), ("members", ctypes.c_void_p),
        ("n_segments", ctypes.c_int32), ("segments", ctypes.c_void_p),
        ("n_groups", ctypes.c_int32), ("groups", ctypes.c_void_p),
        ("n_index", ctypes.c_int64), ("index", ctypes.c_void_p),
        ("n_values", ctypes.c_int64), ("values_f64", ctypes.c_void_p),
        ("values_f32", ctypes.c_void_p),
    ]


_lib = None


def load() -> ctypes.CDLL:
    """Load (once) the native library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH.name} not built: run `python -m paper_1407_7737_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(str(LIB_PATH))
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    lib.rb_initialize.argtypes = [ctypes.POINTER(RbPack), i64, i32, ctypes.POINTER(vp)]
    lib.rb_dispose.argtypes = [ctypes.POINTER(vp)]
    for name in ("rb_func_evaluate", "rb_func_evaluatef"):
        getattr(lib, name).argtypes = [vp, i32, vp, i64, vp, vp]
    for name in ("rb_h_func_evaluate", "rb_h_func_evaluatef"):
        getattr(lib, name).argtypes = [vp, i32, vp, i64, vp]
    for name in ("rb_initialize", "rb_dispose", "rb_func_evaluate", "rb_func_evaluatef",
                 "rb_h_func_evaluate", "rb_h_func_evaluatef"):
        getattr(lib, name).restype = i32
    lib.rb_last_error.restype = ctypes.c_char_p
    lib.rb_abi_version.restype = i32
    lib.rb_struct_sizes.argtypes = [ctypes.POINTER(ctypes.c_int64)]
    lib.rb_launch_count.restype = i64
    lib.rb_np_powf.argtypes = [vp, vp, vp, i64, vp]
    lib.rb_np_powf.restype = i32
    u64 = ctypes.c_uint64
    lib.rb_uniform_population.argtypes = [u64, u64, u64, i64, ctypes.c_double, ctypes.c_double,
                                          vp, vp, vp]
    lib.rb_uniform_population.restype = i32
    lib.rb_debug_phases.argtypes = [i32, ctypes.POINTER(ctypes.c_uint64), i32]
    lib.rb_debug_phases.restype = None
    lib.rb_func_evaluate_async.argtypes = [vp, i32, i32, vp, i64, vp, vp, ctypes.POINTER(i64)]
    lib.rb_h_func_evaluate_x64.argtypes = [vp, i32, i32, vp, i64, vp]
    lib.rb_func_evaluate_many.argtypes = [vp, i32, ctypes.POINTER(i32), ctypes.POINTER(i32),
                                          ctypes.POINTER(vp), ctypes.POINTER(i64), ctypes.POINTER(vp),
                                          vp, ctypes.POINTER(i64)]
    lib.rb_func_evaluate_many.restype = i32
    lib.rb_h_func_evaluate_many.argtypes = [vp, i32, ctypes.POINTER(i32), ctypes.POINTER(i32), vp, i64,
                                            ctypes.POINTER(vp)]
    lib.rb_h_func_evaluate_many.restype = i32
    lib.rb_h_func_evaluate_x64.restype = i32
    lib.rb_ticket_status.argtypes = [vp, i64]
    lib.rb_initialize_sharded.argtypes = [ctypes.POINTER(RbPack), i64, ctypes.POINTER(i32), i32,
                                          ctypes.POINTER(vp)]
    lib.rb_func_evaluate_sharded.argtypes = [vp, i32, i32, ctypes.POINTER(vp), i64, ctypes.POINTER(vp),
                                             ctypes.POINTER(vp), ctypes.POINTER(i64)]
    lib.rb_sharded_ticket_status.argtypes = [vp, i32, i64]
    lib.rb_dispose_sharded.argtypes = [ctypes.POINTER(vp)]
    lib.rb_graph_capture.argtypes = [vp, i32, i32, vp, i64, vp, ctypes.POINTER(vp)]
    lib.rb_graph_launch.argtypes = [vp, vp]
    lib.rb_graph_status.argtypes = [vp]
    lib.rb_graph_destroy.argtypes = [ctypes.POINTER(vp)]
    for name in ("rb_func_evaluate_async", "rb_ticket_status", "rb_initialize_sharded",
                 "rb_func_evaluate_sharded", "rb_sharded_ticket_status", "rb_dispose_sharded",
                 "rb_h_func_evaluate_x64", "rb_func_evaluate_many", "rb_h_func_evaluate_many",
                 "rb_graph_capture", "rb_graph_launch", "rb_graph_status", "rb_graph_destroy"):
        getattr(lib, name).restype = i32
    _check_layout(lib)
    _lib = lib
    return lib


def _check_layout(lib) -> None:
    sizes = (ctypes.c_int64 * 5)()
    lib.rb_struct_sizes(sizes)
    want = (pack.GROUP_DT.itemsize, pack.SEGMENT_DT.itemsize, pack.MEMBER_DT.itemsize,
            pack.FUNCTION_DT.itemsize, ctypes.sizeof(RbPack))
    if tuple(sizes) != want:
        raise ImportError(f"ABI layout mismatch: library {tuple(sizes)} vs Python {want}")


def check(status: int) -> None:
    if status != RB_OK:
        msg = load().rb_last_error().decode(errors="replace")
        raise _STATUS.get(status, errors.DeviceError)(msg)


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def make_pack(p: pack.Pack) -> RbPack:
    s = RbPack()
    s.dim, s.n_functions = p.dim, len(p.functions)
    s.functions = ptr(p.functions)
    s.n_members, s.members = len(p.members), ptr(p.members)
    s.n_segments, s.segments = len(p.segments), ptr(p.segments)
    s.n_groups, s.groups = len(p.groups), ptr(p.groups)
    s.n_index, s.index = p.index.size, ptr(p.index)
    s.n_values = p.values_f64.size
    s.values_f64, s.values_f32 = ptr(p.values_f64), ptr(p.values_f32)
    return s


def launch_count() -> int:
    return int(load().rb_launch_count())


def debug_phases(precision: str, reset: bool = True) -> list[int]:
    """Phase clock sums (diagnostic builds with -DRB_PHASE_TIMING)."""
    out = (ctypes.c_uint64 * 8)()
    load().rb_debug_phases(0 if precision == "double" else 1, out, int(reset))
    return list(out)
