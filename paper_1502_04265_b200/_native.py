"""ctypes binding of the C-ABI in include/piecy_b200.h.

The product path has no CPU fallback: if the shared library is missing or a
call fails, this module raises.  Device buffers are torch CUDA tensors; only
raw pointers and the current CUDA stream cross the boundary.
"""

from __future__ import annotations

import ctypes
import os

from . import _build

_lib = None

c_i32, c_i64, c_f64, c_vp = ctypes.c_int, ctypes.c_longlong, ctypes.c_double, ctypes.c_void_p
P_i64 = ctypes.POINTER(c_i64)
P_i32 = ctypes.POINTER(c_i32)
P_f64 = ctypes.POINTER(c_f64)

_SIGS = {
    "pcy_last_error": (ctypes.c_char_p, []),
    # engine (include/piecy_b200.h)
    "pcy_engine_create": (c_i32, [c_i32, c_i32, c_i64, c_i64, c_i64, ctypes.POINTER(c_vp)]),
    "pcy_engine_destroy": (c_i32, [c_vp]),
    "pcy_engine_insert": (c_i32, [c_vp, c_vp, c_i32, c_i64, c_vp, c_i64, c_vp, P_i64, P_i32]),
    "pcy_engine_stats": (c_i32, [c_vp, P_i64, P_f64, P_i64, P_i32, c_vp]),
    "pcy_engine_features": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, P_i64, c_vp]),
    "pcy_engine_extract": (c_i32, [c_vp, c_vp, c_vp, c_i64, P_i64, c_vp]),
    "pcy_engine_counters": (c_i32, [c_vp, c_vp]),
    "pcy_engine_counters_total": (c_i32, [c_vp]),
    "pcy_engine_work": (c_i32, [c_vp, c_vp]),
    # instrumentation
    "pcy_launch_count": (c_i64, []),
    "pcy_prof_enable": (c_i32, [c_i32]),
    "pcy_prof_reset": (c_i32, []),
    "pcy_prof_read": (c_i32, [c_i32, P_f64, P_i64, P_i64]),
    # tensor-core distance contraction (test entry)
    "pcy_tc_dots_f64": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_i64, c_i32, c_i32, c_vp, P_f64, c_vp]),
}

PCY_ENONFINITE = -2   # include/piecy_b200.h error codes

PROF_SLOTS = {"resolve": 0, "chain": 1, "reattach": 2, "seed": 3, "lloyd": 4, "gemm": 5}


def engine_counters_total() -> dict:
    import numpy as np
    out = np.zeros(6, dtype=np.int64)
    lib().pcy_engine_counters_total(out.ctypes.data)
    keys = ("levels", "tc_rechecks", "demand_loads", "slow_capacity", "items", "max_depth")
    return {k: int(v) for k, v in zip(keys, out)}


def launch_count() -> int:
    return int(lib().pcy_launch_count())


def prof_enable(on: bool = True) -> None:
    lib().pcy_prof_enable(1 if on else 0)


def prof_reset() -> None:
    lib().pcy_prof_reset()


def prof_read(name: str):
    """(total ms, launches, units) accumulated for a profiled kernel."""
    ms, cnt, units = c_f64(), c_i64(), c_i64()
    lib().pcy_prof_read(PROF_SLOTS[name], ctypes.byref(ms), ctypes.byref(cnt), ctypes.byref(units))
    return ms.value, cnt.value, units.value

_OPTIONAL = set()


class NativeError(RuntimeError):
    pass


def lib():
    global _lib
    if _lib is not None:
        return _lib
    path = _build.LIB
    if not os.path.exists(path):
        if os.environ.get("PCY_AUTOBUILD", "1") == "1":
            _build.build()
        if not os.path.exists(path):
            raise NativeError(f"native library {path} is missing; run __graft_entry__.build()")
    L = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        try:
            fn = getattr(L, name)
        except AttributeError:
            if name in _OPTIONAL:
                continue
            raise NativeError(f"{path} does not export {name}")
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def register(name, res, args, optional=False):
    _SIGS[name] = (res, args)
    if optional:
        _OPTIONAL.add(name)
    if _lib is not None:   # library already loaded: bind the new symbol now
        try:
            fn = getattr(_lib, name)
        except AttributeError:
            if optional:
                return
            raise NativeError(f"{_build.LIB} does not export {name}")
        fn.restype = res
        fn.argtypes = args


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = lib().pcy_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed ({rc}): {msg}")


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int | None:
    return None if t is None else int(t.data_ptr())
