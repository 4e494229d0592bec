"""ctypes binding of libheomb200.so (the C ABI declared in include/heom_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no CPU fallback: if the library or a CUDA device is missing, every
compute entry point raises.  ctypes releases the GIL around each call, so
independent handles can be driven from Python threads concurrently (the
reference relies on numba's nogil for the same, cli.py:279-284).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_NAME = "libheomb200.so"
#: HEOM_B200_LIB selects another build of the same library (the test-suite's
#: bounds-checked libheomb200_checked.so); default: the in-tree release build
LIB_PATH = Path(os.environ.get("HEOM_B200_LIB") or Path(__file__).resolve().parent / LIB_NAME)

HB_OK, HB_ERR_ARG, HB_ERR_CUDA, HB_DIVERGED, HB_HARDCAP, HB_ERR_RANGE = 0, 1, 2, 3, 4, 5
HB_STOP_NONE, HB_STOP_T_END, HB_STOP_RESIDUAL = 0, 1, 2
HB_LAYOUT = {"auto": 0, "hermitian": 1, "general": 2}
HB_ORDER = {"lex": 0, "reference": 1, "lex-split": 2}
HB_KERNEL = {"auto": 0, "generic": 1}
HB_PREC = {"double": 0, "single": 1}

#: every symbol include/heom_b200.h declares (checked by the CPU test-suite)
EXPORTS = ("hb_last_error", "hb_device_count", "hb_hierarchy_size", "hb_graph_build",
           "hb_rhs", "hb_heom_rhs", "hb_add_scaled", "hb_rk4_update", "hb_max_abs2", "hb_create",
           "hb_destroy", "hb_set_rho0", "hb_set_state", "hb_pool_trim", "hb_io_bytes", "hb_run", "hb_get_records", "hb_record_count", "hb_get_state",
           "hb_get_sigma0", "hb_time_steps", "hb_launch_count", "hb_create_shard", "hb_sync",
           "hb_nccl_unique_id", "hb_nccl_init", "hb_halo_set", "hb_shard_steps",
           "hb_shard_steps_local")


class HbParams(C.Structure):
    _fields_ = [
        ("d", C.c_int), ("n_sites", C.c_int), ("kp1", C.c_int), ("n_max", C.c_int),
        ("h", C.c_void_p), ("site_of", C.c_void_p), ("decay", C.c_void_p),
        ("nu", C.c_void_p), ("a", C.c_void_p), ("b", C.c_void_p),
        ("n_sinks", C.c_int), ("sink_nterms", C.c_void_p), ("sink_rate", C.c_void_p),
        ("sink_pos", C.c_void_p), ("n_site_pos", C.c_int), ("site_pos", C.c_void_p),
        ("d_full", C.c_int), ("block_full", C.c_void_p), ("sink_full", C.c_void_p),
        ("dt", C.c_double), ("has_t_end", C.c_int), ("t_end", C.c_double),
        ("has_residual", C.c_int), ("residual", C.c_double), ("hard_cap", C.c_double),
        ("record_stride", C.c_int64), ("record_matrices", C.c_int),
        ("blowup_norm", C.c_double), ("device", C.c_int), ("layout", C.c_int),
        ("ordering", C.c_int), ("chunk_steps", C.c_int), ("kernel_variant", C.c_int),
        ("precision", C.c_int),
    ]


class HbShardTables(C.Structure):
    _fields_ = [("n_local", C.c_int), ("own_tiles", C.c_int), ("top_tile", C.c_int),
                ("root", C.c_int), ("plus", C.c_void_p), ("minus", C.c_void_p),
                ("nvec", C.c_void_p), ("groups", C.c_void_p), ("group_count", C.c_int * 4)]


class HbResult(C.Structure):
    _fields_ = [("stop_reason", C.c_int), ("layout", C.c_int), ("steps", C.c_int64),
                ("n_records", C.c_int64), ("n_tot", C.c_int64)]


_lib = None
_p = C.c_void_p
_d = C.c_double
_i = C.c_int
_i64 = C.c_int64


class NativeError(RuntimeError):
    """A CUDA-side failure (HB_ERR_CUDA) or a missing library / device."""


def lib():
    """Load libheomb200.so once (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a); "
                          "the propagator has no CPU fallback")
    L = C.CDLL(str(LIB_PATH))
    sig = {
        "hb_last_error": (C.c_char_p, []),
        "hb_device_count": (_i, []),
        "hb_hierarchy_size": (_i64, [_i, _i]),
        "hb_graph_build": (_i, [_i, _i, _i, _p, _p, _p, _p, _p]),
        "hb_rhs": (_i, [_p, _p, _i64, _i, _p, _p, _p, _p, _i, _p, _p, _d, _d, _p, _i]),
        "hb_heom_rhs": (_i, [_p, _p, _i64, _i, _p, _p, _p, _p, _i, _p, _p, _d, _d, _p, _i, _p, _p,
                             _p, _i]),
        "hb_add_scaled": (_i, [_p, _p, _p, _d, _i64, _i]),
        "hb_rk4_update": (_i, [_p, _p, _p, _p, _p, _d, _i64, _i]),
        "hb_max_abs2": (_i, [_p, _i64, C.POINTER(_d), _i]),
        "hb_create": (_i, [C.POINTER(HbParams), C.POINTER(_p)]),
        "hb_destroy": (None, [_p]),
        "hb_set_rho0": (_i, [_p, _p, _p]),
        "hb_set_state": (_i, [_p, _p, _p]),
        "hb_pool_trim": (None, []),
        "hb_io_bytes": (None, [C.POINTER(_i64), C.POINTER(_i64)]),
        "hb_run": (_i, [_p, C.POINTER(HbResult)]),
        "hb_get_records": (_i, [_p, _p, _p, _p, _i64]),
        "hb_record_count": (_i64, [_p]),
        "hb_get_state": (_i, [_p, _p, _p]),
        "hb_get_sigma0": (_i, [_p, _p, _p]),
        "hb_time_steps": (_i, [_p, _i64, C.POINTER(_d), _p]),
        "hb_launch_count": (_i64, [_p]),
        "hb_create_shard": (_i, [C.POINTER(HbParams), C.POINTER(HbShardTables), C.POINTER(_p)]),
        "hb_sync": (_i, [_p, C.POINTER(_i), C.POINTER(_i64)]),
        "hb_nccl_unique_id": (_i, [C.c_char_p]),
        "hb_nccl_init": (_i, [_p, C.c_char_p, _i, _i]),
        "hb_halo_set": (_i, [_p, _i, _p, _p, _p, _p, _p]),
        "hb_shard_steps": (_i, [_p, _i64, C.POINTER(_d)]),
        "hb_shard_steps_local": (_i, [C.POINTER(_p), _i, _i64, C.POINTER(_d)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def last_error() -> str:
    return lib().hb_last_error().decode()


def device_count() -> int:
    return int(lib().hb_device_count())


def require_device(device: int = 0) -> None:
    n = device_count()
    if n == 0:
        raise NativeError("no CUDA device visible: the B200 HEOM propagator has no CPU path")
    if not 0 <= device < n:
        raise ValueError(f"device {device} out of range (found {n})")


def check(rc: int, what: str = "") -> None:
    """Map a C return code to the reference's exception types."""
    if rc == HB_OK:
        return
    msg = last_error()
    if rc in (HB_ERR_ARG, HB_ERR_RANGE):
        raise ValueError(msg)
    raise NativeError(f"{what}: {msg}" if what else msg)


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def io_bytes():
    """(host->device, device->host) bytes the library has copied so far."""
    a, b = _i64(), _i64()
    lib().hb_io_bytes(C.byref(a), C.byref(b))
    return int(a.value), int(b.value)
