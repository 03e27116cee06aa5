"""ctypes binding of the C ABI in include/hsewald_b200.h (libhsewald_b200.so).

This is the only way the package reaches the GPU.  There is no CPU fallback:
if the shared library is missing or no sm_100-class device is present, every
entry point raises :class:`~.errors.DeviceError`.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import DeviceError, raise_for_status

# HSEWALD_LIB: alternative build of the same library (kernel-variant A/B runs in tools/)
_HERE = os.path.dirname(os.path.abspath(__file__))
# HSEWALD_CHECKED=1: the checked build (device-side bounds / ring-index checks, hs_debug_checks)
LIB_PATH = os.environ.get("HSEWALD_LIB") or os.path.join(
    _HERE, "libhsewald_b200_checked.so" if os.environ.get("HSEWALD_CHECKED") == "1" else "libhsewald_b200.so")

HS_MEM_DEVICE, HS_MEM_HOST = 0, 1
KIND_ID = {"stokeslet": 0, "stresslet": 1, "rotlet": 2, "mixed": 3}
GEOM_ID = {"free": 0, "half": 1}
TABLE_ID = {"harmonic": 0, "biharmonic": 1}

_i64p = C.POINTER(C.c_int64)
_dp = C.POINTER(C.c_double)


class HsParams(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("geometry", C.c_int), ("L", C.c_double),
        ("xi", C.c_double), ("rc", C.c_double), ("M", C.c_int64), ("P", C.c_int64),
        ("h", C.c_double), ("eta", C.c_double), ("origin", C.c_double * 3),
        ("dims", C.c_int64 * 3), ("padded", C.c_int64 * 3), ("n", C.c_int64),
        ("n_targets", C.c_int64), ("targets_are_sources", C.c_int),
    ]


class HsSlab(C.Structure):
    _fields_ = [
        ("rank", C.c_int64), ("world", C.c_int64), ("y0", C.c_int64), ("y1", C.c_int64),
        ("kz0", C.c_int64), ("kz1", C.c_int64), ("kz_split", C.c_int64 * 65), ("y_split", C.c_int64 * 65),
    ]


MAX_SLAB_RANKS = 64

# (name, restype, argtypes)
_SIGS = [
    ("hs_ctx_create", C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    ("hs_ctx_destroy", C.c_int, [C.c_void_p]),
    ("hs_ctx_set_stream", C.c_int, [C.c_void_p, C.c_void_p]),
    ("hs_last_error", C.c_char_p, []),
    ("hs_ctx_launch_count", C.c_int64, [C.c_void_p]),
    ("hs_cell_dims", C.c_int, [C.c_double, _dp, _dp, _i64p, _dp]),
    ("hs_cell_list", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_double, _dp, _dp, C.c_void_p,
                               C.c_void_p, C.c_int]),
    ("hs_spread", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, _dp, C.c_double, _i64p,
                            C.c_int, C.c_double, C.c_double, C.c_void_p, C.c_int]),
    ("hs_gather", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int64, _dp, C.c_double, _i64p,
                            C.c_int, C.c_double, C.c_double, C.c_void_p, C.c_int]),
    ("hs_precompute_greens", C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_double, _i64p, _i64p, _i64p,
                                       C.c_void_p, C.c_int]),
    ("hs_plan_create", C.c_int, [C.c_void_p, C.POINTER(HsParams), C.POINTER(C.c_void_p)]),
    ("hs_plan_destroy", C.c_int, [C.c_void_p]),
    ("hs_plan_bytes", C.c_int64, [C.c_void_p]),
    ("hs_plan_set_table", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int]),
    ("hs_plan_build_tables", C.c_int, [C.c_void_p, _i64p, C.c_double, _i64p]),
    ("hs_plan_execute", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, _dp]),
    ("hs_plan_real_parts", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    ("hs_plan_fft_counts", C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("hs_plan_pair_audit", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_int]),
    ("hs_plan_create_slab", C.c_int, [C.c_void_p, C.POINTER(HsParams), C.POINTER(HsSlab), C.POINTER(C.c_void_p)]),
    ("hs_slab_sizes", C.c_int, [C.c_void_p, _i64p]),
    ("hs_slab_begin", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                C.c_void_p]),
    ("hs_slab_forward", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("hs_slab_kspace", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("hs_slab_backward", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("hs_slab_finish", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, _dp]),
    ("hs_slab_forward_range", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    ("hs_slab_kspace_part", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    ("hs_slab_backward_range", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    ("hs_direct_sum", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    ("hs_debug_checks", C.c_int, [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_int]),
]
EXPORTED = [s[0] for s in _SIGS]

_lib = None
_lib_lock = threading.Lock()


def load_library():
    """Load and type the shared library (no device needed)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DeviceError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                                  "(the package has no CPU fallback)")
            lib = C.CDLL(LIB_PATH)
            for name, res, args in _SIGS:
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(status: int) -> None:
    if status:
        msg = load_library().hs_last_error().decode(errors="replace")
        raise_for_status(status, msg)


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def i64ptr(a: np.ndarray):
    return a.ctypes.data_as(_i64p)


def vec3(values, ctype=C.c_double):
    return (ctype * 3)(*values)


class Context:
    """One hs_ctx per (process, device); bound to torch's current stream when torch is used."""

    _instances: dict = {}
    _lock = threading.Lock()

    def __init__(self, device: int = 0):
        self.lib = load_library()
        self.device = device
        h = C.c_void_p()
        check(self.lib.hs_ctx_create(device, C.byref(h)))
        self.handle = h
        self._stream = None

    @classmethod
    def get(cls, device: int | None = None) -> "Context":
        if device is None:
            device = int(os.environ.get("HSEWALD_DEVICE", "0"))
        with cls._lock:
            ctx = cls._instances.get(device)
            if ctx is None:
                ctx = cls(device)
                cls._instances[device] = ctx
            return ctx

    def bind_stream(self, stream_ptr: int | None) -> None:
        if stream_ptr != self._stream:
            check(self.lib.hs_ctx_set_stream(self.handle, C.c_void_p(stream_ptr or 0)))
            self._stream = stream_ptr

    def bind_torch_stream(self) -> None:
        import torch
        self.bind_stream(torch.cuda.current_stream(self.device).cuda_stream)

    def launches(self) -> int:
        return int(self.lib.hs_ctx_launch_count(self.handle))


def debug_checks(reset: bool = True) -> dict:
    """Device-side check results of the checked build (hs_debug_checks): failures since the last
    reset and the first failing (translation unit, source line)."""
    lib = load_library()
    first, count = C.c_uint64(), C.c_uint64()
    check(lib.hs_debug_checks(C.byref(first), C.byref(count), 1 if reset else 0))
    tu = {1: "pair.cu", 2: "gridding.cu", 3: "fft.cu", 4: "plan.cu", 5: "sort.cu", 6: "kspace.cu",
          7: "cell_list.cu", 8: "api.cu"}
    f = first.value
    return {"failures": int(count.value), "first": None if not f else f"{tu.get(f >> 32, f >> 32)}:{f & 0xffffffff}"}

