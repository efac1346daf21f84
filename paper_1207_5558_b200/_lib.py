"""ctypes binding of the C ABI in include/slsht_cuda.h (libslsht_cuda.so, built in-tree).

The library is the product: there is no Python or CPU fallback. Loading fails loudly when
the shared object is missing, and every compute entry point returns SLSHT_ERR_DEVICE when no
sm_100a device is present.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libslsht_cuda.so"

SLSHT_OK = 0
SLSHT_ERR_VALIDATION = 2
SLSHT_ERR_NUMERIC = 3
SLSHT_ERR_DEVICE = 4
DIGEST_WIDTH = 8

# every symbol include/slsht_cuda.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "slsht_cuda_plan_create",
    "slsht_cuda_plan_destroy",
    "slsht_cuda_last_error",
    "slsht_cuda_forward",
    "slsht_cuda_forward_scatter",
    "slsht_cuda_forward_device",
    "slsht_cuda_forward_capture",
    "slsht_cuda_device_output",
    "slsht_cuda_volume_elems",
    "slsht_cuda_computed_count",
    "slsht_cuda_emitted_count",
    "slsht_cuda_stream",
    "slsht_cuda_launch_count",
    "slsht_cuda_stage_times",
    "slsht_cuda_set_profiling",
    "slsht_cuda_kernel_time",
    "slsht_cuda_delta_tables",
    "slsht_cuda_modulated",
    "slsht_cuda_inverse",
    "slsht_cuda_eigenfunction_window",
    "slsht_cuda_forward_direct",
    "slsht_cuda_copy_sink",
    "slsht_cuda_shard_bounds",
    "slsht_cuda_device_count",
    "slsht_cuda_theta_weights",
    "slsht_cuda_beta_weights",
    "slsht_cuda_legendre_rows",
    "slsht_cuda_gauss_legendre_half",
]


class slsht_cuda_desc(C.Structure):
    _fields_ = [
        ("L_f", C.c_int),
        ("L_h", C.c_int),
        ("lmax", C.c_int),
        ("real_mode", C.c_int),
        ("emit_negative_m", C.c_int),
        ("device", C.c_int),
        ("l_begin", C.c_int),
        ("l_end", C.c_int),
        ("materialize", C.c_int),
        ("n_devices", C.c_int),
        ("ring_bytes", C.c_longlong),
        ("stream", C.c_void_p),
        ("devices", C.POINTER(C.c_int)),
    ]


class slsht_copy_target(C.Structure):
    _fields_ = [
        ("base", C.c_void_p),
        ("first_index", C.c_longlong),
        ("count", C.c_longlong),
        ("volume_elems", C.c_longlong),
        ("delivered", C.c_longlong),
        ("dropped", C.c_longlong),
    ]


SINK = C.CFUNCTYPE(None, C.c_int, C.c_int, C.POINTER(C.c_double), C.c_void_p)
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)

_lib = None


def load() -> C.CDLL:
    """Load libslsht_cuda.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `make -C {HERE}` or __graft_entry__.build(); "
            "the SLSHT engine has no CPU fallback")
    lib = C.CDLL(str(LIB_PATH))
    lib.slsht_cuda_plan_create.argtypes = [C.POINTER(slsht_cuda_desc), C.POINTER(C.c_void_p)]
    lib.slsht_cuda_plan_create.restype = C.c_int
    lib.slsht_cuda_plan_destroy.argtypes = [C.c_void_p]
    lib.slsht_cuda_plan_destroy.restype = None
    lib.slsht_cuda_last_error.argtypes = [C.c_void_p]
    lib.slsht_cuda_last_error.restype = C.c_char_p
    lib.slsht_cuda_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.slsht_cuda_forward.restype = C.c_int
    lib.slsht_cuda_forward_scatter.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                               C.c_longlong, C.c_int, C.POINTER(C.c_longlong)]
    lib.slsht_cuda_forward_scatter.restype = C.c_int
    lib.slsht_cuda_forward_device.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                              C.c_void_p, C.c_int, C.c_int]
    lib.slsht_cuda_forward_device.restype = C.c_int
    lib.slsht_cuda_forward_capture.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                               C.c_int, _ip, _ip, C.c_void_p]
    lib.slsht_cuda_forward_capture.restype = C.c_int
    lib.slsht_cuda_device_output.argtypes = [C.c_void_p]
    lib.slsht_cuda_device_output.restype = C.c_void_p
    for name in ("slsht_cuda_volume_elems", "slsht_cuda_computed_count",
                 "slsht_cuda_emitted_count", "slsht_cuda_launch_count"):
        getattr(lib, name).argtypes = [C.c_void_p]
        getattr(lib, name).restype = C.c_longlong
    lib.slsht_cuda_stream.argtypes = [C.c_void_p]
    lib.slsht_cuda_stream.restype = C.c_void_p
    lib.slsht_cuda_stage_times.argtypes = [C.c_void_p, _dp, C.c_int]
    lib.slsht_cuda_stage_times.restype = C.c_int
    lib.slsht_cuda_set_profiling.argtypes = [C.c_void_p, C.c_int]
    lib.slsht_cuda_set_profiling.restype = C.c_int
    lib.slsht_cuda_kernel_time.argtypes = [C.c_void_p, _dp]
    lib.slsht_cuda_kernel_time.restype = C.c_int
    lib.slsht_cuda_delta_tables.argtypes = [C.c_int, C.c_int, _dp]
    lib.slsht_cuda_delta_tables.restype = C.c_int
    lib.slsht_cuda_theta_weights.argtypes = [C.c_int, C.c_int, _dp]
    lib.slsht_cuda_theta_weights.restype = C.c_int
    lib.slsht_cuda_beta_weights.argtypes = [C.c_int, C.c_int, _dp]
    lib.slsht_cuda_beta_weights.restype = C.c_int
    lib.slsht_cuda_legendre_rows.argtypes = [C.c_int, C.c_int, C.c_int, _dp, C.c_int, _dp]
    lib.slsht_cuda_legendre_rows.restype = C.c_int
    lib.slsht_cuda_gauss_legendre_half.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp]
    lib.slsht_cuda_gauss_legendre_half.restype = C.c_int
    lib.slsht_cuda_eigenfunction_window.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int,
                                                    C.c_int, C.c_void_p, _dp]
    lib.slsht_cuda_eigenfunction_window.restype = C.c_int
    lib.slsht_cuda_forward_direct.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p,
                                              C.c_int, C.c_void_p, C.c_longlong, C.c_void_p]
    lib.slsht_cuda_forward_direct.restype = C.c_int
    lib.slsht_cuda_modulated.argtypes = [C.c_void_p, C.c_void_p, C.c_int, _ip, _ip, _dp]
    lib.slsht_cuda_modulated.restype = C.c_int
    lib.slsht_cuda_inverse.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                                       C.c_double, C.c_int, C.c_void_p]
    lib.slsht_cuda_inverse.restype = C.c_int
    lib.slsht_cuda_shard_bounds.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _ip]
    lib.slsht_cuda_shard_bounds.restype = C.c_int
    lib.slsht_cuda_device_count.argtypes = []
    lib.slsht_cuda_device_count.restype = C.c_int
    _lib = lib
    return lib
