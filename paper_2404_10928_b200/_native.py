"""ctypes binding of ``libpactgpu.so`` (the C ABI declared in include/pactgpu.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).  There is
no CPU fallback: if the library is missing or no CUDA device is visible, every device
entry point raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import sys
import threading

_PKG = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_PKG)
LIB_PATH = os.environ.get("PK_LIB") or os.path.join(_PKG, "libpactgpu.so")  # PK_LIB: experiment builds
SOURCES = [
    os.path.join(_PKG, "csrc", "pactgpu.cu"),
    os.path.join(_PKG, "csrc", "pk_kernels.cuh"),
    os.path.join(_PKG, "csrc", "pk_common.cuh"),
    os.path.join(_PKG, "csrc", "pk_freq.cuh"),
    os.path.join(_PKG, "csrc", "pk_dense.cuh"),
    os.path.join(_ROOT, "include", "pactgpu.h"),
]

PK_OK = 0
PK_ERR_INVALID = -1
PK_ERR_CUDA = -2
PK_ERR_UNSUPPORTED = -3
PK_ERR_GEOMETRY = -4
PK_F32 = 0
PK_F64 = 1
PK_PEER_MAX = 8
PK_PEER_HANDLE_BYTES = 64
STOPPED_BY = {0: "max_iterations", 1: "tolerance", 2: "divergence"}


class NativeUnavailable(RuntimeError):
    """libpactgpu.so could not be loaded (not built, or no CUDA driver)."""


class PkError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"pactgpu error {code}: {msg}")
        self.code = code


class GeometryDesc(ctypes.Structure):
    _fields_ = [
        ("nx", ctypes.c_int32),
        ("ny", ctypes.c_int32),
        ("pixel_x", ctypes.POINTER(ctypes.c_double)),
        ("pixel_y", ctypes.POINTER(ctypes.c_double)),
        ("sensors", ctypes.c_int32),
        ("sensor_xy", ctypes.POINTER(ctypes.c_double)),
        ("sensor_begin", ctypes.c_int32),
        ("sensor_end", ctypes.c_int32),
        ("samples", ctypes.c_int32),
        ("c", ctypes.c_double),
        ("dt", ctypes.c_double),
        ("dtype", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("frames", ctypes.c_int32),
        ("concurrency", ctypes.c_int32),
        ("sensor_list", ctypes.POINTER(ctypes.c_int32)),
        ("sensor_list_len", ctypes.c_int32),
    ]


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("local_sensors", ctypes.c_int32),
        ("pixels", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("may_truncate", ctypes.c_int32),
        ("c_dt", ctypes.c_double),
        ("weight", ctypes.c_double),
        ("bp_tile", ctypes.c_int32),
        ("bp_window", ctypes.c_int32),
        ("bp_chunk", ctypes.c_int32),
        ("bp_buffers", ctypes.c_int32),
        ("fp_tile", ctypes.c_int32),
        ("fp_window", ctypes.c_int32),
        ("fp_bits", ctypes.c_int32),
        ("device_bytes", ctypes.c_int64),
        ("frames", ctypes.c_int32),
        ("bp_split", ctypes.c_int32),
        ("symmetric", ctypes.c_int32),
    ]


class DenseInfo(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.c_int64),
        ("cols", ctypes.c_int64),
        ("dtype", ctypes.c_int32),
        ("complex_entries", ctypes.c_int32),
        ("fused", ctypes.c_int32),
        ("splits", ctypes.c_int32),
        ("device_bytes", ctypes.c_int64),
    ]


class SolverParams(ctypes.Structure):
    _fields_ = [
        ("alpha", ctypes.c_double),
        ("beta", ctypes.c_double),
        ("step", ctypes.c_double),
        ("tv_epsilon", ctypes.c_double),
        ("tolerance", ctypes.c_double),
        ("iterations", ctypes.c_int32),
        ("nonneg", ctypes.c_int32),
    ]


# (name, restype, argtypes) -- every symbol include/pactgpu.h declares
_vp = ctypes.c_void_p
_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
SYMBOLS = [
    ("pk_plan_create", ctypes.c_int, [ctypes.POINTER(GeometryDesc), ctypes.POINTER(_vp)]),
    ("pk_plan_destroy", ctypes.c_int, [_vp]),
    ("pk_plan_get_info", ctypes.c_int, [_vp, ctypes.POINTER(PlanInfo)]),
    ("pk_matvec", ctypes.c_int, [_vp, _vp, _vp, _vp]),
    ("pk_adjoint_matvec", ctypes.c_int, [_vp, _vp, _vp, ctypes.c_double, _vp]),
    ("pk_reconstruct", ctypes.c_int, [_vp, ctypes.POINTER(SolverParams), _vp, _vp, _vp, _vp, _vp]),
    ("pk_reconstruct_host", ctypes.c_int,
     [_vp, ctypes.POINTER(SolverParams), _dp, _dp, _dp, _ip, _vp]),
    ("pk_reconstruct_host_async", ctypes.c_int,
     [_vp, ctypes.POINTER(SolverParams), _dp, _dp, _dp, _ip, _vp]),
    ("pk_grad_update", ctypes.c_int, [_vp, ctypes.POINTER(SolverParams), _vp, _vp, _vp, _vp, _vp]),
    ("pk_residual", ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    ("pk_adjoint_residual", ctypes.c_int, [_vp, _vp, ctypes.c_double, _vp]),
    ("pk_index_dump", ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_int32, _vp, _vp, _vp]),
    ("pk_delay_census_f32", ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _vp, _vp, _vp]),
    ("pk_peer_handle", ctypes.c_int, [_vp, ctypes.c_char_p]),
    ("pk_peer_connect", ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_char_p]),
    ("pk_peer_buffer", ctypes.c_int, [_vp, ctypes.c_int32, ctypes.POINTER(_vp)]),
    ("pk_peer_grad_update", ctypes.c_int,
     [_vp, ctypes.POINTER(SolverParams), _vp, ctypes.c_int32, _vp, _vp, _vp]),
    ("pk_peer_status", ctypes.c_int, [_vp, _ip]),
    ("pk_freq_matvec", ctypes.c_int, [_vp, ctypes.c_int32, _vp, _vp, _vp]),
    ("pk_freq_adjoint", ctypes.c_int, [_vp, ctypes.c_int32, _vp, _vp, ctypes.c_double, _vp]),
    ("pk_profile_iterations", ctypes.c_int,
     [_vp, ctypes.POINTER(SolverParams), _vp, ctypes.POINTER(ctypes.c_float), _ip, _vp]),
    ("pk_profile_stages", ctypes.c_int,
     [_vp, ctypes.POINTER(SolverParams), _vp, ctypes.POINTER(ctypes.c_float), _ip, _vp]),
    ("pk_measure_fp32_peak", ctypes.c_int, [ctypes.c_int32, _dp]),
    ("pk_dense_create", ctypes.c_int,
     [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(_vp)]),
    ("pk_dense_destroy", ctypes.c_int, [_vp]),
    ("pk_dense_get_info", ctypes.c_int, [_vp, ctypes.POINTER(DenseInfo)]),
    ("pk_dense_set_entries", ctypes.c_int, [_vp, _vp, ctypes.c_int32, _vp]),
    ("pk_dense_from_plan", ctypes.c_int, [_vp, _vp, _vp]),
    ("pk_dense_matvec", ctypes.c_int, [_vp, _vp, ctypes.c_int32, _vp, _vp]),
    ("pk_dense_adjoint", ctypes.c_int, [_vp, _vp, ctypes.c_int32, _vp, ctypes.c_double, _vp]),
    ("pk_dense_matmat", ctypes.c_int, [_vp, ctypes.c_int32, _vp, _vp, _vp]),
    ("pk_dense_rmatmat", ctypes.c_int, [_vp, ctypes.c_int32, _vp, _vp, _vp]),
    ("pk_dense_reconstruct", ctypes.c_int,
     [_vp, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(SolverParams), _vp, _vp, _vp, _vp, _vp]),
    ("pk_last_error", ctypes.c_char_p, []),
    ("pk_version", ctypes.c_int, []),
]

_lib = None
_lock = threading.Lock()


def nvcc_command(out: str = LIB_PATH) -> list[str]:
    """The in-tree build of the C ABI library for sm_100a."""
    return [
        "nvcc",
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-O3", "-lineinfo", "-std=c++17",
        "-I", os.path.join(_ROOT, "include"),
        "-shared", "-Xcompiler", "-fPIC", "-lpthread",
        "-o", out,
        os.path.join(_PKG, "csrc", "pactgpu.cu"),
    ]


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libpactgpu.so in-tree (cross-compiles without a GPU)."""
    stale = not os.path.exists(LIB_PATH) or any(
        os.path.getmtime(s) > os.path.getmtime(LIB_PATH) for s in SOURCES if os.path.exists(s)
    )
    if force or stale:
        tmp = LIB_PATH + ".tmp"
        r = subprocess.run(nvcc_command(tmp), capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
        os.replace(tmp, LIB_PATH)
        if verbose:
            print(r.stderr, file=sys.stderr)
    return LIB_PATH


def load() -> ctypes.CDLL:
    """Load the library and bind every C-ABI symbol (no GPU needed to load)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} is missing; run __graft_entry__.build() (there is no CPU fallback)"
            )
        try:
            L = ctypes.CDLL(LIB_PATH)
        except OSError as e:  # pragma: no cover - depends on the driver stack
            raise NativeUnavailable(f"cannot load {LIB_PATH}: {e}") from e
        for name, res, args in SYMBOLS:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
        return L


def check(rc: int):
    if rc != PK_OK:
        msg = load().pk_last_error().decode(errors="replace")
        if rc == PK_ERR_INVALID or rc == PK_ERR_GEOMETRY:
            # the reference raises ValueError (GeometryError is a ValueError)
            raise ValueError(msg)
        raise PkError(rc, msg)


def last_error() -> str:
    return load().pk_last_error().decode(errors="replace")
