"""ctypes binding of the C ABI in ``include/bed200.h`` (``_lib/libbed200.so``).

The shared library is built in-tree (``csrc/Makefile``, sm_100a only) and
loaded from ``paper_2207_04228_b200/_lib``.  There is no fallback: if the
library is missing, :func:`lib` raises, and every solve fails loudly.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libbed200.so")

BED_SUCCESS = 0
STATUS_OK = 0
STATUS_NO_CONVERGENCE = 1
STATUS_NON_FINITE = 2
STATUS_NON_SYMMETRIC = 3
STATUS_NON_POSITIVE = 4

# every symbol include/bed200.h declares
EXPORTS = (
    "bed_forward_f32",
    "bed_forward_ws_f32",
    "bed_forward_workspace_bytes",
    "bed_forward_host_f32",
    "bed_forward_host_f64",
    "bed_backward_f32",
    "bed_matrix_power_f32",
    "bed_forward_power_f32",
    "bed_forward_power_workspace_bytes",
    "bed_scatter_f32",
    "bed_scatter_forward_f32",
    "bed_scatter_forward_workspace_bytes",
    "bed_error_string",
    "bed_last_cuda_error",
    "bed_abi_version",
)


class BedConfig(ctypes.Structure):
    """``bed_config`` of include/bed200.h."""

    _fields_ = [
        ("deflation_tol", ctypes.c_float),
        ("symmetry_tol", ctypes.c_float),
        ("max_double_steps", ctypes.c_int32),
        ("sort", ctypes.c_int32),
        ("compute_vectors", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


class NativeError(RuntimeError):
    """A C ABI call returned an error code."""


_LIB = None


def lib() -> ctypes.CDLL:
    """Load libbed200.so (raises if it has not been built)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()' or make -C "
            "paper_2207_04228_b200/csrc). There is no CPU fallback."
        )
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
    L.bed_forward_f32.restype = ctypes.c_int
    L.bed_forward_f32.argtypes = [vp, i64, i32, vp, vp, vp, vp, vp, ctypes.POINTER(BedConfig), vp]
    L.bed_forward_ws_f32.restype = ctypes.c_int
    L.bed_forward_ws_f32.argtypes = [vp, i64, i32, vp, vp, vp, vp, vp, vp, vp,
                                     ctypes.POINTER(BedConfig), vp, ctypes.c_size_t, vp]
    L.bed_forward_workspace_bytes.restype = ctypes.c_size_t
    L.bed_forward_workspace_bytes.argtypes = [i64, i32, ctypes.POINTER(BedConfig)]
    L.bed_forward_host_f32.restype = ctypes.c_int
    L.bed_forward_host_f32.argtypes = [vp, i64, i32, vp, vp, vp, vp, ctypes.POINTER(BedConfig), i32]
    L.bed_forward_host_f64.restype = ctypes.c_int
    L.bed_forward_host_f64.argtypes = [vp, i64, i32, vp, vp, vp, vp, vp, vp,
                                       ctypes.POINTER(BedConfig), i32, i32]
    L.bed_backward_f32.restype = ctypes.c_int
    L.bed_backward_f32.argtypes = [vp, vp, vp, vp, vp, i64, i32, i32, vp, vp, vp]
    L.bed_matrix_power_f32.restype = ctypes.c_int
    L.bed_matrix_power_f32.argtypes = [vp, vp, vp, vp, vp, i64, i32, ctypes.c_float,
                                       ctypes.c_float, vp]
    L.bed_forward_power_f32.restype = ctypes.c_int
    L.bed_forward_power_f32.argtypes = [vp, i64, i32, vp, vp, vp, vp, ctypes.POINTER(BedConfig),
                                        ctypes.c_float, ctypes.c_float, vp, ctypes.c_size_t, vp]
    L.bed_forward_power_workspace_bytes.restype = ctypes.c_size_t
    L.bed_forward_power_workspace_bytes.argtypes = [i64, i32, ctypes.POINTER(BedConfig)]
    L.bed_scatter_f32.restype = ctypes.c_int
    L.bed_scatter_f32.argtypes = [vp, i64, i32, i32, ctypes.c_float, vp, vp]
    L.bed_scatter_forward_f32.restype = ctypes.c_int
    L.bed_scatter_forward_f32.argtypes = [vp, i64, i32, i32, ctypes.c_float, vp, vp, vp, vp,
                                          ctypes.POINTER(BedConfig), i32, ctypes.c_float,
                                          ctypes.c_float, vp, ctypes.c_size_t, vp]
    L.bed_scatter_forward_workspace_bytes.restype = ctypes.c_size_t
    L.bed_scatter_forward_workspace_bytes.argtypes = [i64, i32, i32, ctypes.POINTER(BedConfig), i32]
    L.bed_error_string.restype = ctypes.c_char_p
    L.bed_error_string.argtypes = [ctypes.c_int]
    L.bed_last_cuda_error.restype = ctypes.c_char_p
    L.bed_last_cuda_error.argtypes = []
    L.bed_abi_version.restype = ctypes.c_int
    L.bed_abi_version.argtypes = []
    _LIB = L
    return L


def check(rc: int, what: str) -> None:
    if rc != BED_SUCCESS:
        L = lib()
        msg = L.bed_error_string(rc).decode()
        if rc == 3:
            msg += ": " + L.bed_last_cuda_error().decode()
        raise NativeError(f"{what} failed with code {rc}: {msg}")


def make_config(cfg, n: int) -> BedConfig:
    return BedConfig(
        float(cfg.deflation_tol),
        float(cfg.symmetry_tol),
        int(cfg.resolved_max_steps(n)),
        int(cfg.sort_code),
        int(bool(cfg.compute_vectors)),
        0,
    )


def forward_f32(A_ptr, batch, n, evals_ptr, evecs_ptr, status_ptr, steps_ptr, flags_ptr,
                cfg: BedConfig, stream: int) -> None:
    rc = lib().bed_forward_f32(A_ptr, batch, n, evals_ptr, evecs_ptr, status_ptr, steps_ptr,
                               flags_ptr, ctypes.byref(cfg), stream)
    check(rc, "bed_forward_f32")


def forward_ws_f32(A_ptr, batch, n, evals_ptr, evecs_ptr, status_ptr, steps_ptr, flags_ptr,
                   diag_ptr, resid_ptr, cfg: BedConfig, ws_ptr, ws_bytes: int, stream: int) -> None:
    rc = lib().bed_forward_ws_f32(A_ptr, batch, n, evals_ptr, evecs_ptr, status_ptr, steps_ptr,
                                  flags_ptr, diag_ptr, resid_ptr, ctypes.byref(cfg), ws_ptr,
                                  ws_bytes, stream)
    check(rc, "bed_forward_ws_f32")


def workspace_bytes(batch: int, n: int, cfg: BedConfig) -> int:
    return int(lib().bed_forward_workspace_bytes(batch, n, ctypes.byref(cfg)))


def backward_f32(V_ptr, evals_ptr, gV_ptr, gL_ptr, gA_ptr, batch, n, degree, status_ptr,
                 flags_ptr, stream) -> None:
    rc = lib().bed_backward_f32(V_ptr, evals_ptr, gV_ptr, gL_ptr, gA_ptr, batch, n, degree,
                                status_ptr, flags_ptr, stream)
    check(rc, "bed_backward_f32")


def forward_host_f32(A_ptr, batch, n, evals_ptr, evecs_ptr, status_ptr, steps_ptr,
                     cfg: BedConfig, device: int) -> None:
    rc = lib().bed_forward_host_f32(A_ptr, batch, n, evals_ptr, evecs_ptr, status_ptr, steps_ptr,
                                    ctypes.byref(cfg), device)
    check(rc, "bed_forward_host_f32")


def forward_host_f64(A_ptr, batch, n, evals_ptr, evecs_ptr, status_ptr, steps_ptr, diag_ptr,
                     resid_ptr, cfg: BedConfig, device: int, threads: int = 0) -> None:
    rc = lib().bed_forward_host_f64(A_ptr, batch, n, evals_ptr, evecs_ptr, status_ptr, steps_ptr,
                                    diag_ptr, resid_ptr, ctypes.byref(cfg), device, threads)
    check(rc, "bed_forward_host_f64")


def matrix_power_f32(V_ptr, evals_ptr, out_ptr, status_ptr, flags_ptr, batch, n, p, floor,
                     stream) -> None:
    rc = lib().bed_matrix_power_f32(V_ptr, evals_ptr, out_ptr, status_ptr, flags_ptr, batch, n,
                                    p, floor, stream)
    check(rc, "bed_matrix_power_f32")


def forward_power_f32(A_ptr, batch, n, evals_ptr, out_ptr, status_ptr, flags_ptr, cfg: BedConfig,
                      p, floor, ws_ptr, ws_bytes, stream) -> None:
    rc = lib().bed_forward_power_f32(A_ptr, batch, n, evals_ptr, out_ptr, status_ptr, flags_ptr,
                                     ctypes.byref(cfg), p, floor, ws_ptr, ws_bytes, stream)
    check(rc, "bed_forward_power_f32")


def power_workspace_bytes(batch: int, n: int, cfg: BedConfig) -> int:
    return int(lib().bed_forward_power_workspace_bytes(batch, n, ctypes.byref(cfg)))


def scatter_forward_f32(X_ptr, batch, n, m, eps, evals_ptr, out_ptr, status_ptr, flags_ptr,
                        cfg: BedConfig, power, p, floor, ws_ptr, ws_bytes, stream) -> None:
    rc = lib().bed_scatter_forward_f32(X_ptr, batch, n, m, eps, evals_ptr, out_ptr, status_ptr,
                                       flags_ptr, ctypes.byref(cfg), int(power), p, floor, ws_ptr,
                                       ws_bytes, stream)
    check(rc, "bed_scatter_forward_f32")


def scatter_forward_workspace_bytes(batch: int, n: int, m: int, cfg: BedConfig, power) -> int:
    return int(lib().bed_scatter_forward_workspace_bytes(batch, n, m, ctypes.byref(cfg), int(power)))


def scatter_f32(X_ptr, batch, n, m, eps, out_ptr, stream) -> None:
    rc = lib().bed_scatter_f32(X_ptr, batch, n, m, eps, out_ptr, stream)
    check(rc, "bed_scatter_f32")
