"""TEST INFRASTRUCTURE -- ctypes wrapper over the C restatement plus numpy
restatements of the backward and the input generator.  See ``oracle/__init__.py``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

GATE_BATCH = 0
GATE_MATRIX = 1
_SORT = {"none": 0, "descending": 1, "ascending": 2}

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def library_path() -> str:
    return os.path.join(_HERE, "_build", "libbedoracle.so")


def build(force: bool = False) -> str:
    """Compile ``bed_oracle.c`` (gcc, IEEE double) if the .so is missing."""
    path = library_path()
    src = os.path.join(_HERE, "bed_oracle.c")
    if force or not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return path


class _Config(ctypes.Structure):
    _fields_ = [
        ("deflation_tol", ctypes.c_double),
        ("symmetry_tol", ctypes.c_double),
        ("max_double_steps", ctypes.c_int32),
        ("sort", ctypes.c_int32),
        ("compute_vectors", ctypes.c_int32),
        ("strict", ctypes.c_int32),
        ("gate", ctypes.c_int32),
        ("threads", ctypes.c_int32),
        ("chunk", ctypes.c_int64),
    ]


class _Outputs(ctypes.Structure):
    _fields_ = [
        ("status", ctypes.c_void_p),
        ("converged_steps", ctypes.c_void_p),
        ("double_steps", ctypes.c_void_p),
        ("rotations", ctypes.c_void_p),
        ("residual", ctypes.c_void_p),
    ]


def _lib():
    global _LIB
    if _LIB is None:
        _LIB = ctypes.CDLL(build())
        _LIB.bedo_forward.restype = ctypes.c_int
        _LIB.bedo_forward.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(_Config),
            ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(_Outputs),
        ]
        _LIB.bedo_wilkinson.restype = None
        _LIB.bedo_wilkinson.argtypes = [ctypes.c_double] * 3 + [ctypes.c_void_p]
        _LIB.bedo_tridiagonalize.restype = None
        _LIB.bedo_tridiagonalize.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p]
    return _LIB


@dataclass
class OracleResult:
    eigenvalues: np.ndarray          # (b, n) float64
    eigenvectors: np.ndarray | None  # (b, n, n) float64
    status: np.ndarray               # (b,) int32: 0 ok, 1 no-conv, 2 non-finite, 3 non-symmetric
    converged_steps: np.ndarray      # (b,) int32
    double_steps: np.ndarray         # (b,) int32
    rotations: np.ndarray            # (b,) int64
    residual: np.ndarray             # (b,) float64


def forward(a, deflation_tol: float = 3e-12, max_double_steps: int | None = None,
            sort: str = "descending", compute_vectors: bool = True, strict: bool = True,
            symmetry_tol: float = 1e-12, gate: int = GATE_MATRIX, threads: int = 1,
            chunk: int = 0) -> OracleResult:
    """Reference ``batched_eig`` restated in C, float64.

    Defaults are the reference's *verify* profile (``bench.py:40``,
    ``bench.py:227-228``: tol 3e-12, budget 4n) with per-matrix gating.
    ``gate=GATE_BATCH`` with ``chunk=0`` reproduces the reference's
    batch-wide gate over the whole batch.
    """
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 3 or a.shape[1] != a.shape[2]:
        raise ValueError(f"expected (batch, n, n), got {a.shape}")
    b, n, _ = a.shape
    steps = 4 * n if max_double_steps is None else int(max_double_steps)
    cfg = _Config(deflation_tol, symmetry_tol, steps, _SORT[sort], int(compute_vectors),
                  int(strict), gate, max(1, threads), chunk)
    evals = np.zeros((b, n))
    evecs = np.zeros((b, n, n)) if compute_vectors else None
    status = np.zeros(b, np.int32)
    conv = np.zeros(b, np.int32)
    dsteps = np.zeros(b, np.int32)
    rots = np.zeros(b, np.int64)
    resid = np.zeros(b)
    outs = _Outputs(status.ctypes.data, conv.ctypes.data, dsteps.ctypes.data,
                    rots.ctypes.data, resid.ctypes.data)
    rc = _lib().bedo_forward(a.ctypes.data, b, n, ctypes.byref(cfg), evals.ctypes.data,
                             evecs.ctypes.data if evecs is not None else None,
                             ctypes.byref(outs))
    if rc != 0:
        raise ValueError("bedo_forward rejected its arguments")
    return OracleResult(evals, evecs, status, conv, dsteps, rots, resid)


def wilkinson(a: float, b: float, d: float):
    """(lo, hi, c, s) of [[a, b], [b, d]] -- ``_kernels.py:205-218``."""
    out = np.zeros(4)
    _lib().bedo_wilkinson(a, b, d, out.ctypes.data)
    return tuple(float(x) for x in out)


def tridiagonalize(a):
    """Householder reduction of each matrix (``_kernels.py:36-92``).

    Returns (work (b,n,n), vectors (n-2 per matrix, as (b, n-2, n))).
    """
    w = np.array(a, dtype=np.float64, order="C", copy=True)
    b, n, _ = w.shape
    vec = np.zeros((b, max(n - 2, 1), n))
    _lib().bedo_tridiagonalize(w.ctypes.data, b, n, vec.ctypes.data)
    return w, vec[:, : max(n - 2, 0)]


# ---------------------------------------------------------------------------
# backward (absent from the reference; restated from the paper)


def taylor_k(evals, degree: int = 9) -> np.ndarray:
    """Taylor-polynomial stand-in for F_ij = 1/(lambda_j - lambda_i).

    For a pair i < j with lambda_i >= lambda_j (descending order, ties by
    index) F_ij = -(1/lambda_i) * sum_{k=0..degree} (lambda_j/lambda_i)^k and
    F_ji = -F_ij; if lambda_i < lambda_j the roles swap.  F_ii = 0.  Paper:
    PAPER.md:668 (backward reuses [song2021approximate])
    (Taylor degree 9).

    The series sums to 1/(l_big - l_small) only for |l_small/l_big| < 1 (and
    is (degree+1)/l on ties): the positive spectra the paper's covariance
    inputs have.  A pair outside that domain (l_big <= 0, or l_small <=
    -l_big, not a tie) takes the exact 1/(lambda_j - lambda_i); two zero
    eigenvalues, or a tie outside the domain, give F = 0.  :func:`taylor_domain` reports which matrices
    had such a pair (the kernel's BED_STATUS_NON_POSITIVE).
    """
    lam = np.asarray(evals, dtype=np.float64)
    b, n = lam.shape
    li = lam[:, :, None]
    lj = lam[:, None, :]
    idx = np.arange(n)
    upper = idx[:, None] < idx[None, :]
    # hi_first: the row eigenvalue is the larger one of the pair (index order on ties)
    hi_first = np.where(upper, li >= lj, li > lj)
    big = np.where(hi_first, li, lj)
    small = np.where(hi_first, lj, li)
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = np.where(big != 0, small / np.where(big != 0, big, 1.0), 0.0)
        inv = np.where(big != 0, 1.0 / np.where(big != 0, big, 1.0), 0.0)
        gap = big - small
        exact = np.where(gap != 0, 1.0 / np.where(gap != 0, gap, 1.0), 0.0)
    acc = np.ones_like(ratio)
    term = np.ones_like(ratio)
    for _ in range(degree):
        term = term * ratio
        acc = acc + term
    t = np.where(_in_domain(big, small, ratio), inv * acc, exact)
    f = np.where(hi_first, -t, t)
    f[:, idx, idx] = 0.0
    return f


def _in_domain(big, small, ratio):
    return ((big > 0) & ((np.abs(ratio) < 1) | (small == big))) | ((big == 0) & (small == 0))


def taylor_domain(evals) -> np.ndarray:
    """True per matrix when every eigenvalue pair is inside the Taylor
    series' domain (see :func:`taylor_k`)."""
    lam = np.asarray(evals, dtype=np.float64)
    li, lj = lam[:, :, None], lam[:, None, :]
    big, small = np.maximum(li, lj), np.minimum(li, lj)
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = np.where(big != 0, small / np.where(big != 0, big, 1.0), 0.0)
    ok = _in_domain(big, small, ratio)
    n = lam.shape[1]
    ok[:, np.arange(n), np.arange(n)] = True
    return ok.all(axis=(1, 2))


def taylor_backward(v, evals, g_v=None, g_evals=None, degree: int = 9) -> np.ndarray:
    """gA = sym( V (F o (V^T gV) + diag(gLambda)) V^T ), float64.

    sym(M) = (M + M^T)/2, F from :func:`taylor_k`.  Missing cotangents are
    zero.  As degree -> inf this is the exact eigh backward (the symmetrised
    form torch.linalg.eigh autograd returns).
    """
    v = np.asarray(v, dtype=np.float64)
    lam = np.asarray(evals, dtype=np.float64)
    b, n, _ = v.shape
    inner = np.zeros((b, n, n))
    if g_v is not None:
        inner += taylor_k(lam, degree) * (v.transpose(0, 2, 1) @ np.asarray(g_v, np.float64))
    if g_evals is not None:
        idx = np.arange(n)
        inner[:, idx, idx] += np.asarray(g_evals, np.float64)
    g = v @ inner @ v.transpose(0, 2, 1)
    return (g + g.transpose(0, 2, 1)) / 2.0


def matrix_power(v, evals, p: float, floor: float | None = None) -> np.ndarray:
    """V diag(max(w, floor)^p) V^T, symmetrised -- reference ``matrix_power``
    (solver.py:115-143), float64.  Returns (out, bad) where ``bad`` marks the
    matrices whose clamped spectrum is not positive for a negative or
    fractional p (the reference raises NonPositiveSpectrum on the first)."""
    v = np.asarray(v, np.float64)
    w = np.asarray(evals, np.float64)
    if floor is None:
        clamped = np.maximum(w, 1e-12 * w.max(axis=1, keepdims=True))
    else:
        clamped = np.maximum(w, floor)
    needs_positive = p < 0 or not float(p).is_integer()
    bad = (clamped.min(axis=1) <= 0) if needs_positive else np.zeros(len(w), bool)
    with np.errstate(all="ignore"):
        powered = np.where(bad[:, None], 0.0, clamped) ** p
    powered[bad] = 0.0
    out = (v * powered[:, None, :]) @ v.transpose(0, 2, 1)
    return (out + out.transpose(0, 2, 1)) / 2.0, bad


# ---------------------------------------------------------------------------
# input generator


def gen_spd(batch: int, dim: int, seed: int, condition_decades: float = 3.0) -> np.ndarray:
    """Seeded SPD batch Q diag(lam) Q^T -- reference ``bench.py:112-134``.

    Bit-identical to the reference generator (same numpy Generator calls in
    the same order).  Returns a float64 (batch, dim, dim) array.
    """
    rng = np.random.default_rng(seed)
    raw = rng.standard_normal((dim, batch, dim))
    exps = rng.uniform(0.0, condition_decades, (batch, dim))
    scale = 10.0 ** rng.uniform(-0.5, 0.5, batch)
    lam = scale[:, None] * 10.0 ** (-exps)
    q = np.broadcast_to(np.eye(dim), (batch, dim, dim)).copy()
    for k in range(dim):
        vk = raw[k]
        vk = vk / np.sqrt((vk * vk).sum(axis=-1))[:, None]
        qv = q @ vk[:, :, None]
        q -= 2.0 * qv * vk[:, None, :]
    a = (q * lam[:, None, :]) @ q.transpose(0, 2, 1)
    return (a + a.transpose(0, 2, 1)) / 2.0
