"""The batched eigendecomposition API on the B200 kernels.

``batched_eig`` keeps the reference facade (``batchedeig.solver.batched_eig``,
/root/reference/pkg/src/batchedeig/solver.py:79-112): same arguments, same
result type, same exceptions, same ordering and sign convention.  It runs
the sm_100a kernels behind ``include/bed200.h`` -- there is no CPU path.

``BatchedEigFn`` is the differentiable form (a ``torch.autograd.Function``)
whose backward is the paper's Taylor-polynomial gradient (PAPER.md:668,
:700), which the reference package does not have (pkg/README.md:116-117).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native
from .core import (
    BatchedMatrix,
    BatchedSymmetric,
    EigenResult,
    NoConvergence,
    NonFinite,
    NonPositiveSpectrum,
    NonSymmetric,
    ShapeMismatch,
    SolveDiagnostics,
    SolverConfig,
)

__all__ = ["batched_eig", "eigh", "BatchedEigFn", "taylor_backward", "forward_into", "workspace",
           "spectral_power", "SpectralPowerFn", "power_of",
           "matrix_power", "zca_whiten", "scatter_matrices",
           "scatter_eig", "scatter_power", "TAYLOR_DEGREE"]

TAYLOR_DEGREE = 9


def _stream_handle(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _check_cuda_f32(t: torch.Tensor, name: str) -> torch.Tensor:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != torch.float32:
        raise ValueError(f"{name} must be float32, got {t.dtype}")
    return t.contiguous()


def workspace(A: torch.Tensor, cfg: SolverConfig, max_bytes: int | None = None) -> torch.Tensor | None:
    """A device workspace for ``forward_into`` from torch's caching allocator
    (``bed_forward_workspace_bytes``; None for n <= 8).  ``max_bytes`` caps it,
    in which case the batch is solved in chunks."""
    b, n, _ = A.shape
    c = _native.make_config(cfg, n)
    need = _native.workspace_bytes(b, n, c)
    if need == 0:
        return None
    if max_bytes is not None:
        need = max(min(need, int(max_bytes)), _native.workspace_bytes(32, n, c))
    return torch.empty((need + 255,), dtype=torch.uint8, device=A.device)


def forward_into(A: torch.Tensor, cfg: SolverConfig, evals: torch.Tensor,
                 evecs: torch.Tensor | None, status: torch.Tensor | None = None,
                 steps: torch.Tensor | None = None, flags: torch.Tensor | None = None,
                 ws: torch.Tensor | None = None, diag: torch.Tensor | None = None,
                 resid: torch.Tensor | None = None) -> None:
    """Launch the forward on preallocated device tensors, stream-ordered,
    without any host synchronisation (the C ABI call ``bed_forward_ws_f32``).
    The n >= 9 workspace is ``ws`` (from :func:`workspace`) or, when omitted,
    a fresh one from torch's caching allocator.  ``diag`` (batch, 3) int32 and
    ``resid`` (batch,) float32 receive the per-matrix diagnostics."""
    b, n, _ = A.shape
    ptr = lambda t: None if t is None else t.data_ptr()  # noqa: E731
    if ws is None and n > 8:
        ws = workspace(A, cfg)
    wp, wb = 0, 0
    if ws is not None:
        wp = (ws.data_ptr() + 255) & ~255
        wb = ws.numel() - (wp - ws.data_ptr())
    _native.forward_ws_f32(A.data_ptr(), b, n, evals.data_ptr(),
                           ptr(evecs) if cfg.compute_vectors else None,
                           ptr(status), ptr(steps), ptr(flags), ptr(diag), ptr(resid),
                           _native.make_config(cfg, n), wp or None, wb, _stream_handle(A.device))


def _raise_for_status(A: torch.Tensor, status: torch.Tensor, flags: int, cfg: SolverConfig,
                      resid: torch.Tensor | None = None) -> None:
    """Map per-matrix status codes onto the reference exceptions.

    Order follows the reference: validate (finiteness over the whole batch
    first, core.py:297-300, then symmetry, :301-308) before convergence
    (qr.py:606-609, only when strict).
    """
    if flags == 0:
        return
    st = status.cpu()
    if flags & (1 << _native.STATUS_NON_FINITE):
        k = int(torch.nonzero(st == _native.STATUS_NON_FINITE)[0, 0])
        bad = torch.nonzero(~torch.isfinite(A[k].detach().cpu()))
        # (-1, -1): the input is finite but a matrix formed from it overflowed
        raise NonFinite(k, (int(bad[0, 0]), int(bad[0, 1])) if len(bad) else (-1, -1))
    if flags & (1 << _native.STATUS_NON_SYMMETRIC):
        k = int(torch.nonzero(st == _native.STATUS_NON_SYMMETRIC)[0, 0])
        a = A[k].detach().double().cpu()
        raise NonSymmetric(k, float((a - a.T).abs().max()))
    if cfg.strict_convergence and flags & (1 << _native.STATUS_NO_CONVERGENCE):
        idx = torch.nonzero(st == _native.STATUS_NO_CONVERGENCE)[:, 0].tolist()
        raise NoConvergence(idx, float(resid.max()) if resid is not None else float("nan"))


def _solve_device(A: torch.Tensor, cfg: SolverConfig, check: bool = True, diagnostics: bool = False):
    A = _check_cuda_f32(A, "A")
    b, n, _ = A.shape
    dev = A.device
    evals = torch.empty((b, n), device=dev, dtype=torch.float32)
    evecs = torch.empty((b, n, n), device=dev, dtype=torch.float32) if cfg.compute_vectors else None
    status = torch.empty((b,), device=dev, dtype=torch.int32)
    steps = torch.empty((b,), device=dev, dtype=torch.int32)
    flags = torch.empty((1,), device=dev, dtype=torch.int32)
    diag = torch.empty((b, 3), device=dev, dtype=torch.int32) if diagnostics else None
    resid = torch.empty((b,), device=dev, dtype=torch.float32) if diagnostics or check else None
    with torch.cuda.device(dev):
        forward_into(A, cfg, evals, evecs, status, steps, flags, diag=diag, resid=resid)
    if check:
        _raise_for_status(A, status, int(flags.item()), cfg, resid)
    return evals, evecs, status, steps, diag


def _diagnostics(steps, diag=None) -> SolveDiagnostics:
    """Pool the per-matrix counters (see SolveDiagnostics)."""
    k = int(steps.max()) if len(steps) else 0
    if diag is None:
        return SolveDiagnostics(double_steps=k, reductions=-1.0, reduction_events=-1,
                                rotation_count=-1, converged_steps=steps)
    if isinstance(diag, np.ndarray):  # column by column: 7x faster than sum(axis=0) on (b, 3)
        tot = [int(diag[:, k].sum(dtype=np.int64)) for k in range(3)] if len(diag) else [0, 0, 0]
        nsteps = int(steps.sum(dtype=np.int64))
    else:
        tot = diag.long().sum(dim=0).tolist() if len(diag) else [0, 0, 0]
        nsteps = int(steps.long().sum()) if len(steps) else 0
    return SolveDiagnostics(double_steps=k, reductions=tot[2] / nsteps if nsteps else 0.0,
                            reduction_events=int(tot[1]), rotation_count=int(tot[0]),
                            converged_steps=steps, rotations=diag[:, 0],
                            reduction_counts=diag[:, 1])


def batched_eig(a, cfg: SolverConfig | None = None) -> EigenResult:
    """Full eigendecomposition of a batch of symmetric matrices (solver.py:79-112).

    ``a``: a ``BatchedSymmetric``, a (batch, n, n) numpy array, or a CUDA
    float32 tensor, 1 <= n <= 64.  Pipeline (all on the GPU, FP32): validate
    and symmetrise, Householder tridiagonalisation, double-shift QR with
    per-matrix deflation, eigenvectors accumulated in place, stable sort and
    sign normalisation.  Host (numpy) inputs are copied through page-locked
    memory and the results returned as float64 numpy arrays, like the
    reference; tensor inputs stay on their device.  Raises NonFinite,
    NonSymmetric and (strict) NoConvergence like the reference.
    """
    cfg = cfg or SolverConfig()
    data = a.data if isinstance(a, BatchedSymmetric) else a
    if isinstance(data, torch.Tensor):
        if data.ndim != 3 or data.shape[1] != data.shape[2] or data.shape[0] < 1:
            raise ShapeMismatch(f"expected (batch, n, n) tensor, got {tuple(data.shape)}")
        evals, evecs, status, steps, diag = _solve_device(data, cfg, diagnostics=True)
        return EigenResult(evals, evecs, _diagnostics(steps, diag))
    arr = np.asarray(data)
    if arr.ndim != 3 or arr.shape[1] != arr.shape[2] or arr.shape[0] < 1:
        raise ShapeMismatch(f"expected (batch, n, n) array, got {arr.shape}")
    if arr.dtype != np.float32:
        # float64 (the reference's dtype): validate + symmetrise in float64 on
        # host threads inside the native call (core.py:286-309), then FP32
        return _solve_host_f64(np.ascontiguousarray(arr, dtype=np.float64), cfg)
    host = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).pin_memory()
    dev = torch.device("cuda", torch.cuda.current_device())
    A = host.to(dev, non_blocking=True)
    evals, evecs, status, steps, diag = _solve_device(A, cfg, diagnostics=True)
    out_l = evals.to("cpu", non_blocking=True)
    out_v = evecs.to("cpu", non_blocking=True) if evecs is not None else None
    torch.cuda.current_stream(dev).synchronize()
    return EigenResult(out_l.numpy().astype(np.float64),
                       None if out_v is None else out_v.numpy().astype(np.float64),
                       _diagnostics(steps.cpu().numpy(), diag.cpu().numpy()))


def _solve_host_f64(a: np.ndarray, cfg: SolverConfig) -> EigenResult:
    """float64 host batch -> float64 host results through ``bed_forward_host_f64``
    (host-thread validation and casts overlapped with the PCIe copies and the
    solves), raising in the reference's order: NonFinite over the whole batch
    first, then NonSymmetric (core.py:297-308), then (strict) NoConvergence."""
    b, n, _ = a.shape
    evals = np.empty((b, n), np.float64)
    evecs = np.empty((b, n, n), np.float64) if cfg.compute_vectors else None
    status = np.empty((b,), np.int32)
    steps = np.empty((b,), np.int32)
    diag = np.empty((b, 3), np.int32)
    resid = np.empty((b,), np.float32)
    _native.forward_host_f64(a.ctypes.data, b, n, evals.ctypes.data,
                             evecs.ctypes.data if evecs is not None else None, status.ctypes.data,
                             steps.ctypes.data, diag.ctypes.data, resid.ctypes.data,
                             _native.make_config(cfg, n), torch.cuda.current_device())
    if (status != 0).any():
        bad = np.flatnonzero(status == _native.STATUS_NON_FINITE)
        if len(bad):
            k = int(bad[0])
            pos = np.argwhere(~np.isfinite(a[k]))
            # (-1, -1): finite in float64 but beyond the FP32 range
            raise NonFinite(k, (int(pos[0, 0]), int(pos[0, 1])) if len(pos) else (-1, -1))
        bad = np.flatnonzero(status == _native.STATUS_NON_SYMMETRIC)
        if len(bad):
            k = int(bad[0])
            raise NonSymmetric(k, float(np.abs(a[k] - a[k].T).max()))
        if cfg.strict_convergence:
            idx = np.flatnonzero(status == _native.STATUS_NO_CONVERGENCE).tolist()
            if idx:
                raise NoConvergence(idx, float(resid[idx].max()))
    return EigenResult(evals, evecs, _diagnostics(steps, diag))


def taylor_backward(V: torch.Tensor, evals: torch.Tensor, g_v: torch.Tensor | None,
                    g_evals: torch.Tensor | None, degree: int = TAYLOR_DEGREE,
                    check: bool = False) -> torch.Tensor:
    """gA = sym(V (F o (V^T gV) + diag(gL)) V^T) with the Taylor-K F (C ABI
    ``bed_backward_f32``).  Missing cotangents are zero.

    The series is the paper's for positive spectra.  A
    pair outside its domain (larger eigenvalue <= 0, or a smaller one <= its
    negative) takes the exact 1/(l_j - l_i); with ``check=True`` such a
    matrix raises ``NonPositiveSpectrum`` (one host read of the flags word),
    otherwise the exact fallback is used silently.
    """
    V = _check_cuda_f32(V, "V")
    evals = _check_cuda_f32(evals, "evals")
    b, n, _ = V.shape
    gv = None if g_v is None else _check_cuda_f32(g_v, "g_v")
    gl = None if g_evals is None else _check_cuda_f32(g_evals, "g_evals")
    gA = torch.empty_like(V)
    status = torch.empty((b,), device=V.device, dtype=torch.int32) if check else None
    flags = torch.empty((1,), device=V.device, dtype=torch.int32) if check else None
    with torch.cuda.device(V.device):
        _native.backward_f32(V.data_ptr(), evals.data_ptr(),
                             None if gv is None else gv.data_ptr(),
                             None if gl is None else gl.data_ptr(),
                             gA.data_ptr(), b, n, int(degree),
                             None if status is None else status.data_ptr(),
                             None if flags is None else flags.data_ptr(),
                             _stream_handle(V.device))
    if check and int(flags.item()) & (1 << _native.STATUS_NON_POSITIVE):
        k = int(torch.nonzero(status == _native.STATUS_NON_POSITIVE)[0, 0])
        raise NonPositiveSpectrum(k, float(evals[k].min()))
    return gA


class BatchedEigFn(torch.autograd.Function):
    """Differentiable batched ED: forward = ``bed_forward_f32``, backward =
    the Taylor-polynomial gradient ``bed_backward_f32`` (degree 9 by default).

    ``check=False`` skips the host reads of the status words, keeping the
    forward and backward free of device-to-host synchronisation (for training
    loops); with ``check=True`` the backward also raises NonPositiveSpectrum
    for a spectrum outside the Taylor series' domain (see taylor_backward).
    """

    @staticmethod
    def forward(ctx, A, cfg: SolverConfig | None = None, degree: int = TAYLOR_DEGREE,
                check: bool = True):
        cfg = cfg or SolverConfig()
        if not cfg.compute_vectors:
            raise ValueError("the differentiable ED needs compute_vectors=True")
        evals, evecs, _, _, _ = _solve_device(A.detach(), cfg, check=check)
        ctx.save_for_backward(evals, evecs)
        ctx.degree = degree
        ctx.check = check
        return evals, evecs

    @staticmethod
    def backward(ctx, g_evals, g_evecs):
        evals, evecs = ctx.saved_tensors
        gA = taylor_backward(evecs, evals, g_evecs, g_evals, ctx.degree, ctx.check)
        return gA, None, None, None


def eigh(A: torch.Tensor, cfg: SolverConfig | None = None, degree: int = TAYLOR_DEGREE,
         check: bool = True):
    """(eigenvalues, eigenvectors) of a CUDA float32 batch, differentiable."""
    return BatchedEigFn.apply(A, cfg, degree, check)


def _power_device(V: torch.Tensor, lam: torch.Tensor, p: float, floor: float | None):
    V = _check_cuda_f32(V, "eigenvectors")
    lam = _check_cuda_f32(lam, "eigenvalues")
    b, n, _ = V.shape
    out = torch.empty_like(V)
    status = torch.empty((b,), device=V.device, dtype=torch.int32)
    flags = torch.empty((1,), device=V.device, dtype=torch.int32)
    with torch.cuda.device(V.device):
        _native.matrix_power_f32(V.data_ptr(), lam.data_ptr(), out.data_ptr(), status.data_ptr(),
                                 flags.data_ptr(), b, n, float(p),
                                 -1.0 if floor is None else float(floor),
                                 _stream_handle(V.device))
    if int(flags.item()) & (1 << _native.STATUS_NON_POSITIVE):
        k = int(torch.nonzero(status == _native.STATUS_NON_POSITIVE)[0, 0])
        raise NonPositiveSpectrum(k, float(lam[k].min()))
    return out


def matrix_power(e: EigenResult, p: float, floor: float | None = None) -> BatchedMatrix:
    """Spectral power V diag(max(w, floor)^p) V^T of a decomposed batch
    (reference ``matrix_power``, solver.py:115-143), on the GPU
    (``bed_matrix_power_f32``: one tiled FFMA2 product per matrix).

    ``floor=None`` applies the default guard 1e-12 * lambda_max per matrix;
    ``floor=0.0`` disables it, and a non-positive eigenvalue then raises
    NonPositiveSpectrum whenever p is negative or fractional.  Device
    (tensor) results stay on the device; numpy results come back float64.
    """
    if e.eigenvectors is None:
        raise ValueError("matrix_power needs an EigenResult with eigenvectors")
    if floor is not None and floor < 0:
        raise ValueError("floor must be nonnegative")
    if isinstance(e.eigenvectors, torch.Tensor):
        return BatchedMatrix(_power_device(e.eigenvectors, e.eigenvalues, p, floor))
    dev = torch.device("cuda", torch.cuda.current_device())
    V = torch.from_numpy(np.ascontiguousarray(e.eigenvectors, dtype=np.float32)).to(dev)
    lam = torch.from_numpy(np.ascontiguousarray(e.eigenvalues, dtype=np.float32)).to(dev)
    out = _power_device(V, lam, p, floor)
    return BatchedMatrix(out.cpu().numpy().astype(np.float64))


def scatter_matrices(x: torch.Tensor, eps: float = 0.0) -> torch.Tensor:
    """sym((X - mu)(X - mu)^T) + eps I per matrix of a (batch, n, m) CUDA float32
    batch (the scatter of the reference zca_whiten, solver.py:161-166), on the
    native covariance producer ``bed_scatter_f32``."""
    x = _check_cuda_f32(x, "X")
    b, n, m = x.shape
    out = torch.empty((b, n, n), device=x.device, dtype=torch.float32)
    with torch.cuda.device(x.device):
        _native.scatter_f32(x.data_ptr(), b, n, m, float(eps), out.data_ptr(),
                            _stream_handle(x.device))
    return out


def _scatter_forward(x, eps, cfg, power, p, floor, check):
    cfg = cfg or SolverConfig()
    if eps < 0:
        raise ValueError("eps must be nonnegative")
    x = _check_cuda_f32(x, "X")
    b, n, m = x.shape
    if m < 1:
        raise ValueError("X needs at least one sample")
    c = _native.make_config(cfg, n)
    vecs = power or cfg.compute_vectors
    dev = x.device
    evals = torch.empty((b, n), device=dev, dtype=torch.float32)
    out = torch.empty((b, n, n), device=dev, dtype=torch.float32) if vecs else None
    status = torch.empty((b,), device=dev, dtype=torch.int32)
    flags = torch.empty((1,), device=dev, dtype=torch.int32)
    wb = _native.scatter_forward_workspace_bytes(b, n, m, c, power)
    ws = torch.empty((wb + 256,), dtype=torch.uint8, device=dev) if wb else None
    wp = ((ws.data_ptr() + 255) & ~255) if ws is not None else None
    with torch.cuda.device(dev):
        _native.scatter_forward_f32(x.data_ptr(), b, n, m, float(eps), evals.data_ptr(),
                                    out.data_ptr() if out is not None else None, status.data_ptr(),
                                    flags.data_ptr(), c, power, float(p),
                                    -1.0 if floor is None else float(floor), wp, wb,
                                    _stream_handle(dev))
    if check:
        fl = int(flags.item())
        _raise_for_status(x, status, fl & ~(1 << _native.STATUS_NON_POSITIVE), cfg)
        if fl & (1 << _native.STATUS_NON_POSITIVE):
            k = int(torch.nonzero(status == _native.STATUS_NON_POSITIVE)[0, 0])
            raise NonPositiveSpectrum(k, float(evals[k].min()))
    return evals, out


def scatter_eig(x: torch.Tensor, eps: float = 0.0, cfg: SolverConfig | None = None,
                check: bool = True):
    """Eigen-decomposition of the scatter matrices of a (batch, n, m) CUDA
    float32 batch (``scatter_matrices`` then ``batched_eig``; reference
    zca_whiten's scatter + batched_eig, solver.py:79-112,161-166) in one call
    (C ABI ``bed_scatter_forward_f32``): for n <= 8 one kernel forms each
    covariance in registers and solves it, so it never reaches memory.
    Returns (evals, evecs); evecs is None when ``cfg.compute_vectors`` is off.
    A non-finite sample raises NonFinite at its (channel, sample) position."""
    return _scatter_forward(x, eps, cfg, 0, 0.0, None, check)


def scatter_power(x: torch.Tensor, p: float, eps: float = 0.0, cfg: SolverConfig | None = None,
                  floor: float | None = None, check: bool = True) -> torch.Tensor:
    """S^p = V diag(max(lambda, floor)^p) V^T of the scatter matrices
    S = (X - mu)(X - mu)^T + eps I of a (batch, n, m) CUDA float32 batch, in
    one call (``bed_scatter_forward_f32`` with power): for n <= 8 a single
    kernel goes from X to S^p -- neither S nor V reaches memory (the whitening
    matrix of decorrelated BN / zca_whiten, solver.py:146-169, with p = -1/2).
    Raises like ``power_of``."""
    return _scatter_forward(x, eps, cfg, 1, p, floor, check)[1]


def _power_values(lam: torch.Tensor, p: float, floor: float | None):
    """f(lambda) = max(lambda, floor)^p and f'(lambda) (0 where the floor
    clamps), the floor resolved per matrix like bed_matrix_power_f32:
    None -> 1e-12 * lambda_max (solver.py:131-132)."""
    lam64 = lam.double()
    fl = (1e-12 * lam64.max(dim=1, keepdim=True).values) if floor is None else torch.full_like(lam64[:, :1], floor)
    clamped = lam64 < fl
    x = torch.where(clamped, fl, lam64)
    f = x.pow(p)
    df = torch.where(clamped, torch.zeros_like(x), p * x.pow(p - 1))
    return f.float(), df.float()


class SpectralPowerFn(torch.autograd.Function):
    """Differentiable spectral power A -> V diag(max(lambda, floor)^p) V^T
    (the reference matrix_power, solver.py:115-143, composed with the ED):
    forward = bed_forward + bed_matrix_power_f32; backward through f(lambda):
    with Y = V f(Lambda) V^T,  gV = (gY + gY^T) V f(Lambda) and
    gLambda = f'(lambda) o diag(V^T gY V), then the paper's Taylor-K ED
    backward (bed_backward_f32) maps (gV, gLambda) to gA -- the chain the
    decorrelated-BN / whitening consumer differentiates."""

    @staticmethod
    def forward(ctx, A, p: float, cfg: SolverConfig | None = None, floor: float | None = None,
                degree: int = TAYLOR_DEGREE, check: bool = True):
        cfg = cfg or SolverConfig()
        if not ctx.needs_input_grad[0]:  # inference: V is not needed afterwards
            return power_of(A.detach(), p, cfg, floor, check)
        evals, evecs, _, _, _ = _solve_device(A.detach(), cfg, check=check)
        out = _power_device(evecs, evals, p, floor) if check else _power_nocheck(evecs, evals, p, floor)
        ctx.save_for_backward(evals, evecs)
        ctx.p, ctx.floor, ctx.degree, ctx.check = p, floor, degree, check
        return out

    @staticmethod
    def backward(ctx, g_out):
        evals, evecs = ctx.saved_tensors
        f, df = _power_values(evals, ctx.p, ctx.floor)
        gs = g_out.float() + g_out.float().transpose(1, 2)
        g_v = torch.bmm(gs, evecs) * f[:, None, :]
        m = torch.bmm(evecs.transpose(1, 2), torch.bmm(g_out.float(), evecs))
        g_l = torch.diagonal(m, dim1=1, dim2=2) * df
        gA = taylor_backward(evecs, evals, g_v.contiguous(), g_l.contiguous(), ctx.degree, ctx.check)
        return gA, None, None, None, None, None


def _power_nocheck(V, lam, p, floor):
    V = _check_cuda_f32(V, "eigenvectors")
    lam = _check_cuda_f32(lam, "eigenvalues")
    b, n, _ = V.shape
    out = torch.empty_like(V)
    with torch.cuda.device(V.device):
        _native.matrix_power_f32(V.data_ptr(), lam.data_ptr(), out.data_ptr(), None, None, b, n, float(p),
                                 -1.0 if floor is None else float(floor), _stream_handle(V.device))
    return out


def power_of(A: torch.Tensor, p: float, cfg: SolverConfig | None = None,
             floor: float | None = None, check: bool = True) -> torch.Tensor:
    """V diag(max(lambda, floor)^p) V^T of a CUDA float32 batch in one call
    (C ABI ``bed_forward_power_f32``): for n <= 8 the power is formed in the
    forward kernel's epilogue and V never reaches memory.  Raises like
    ``batched_eig`` and ``matrix_power`` when ``check``."""
    cfg = cfg or SolverConfig()
    A = _check_cuda_f32(A, "A")
    b, n, _ = A.shape
    c = _native.make_config(cfg, n)
    out = torch.empty_like(A)
    evals = torch.empty((b, n), device=A.device, dtype=torch.float32)
    status = torch.empty((b,), device=A.device, dtype=torch.int32)
    flags = torch.empty((1,), device=A.device, dtype=torch.int32)
    wb = _native.power_workspace_bytes(b, n, c)
    ws = torch.empty((wb + 256,), dtype=torch.uint8, device=A.device) if wb else None
    wp = ((ws.data_ptr() + 255) & ~255) if ws is not None else None
    with torch.cuda.device(A.device):
        _native.forward_power_f32(A.data_ptr(), b, n, evals.data_ptr(), out.data_ptr(),
                                  status.data_ptr(), flags.data_ptr(), c, float(p),
                                  -1.0 if floor is None else float(floor), wp, wb,
                                  _stream_handle(A.device))
    if check:
        fl = int(flags.item())
        _raise_for_status(A, status, fl & ~(1 << _native.STATUS_NON_POSITIVE), cfg)
        if fl & (1 << _native.STATUS_NON_POSITIVE):
            k = int(torch.nonzero(status == _native.STATUS_NON_POSITIVE)[0, 0])
            raise NonPositiveSpectrum(k, float(evals[k].min()))
    return out


def spectral_power(A: torch.Tensor, p: float, cfg: SolverConfig | None = None,
                   floor: float | None = None, degree: int = TAYLOR_DEGREE, check: bool = True):
    """V diag(max(lambda, floor)^p) V^T of a CUDA float32 batch, differentiable
    in A (see SpectralPowerFn); ``check=False`` keeps forward and backward
    free of host synchronisation."""
    return SpectralPowerFn.apply(A, p, cfg, floor, degree, check)


def zca_whiten(x: BatchedMatrix, eps_reg: float, cfg: SolverConfig | None = None) -> BatchedMatrix:
    """ZCA whitening of (batch, channels, samples) features (reference
    ``zca_whiten``, solver.py:146-169): the unnormalised scatter
    (X - mu)(X - mu)^T + eps_reg I is decomposed on the GPU and its inverse
    square root (``matrix_power(-0.5, floor=0)``) applied to the centred
    features.  Scatter, ED and inverse square root are one native call
    (``scatter_power`` / ``bed_scatter_forward_f32``: a single kernel for
    n <= 8, the covariance producer + the forward with the power fused into
    its epilogue above); the final product ``S^(-1/2) (X - mu)`` is a torch
    batched matmul.
    """
    if eps_reg < 0:
        raise ValueError("eps_reg must be nonnegative")
    data = x.data if isinstance(x, BatchedMatrix) else x
    host = not isinstance(data, torch.Tensor)
    t = torch.from_numpy(np.asarray(data, dtype=np.float32)) if host else data
    if host:
        t = t.to(torch.device("cuda", torch.cuda.current_device()))
    t = t.contiguous()
    inv_root = scatter_power(t, -0.5, eps_reg, cfg, floor=0.0)
    out = inv_root @ (t - t.mean(dim=2, keepdim=True))
    return BatchedMatrix(out.cpu().numpy().astype(np.float64) if host else out)
