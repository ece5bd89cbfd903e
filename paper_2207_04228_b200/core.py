"""Configuration, result types and errors of the batched eigendecomposition.

Mirrors the reference ``batchedeig.core`` (``/root/reference/pkg/src/batchedeig/core.py``)
names, argument meanings and error behaviour, so reference callers switch by
changing the import:

* ``SolverConfig``       core.py:226-279 (same fields, defaults and validation)
* ``BatchedSymmetric``   core.py:122-146 (shape-checked container; accepts
                         numpy arrays and torch tensors)
* errors                 core.py:42-109 (``NonSymmetric``, ``NonFinite``,
                         ``NoConvergence``, ``ShapeMismatch``, ...)
* ``SolveDiagnostics``   qr.py:101-118
* ``EigenResult``        solver.py:38-57
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Any

import numpy as np

__all__ = [
    "BatchedEigError",
    "NonSymmetric",
    "NonFinite",
    "NoConvergence",
    "NonPositiveSpectrum",
    "BadMagic",
    "TruncatedPayload",
    "DimMismatch",
    "ShapeMismatch",
    "BatchedMatrix",
    "BatchedSymmetric",
    "SolverConfig",
    "SolveDiagnostics",
    "EigenResult",
]


class BatchedEigError(Exception):
    """Base class for every error raised by this package (core.py:42)."""


class NonSymmetric(BatchedEigError):
    """Input matrix is asymmetric beyond the configured tolerance (core.py:46-55)."""

    def __init__(self, batch_index: int, max_asymmetry: float):
        super().__init__(
            f"matrix {batch_index} is not symmetric: "
            f"max |a_ij - a_ji| = {max_asymmetry:.6e} exceeds tolerance"
        )
        self.batch_index = batch_index
        self.max_asymmetry = max_asymmetry


class NonFinite(BatchedEigError):
    """Input contains a NaN or infinity (core.py:58-64)."""

    def __init__(self, batch_index: int, position: tuple[int, ...]):
        super().__init__(f"matrix {batch_index} has a non-finite entry at {position}")
        self.batch_index = batch_index
        self.position = position


class NoConvergence(BatchedEigError):
    """Iteration budget exhausted with off-diagonal mass above threshold (core.py:83-93).

    ``residual_offdiag_max``: the largest coupling left in any offender's
    active block, on its power-of-two equilibrated band (qr.py:385-389).
    """

    def __init__(self, batch_indices, residual_offdiag_max: float):
        indices = sorted(int(i) for i in batch_indices)
        super().__init__(
            f"QR iteration did not converge for batch indices {indices} "
            f"(max residual off-diagonal {residual_offdiag_max:.6e})"
        )
        self.batch_indices = indices
        self.residual_offdiag_max = residual_offdiag_max


class NonPositiveSpectrum(BatchedEigError):
    """A fractional or negative matrix power hit a non-positive eigenvalue (core.py:96-105)."""

    def __init__(self, batch_index: int, min_eigenvalue: float):
        super().__init__(
            f"matrix {batch_index} has min eigenvalue {min_eigenvalue:.6e}; "
            "fractional/negative powers need a positive spectrum (or a floor)"
        )
        self.batch_index = batch_index
        self.min_eigenvalue = min_eigenvalue


class BadMagic(BatchedEigError):
    """Stream does not start with a supported BED1 header (core.py:67-68)."""


class TruncatedPayload(BatchedEigError):
    """Stream ended before the payload its header announced (core.py:71-72)."""


class DimMismatch(BatchedEigError):
    """Header dimensions are invalid or not the expected shape (core.py:75-76)."""


class ShapeMismatch(BatchedEigError):
    """Two batched operands disagree in batch size or matrix dimension (core.py:108-109)."""


@dataclass(frozen=True)
class BatchedMatrix:
    """A batch of dense rectangular matrices, shape (batch, rows, cols) (core.py:150-173).

    Holds a numpy array or a torch tensor (the device path keeps tensors on
    the GPU).
    """

    data: Any

    def __post_init__(self):
        shape = tuple(self.data.shape)
        if len(shape) != 3:
            raise ShapeMismatch(f"expected (batch, rows, cols) array, got {shape}")
        if min(shape) < 1:
            raise ShapeMismatch(f"all dimensions must be positive, got {shape}")

    @property
    def batch(self) -> int:
        return self.data.shape[0]

    @property
    def dim_rows(self) -> int:
        return self.data.shape[1]

    @property
    def dim_cols(self) -> int:
        return self.data.shape[2]


@dataclass(frozen=True)
class BatchedSymmetric:
    """A batch of dense symmetric n x n matrices, shape (batch, n, n) (core.py:122-146).

    Holds the caller's numpy array or torch tensor without copying; only the
    shape is checked here.  Symmetry and finiteness are checked by the solve
    (the reference ``validate``, core.py:286-309, runs inside the kernel).
    """

    data: Any

    def __post_init__(self):
        shape = tuple(self.data.shape)
        if len(shape) != 3 or shape[1] != shape[2]:
            raise ShapeMismatch(f"expected (batch, n, n) array, got {shape}")
        if shape[0] < 1 or shape[1] < 1:
            raise ShapeMismatch(f"batch and dim must be positive, got {shape}")

    @property
    def batch(self) -> int:
        return int(self.data.shape[0])

    @property
    def dim(self) -> int:
        return int(self.data.shape[1])


_SORTS = ("descending", "ascending", "none")


@dataclass(frozen=True)
class SolverConfig:
    """Knobs of the batched eigendecomposition (core.py:226-279).

    deflation_tol
        Absolute threshold on the trailing sub-diagonal of the power-of-two
        equilibrated band below which the active block shrinks.  Gated per
        matrix on the device (the reference gates on the batch-wide maximum,
        _kernels.py:303-318, which makes results depend on the batch).
    max_double_steps
        Cap on double-shift iterations per matrix; ``None`` resolves to 2n.
    strict_convergence
        True: exhausting the budget with couplings above threshold raises
        NoConvergence.  False: lock the diagonal as-is (fixed schedule).
    wy_block
        Accepted for API compatibility ("auto", "disabled" or a block size).
        The device path forms P row by row in registers and folds the QR
        rotations straight into it, so no reflector accumulation runs.
    symmetry_tol
        Relative asymmetry tolerated (then symmetrised away).
    """

    deflation_tol: float = 1e-5
    max_double_steps: int | None = None
    compute_vectors: bool = True
    sort: str = "descending"
    wy_block: int | str = "auto"
    symmetry_tol: float = 1e-12
    strict_convergence: bool = True

    def __post_init__(self):
        if self.deflation_tol < 0:
            raise ValueError("deflation_tol must be nonnegative")
        if self.max_double_steps is not None and self.max_double_steps < 1:
            raise ValueError("max_double_steps must be at least 1")
        if self.sort not in _SORTS:
            raise ValueError(f"unknown sort order {self.sort!r}")
        if isinstance(self.wy_block, str):
            if self.wy_block not in ("auto", "disabled"):
                raise ValueError("wy_block must be 'auto', 'disabled', or an int")
        elif self.wy_block < 1:
            raise ValueError("wy_block must be positive when given as a count")

    def resolved_max_steps(self, dim: int) -> int:
        return 2 * dim if self.max_double_steps is None else self.max_double_steps

    def resolved_wy_block(self, dim: int) -> int | None:
        if self.wy_block == "disabled":
            return None
        if self.wy_block == "auto":
            return 4 if dim >= 16 else None
        return None if dim - 2 < 1 else int(self.wy_block)

    @property
    def sort_code(self) -> int:
        return {"none": 0, "descending": 1, "ascending": 2}[self.sort]


@dataclass(frozen=True)
class SolveDiagnostics:
    """Counters of one solve (qr.py:101-118).

    With per-matrix gating every matrix runs its own loop, so the reference's
    counters exist per matrix (``bed_forward_ws_f32``'s ``diag`` output):
    ``converged_steps`` holds each matrix's double-step count,
    ``rotations`` the rotations applied to it (sum of active - 1 over its
    sweeps), ``reduction_counts`` its trailing deflations.  The scalar fields
    pool them over the batch and equal the reference's for a batch of one:
    ``double_steps`` the largest step count, ``rotation_count`` and
    ``reduction_events`` the totals, ``reductions`` the mean number of
    reductions at the start of a double step over all executed double steps
    (the reference's step_r_sum / double_steps, qr.py:578).  -1 where a solve
    did not collect them.
    """

    double_steps: int
    reductions: float
    reduction_events: int
    rotation_count: int
    converged_steps: Any = None
    rotations: Any = None
    reduction_counts: Any = None


@dataclass(frozen=True)
class EigenResult:
    """Batched eigendecomposition output (solver.py:38-57).

    ``eigenvalues`` (batch, n), ordered per the config; ``eigenvectors``
    (batch, n, n) with column j paired to eigenvalue j, or None on the
    values-only path.  Each column's largest-magnitude entry (first on ties)
    is nonnegative.  numpy inputs give float64 numpy outputs (as the
    reference does); torch inputs give float32 tensors on the input's device.
    """

    eigenvalues: Any
    eigenvectors: Any
    diagnostics: SolveDiagnostics

    def __post_init__(self):
        if isinstance(self.eigenvalues, np.ndarray):
            object.__setattr__(self, "eigenvalues", np.asarray(self.eigenvalues, np.float64))
            if self.eigenvectors is not None:
                object.__setattr__(self, "eigenvectors",
                                   np.asarray(self.eigenvectors, np.float64))
