"""B200-native batched symmetric eigendecomposition (arXiv 2207.04228).

Drop-in for the reference ``batchedeig`` forward API on the GPU (same
names: ``batched_eig``, ``SolverConfig``, ``EigenResult``, ``BatchedSymmetric``
and the error types), plus the differentiable ``eigh`` / ``BatchedEigFn``
with the paper's Taylor-polynomial backward.  All compute runs in the
sm_100a kernels of ``_lib/libbed200.so`` (C ABI: ``include/bed200.h``).
"""

from .core import (  # noqa: F401
    BadMagic,
    BatchedEigError,
    DimMismatch,
    TruncatedPayload,
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
from .solver import (  # noqa: F401
    TAYLOR_DEGREE,
    BatchedEigFn,
    batched_eig,
    eigh,
    forward_into,
    matrix_power,
    power_of,
    scatter_matrices,
    scatter_eig,
    scatter_power,
    spectral_power,
    SpectralPowerFn,
    taylor_backward,
    workspace,
    zca_whiten,
)
from .bed_io import read_batch, read_matrix, write_batch  # noqa: F401
from .sharding import (  # noqa: F401
    batched_eig_devices,
    gather_shards,
    shard_bounds,
    shard_sizes,
    solve_shard,
)

__version__ = "0.1.0"
