"""TEST INFRASTRUCTURE -- the CPU oracle for the batched eigendecomposition path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package.  The product package
``paper_2207_04228_b200`` never imports it, and fails loudly when its CUDA
extension is missing instead of falling back here.

Contents
--------
``forward``            float64 C restatement of the reference ``batched_eig``
                       (``oracle/bed_oracle.c``; reference ``solver.py:79-112``).
``taylor_backward``    float64 numpy restatement of the ED backward with the
                       Taylor-polynomial K (paper ``PAPER.md:668``, ``:700``).
                       The reference package has no backward
                       (``pkg/README.md:116-117``): **parity unpinned** against
                       the reference; pinned instead by the known-answer
                       properties in ``tests/test_oracle_backward.py`` (SURVEY.md 8(c)
                       (i)-(v), including degree -> inf against float64
                       ``torch.linalg.eigh`` autograd).
``matrix_power``       float64 restatement of the reference spectral power
                       (``solver.py:115-143``), the checker of
                       ``bed_matrix_power_f32``.
``gen_spd``            restatement of the reference input generator
                       (``bench.py:112-134``), bit-identical to it.
"""

from .oracle import (  # noqa: F401
    GATE_BATCH,
    GATE_MATRIX,
    OracleResult,
    build,
    forward,
    gen_spd,
    library_path,
    matrix_power,
    taylor_backward,
    taylor_domain,
    taylor_k,
    wilkinson,
    tridiagonalize,
)
