"""The float64 host entry bed_forward_host_f64 -- the path batched_eig takes for
the reference's own input (a float64 numpy batch, solver.py:79-112): host-thread
validation in float64 (core.py:286-309), FP32 staging, chunks streamed through
the device.  Results must equal the device path on the same symmetrised FP32
matrices bit for bit; errors must follow the reference's order."""

import numpy as np
import pytest
import torch

import oracle
import parity as P

pytestmark = pytest.mark.gpu

VERIFY = dict(deflation_tol=3e-12)


@pytest.fixture(scope="module")
def bed():
    import paper_2207_04228_b200 as bed

    return bed


def _host64(bed, a, cfg, threads=0):
    from paper_2207_04228_b200 import _native

    b, n, _ = a.shape
    lam = np.full((b, n), np.nan)
    vec = np.full((b, n, n), np.nan) if cfg.compute_vectors else None
    st = np.full(b, -1, np.int32)
    k = np.full(b, -1, np.int32)
    dg = np.full((b, 3), -1, np.int32)
    rs = np.full(b, np.nan, np.float32)
    _native.forward_host_f64(a.ctypes.data, b, n, lam.ctypes.data,
                             vec.ctypes.data if vec is not None else None, st.ctypes.data,
                             k.ctypes.data, dg.ctypes.data, rs.ctypes.data,
                             _native.make_config(cfg, n), 0, threads)
    return lam, vec, st, k, dg, rs


def _device(bed, a64, cfg):
    sym = ((a64 + a64.transpose(0, 2, 1)) / 2).astype(np.float32)
    lam, vec, st, k, dg = bed.solver._solve_device(torch.from_numpy(sym).cuda(), cfg, check=False,
                                                   diagnostics=True)
    return (lam.cpu().numpy(), None if vec is None else vec.cpu().numpy(), st.cpu().numpy(),
            k.cpu().numpy(), dg.cpu().numpy())


# multi-chunk batches at the default 32 MB chunk: n = 4 -> ~195 K matrices per
# chunk, n = 16 -> ~15.7 K, n = 64 -> ~1 K (a workspace per staging slot)
@pytest.mark.parametrize("n,b", [(1, 7), (3, 1000), (4, 500_000), (8, 70_000), (9, 5000),
                                 (16, 40_000), (33, 3000), (64, 2500)])
def test_host_f64_equals_device_path_bitwise(bed, n, b):
    a = oracle.gen_spd(b, n, 40 + n)
    cfg = bed.SolverConfig(max_double_steps=4 * n, **VERIFY)
    lam, vec, st, k, dg, rs = _host64(bed, a, cfg)
    dl, dv, ds, dk, ddg = _device(bed, a, cfg)
    np.testing.assert_array_equal(lam, dl.astype(np.float64))
    np.testing.assert_array_equal(vec, dv.astype(np.float64))
    np.testing.assert_array_equal(st, ds)
    np.testing.assert_array_equal(k, dk)
    np.testing.assert_array_equal(dg, ddg)
    assert np.isfinite(rs).all()


def test_host_f64_values_only_and_thread_counts(bed):
    n, b = 12, 30_000
    a = oracle.gen_spd(b, n, 3)
    cfg = bed.SolverConfig(max_double_steps=4 * n, **VERIFY)
    full = _host64(bed, a, cfg)
    one = _host64(bed, a, cfg, threads=1)
    for x, y in zip(full, one):
        np.testing.assert_array_equal(x, y)
    vals = _host64(bed, a, bed.SolverConfig(max_double_steps=4 * n, compute_vectors=False, **VERIFY))
    assert vals[1] is None
    o = oracle.forward(a[:64], max_double_steps=4 * n)
    assert np.all(P.eig_err(vals[0][:64], o.eigenvalues) <= P.EIG_TOL)


@pytest.mark.parametrize("n", [4, 16])
def test_host_f64_statuses_and_reference_error_order(bed, n):
    b = 300
    a = oracle.gen_spd(b, n, 9)
    cfg = bed.SolverConfig(max_double_steps=4 * n, **VERIFY)
    clean = _host64(bed, a, cfg)
    bad = a.copy()
    bad[200, 1, 0] = np.nan     # later in the batch, but finiteness is checked first
    bad[17, 0, n - 1] += 1e-3   # asymmetric
    lam, vec, st, _, _, _ = _host64(bed, bad, cfg)
    assert st[200] == 2 and st[17] == 3
    ok = np.ones(b, bool)
    ok[[17, 200]] = False
    np.testing.assert_array_equal(lam[ok], clean[0][ok])
    np.testing.assert_array_equal(vec[ok], clean[1][ok])
    zero = _device(bed, np.zeros((1, n, n)), cfg)  # a rejected matrix solves as the zero matrix
    np.testing.assert_array_equal(lam[17], zero[0][0])
    np.testing.assert_array_equal(vec[200], zero[1][0])
    with pytest.raises(bed.NonFinite) as err:
        bed.batched_eig(bed.BatchedSymmetric(bad), cfg)
    assert err.value.batch_index == 200 and err.value.position == (1, 0)
    bad[200, 1, 0] = a[200, 1, 0]
    with pytest.raises(bed.NonSymmetric) as err:
        bed.batched_eig(bed.BatchedSymmetric(bad), cfg)
    assert err.value.batch_index == 17
    assert err.value.max_asymmetry == pytest.approx(np.abs(bad[17] - bad[17].T).max())
    # asymmetry within symmetry_tol * max(1, ||A||_F) is folded away in float64
    tiny = a.copy()
    tiny[:, 0, 1] *= 1 + 1e-15
    r = bed.batched_eig(bed.BatchedSymmetric(tiny), cfg)
    assert np.all(P.eig_err(r.eigenvalues, clean[0]) <= P.EIG_TOL)


def test_host_f64_no_convergence_payload(bed):
    """strict: NoConvergence lists the offenders and the largest coupling left."""
    n, b = 16, 256
    a = oracle.gen_spd(b, n, 77)
    cfg = bed.SolverConfig(deflation_tol=3e-12, max_double_steps=1)
    with pytest.raises(bed.NoConvergence) as err:
        bed.batched_eig(bed.BatchedSymmetric(a), cfg)
    _, _, st, _, _, rs = _host64(bed, a, cfg)
    idx = np.flatnonzero(st == 1)
    assert list(err.value.batch_indices) == idx.tolist()
    assert err.value.residual_offdiag_max == pytest.approx(float(rs[idx].max()))
    r = bed.batched_eig(bed.BatchedSymmetric(a),
                        bed.SolverConfig(deflation_tol=3e-12, max_double_steps=1,
                                         strict_convergence=False))
    assert r.eigenvalues.shape == (b, n)


def test_integration_stub_runs_as_documented(bed):
    """The ctypes stub of INTEGRATION.md section 2, run verbatim against this
    library: the same results and errors as batched_eig on float64 numpy."""
    import ctypes
    import os
    import re

    from paper_2207_04228_b200 import _native, core

    src = open(os.path.join(os.path.dirname(__file__), "..", "INTEGRATION.md")).read()
    code = re.search(r"```python\n(# batchedeig/_b200\.py.*?)```", src, re.S).group(1)
    code = code.replace("from .core import NoConvergence, NonFinite, NonSymmetric\n", "")
    code = code.replace('ctypes.CDLL("libbed200.so")', "ctypes.CDLL(LIB)")
    ns = {"NoConvergence": core.NoConvergence, "NonFinite": core.NonFinite,
          "NonSymmetric": core.NonSymmetric, "LIB": _native.LIB_PATH, "ctypes": ctypes}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    stub = ns["batched_eig_b200"]
    n, b = 12, 500
    a = oracle.gen_spd(b, n, 4)
    cfg = bed.SolverConfig(max_double_steps=4 * n, **VERIFY)
    lam, vec = stub(bed.BatchedSymmetric(a), cfg)
    r = bed.batched_eig(bed.BatchedSymmetric(a), cfg)
    np.testing.assert_array_equal(lam, r.eigenvalues)
    np.testing.assert_array_equal(vec, r.eigenvectors)
    bad = a.copy()
    bad[7, 2, 3] = np.inf
    with pytest.raises(bed.NonFinite) as err:
        stub(bed.BatchedSymmetric(bad), cfg)
    assert err.value.batch_index == 7 and err.value.position == (2, 3)
