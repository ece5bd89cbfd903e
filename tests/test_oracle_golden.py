"""Pin the CPU oracle (oracle/bed_oracle.c) against the reference's own
outputs, committed as golden fixtures by tests/golden/make_golden.py.

Batch-gated oracle vs reference batched_eig: eigenvalues and diagnostics
bit-exact (same float64 arithmetic), eigenvectors within 1e-12 (the reference
forms P and V=PQ through BLAS matmuls, the oracle through plain loops).
"""

import numpy as np
import pytest

import os

import oracle


_CELLS = sorted({k.split("/")[0] for k in np.load(os.path.join(os.path.dirname(__file__), "golden", "cells.npz")).files if k.endswith("/a")})


def _profile(pname, n):
    return (1e-5, 2 * n) if pname == "default" else (3e-12, 4 * n)


@pytest.mark.parametrize("name", _CELLS)
@pytest.mark.parametrize("pname", ["default", "verify"])
def test_batch_gate_matches_reference(cells, name, pname):
    a = cells[f"{name}/a"].astype(np.float64)
    b, n, _ = a.shape
    tol, steps = _profile(pname, n)
    r = oracle.forward(a, deflation_tol=tol, max_double_steps=steps, strict=False,
                       gate=oracle.GATE_BATCH)
    np.testing.assert_array_equal(r.eigenvalues, cells[f"{name}/{pname}/evals"])
    key = f"{name}/{pname}/evecs"
    if key in cells:
        np.testing.assert_allclose(r.eigenvectors, cells[key], rtol=0, atol=1e-12)
    if n >= 3:
        assert int(r.double_steps[0]) == int(cells[f"{name}/{pname}/double_steps"])
        assert int(r.rotations[0]) == int(cells[f"{name}/{pname}/rotations"])
        np.testing.assert_array_equal(r.converged_steps, cells[f"{name}/{pname}/converged"])


@pytest.mark.parametrize("name", _CELLS)
@pytest.mark.parametrize("pname", ["default", "verify"])
def test_matrix_gate_matches_reference_batch_of_one(cells, name, pname):
    a = cells[f"{name}/a"].astype(np.float64)
    solo = cells[f"{name}/{pname}/solo_evals"]
    k = solo.shape[0]
    n = a.shape[1]
    tol, steps = _profile(pname, n)
    r = oracle.forward(a[:k], deflation_tol=tol, max_double_steps=steps, strict=False,
                       gate=oracle.GATE_MATRIX, threads=2, chunk=3)
    np.testing.assert_array_equal(r.eigenvalues, solo)
    if n >= 3:
        np.testing.assert_array_equal(r.double_steps, cells[f"{name}/{pname}/solo_steps"])
    key = f"{name}/{pname}/solo_evecs"
    if key in cells:
        np.testing.assert_allclose(r.eigenvectors, cells[key], rtol=0, atol=1e-12)


def test_values_only_and_ascending(cells):
    a = cells["n8_b64/a"].astype(np.float64)
    r = oracle.forward(a, deflation_tol=3e-12, max_double_steps=32, compute_vectors=False,
                       gate=oracle.GATE_BATCH)
    assert r.eigenvectors is None
    np.testing.assert_array_equal(r.eigenvalues, cells["n8_b64/values_only/evals"])
    r = oracle.forward(a, deflation_tol=3e-12, max_double_steps=32, sort="ascending",
                       gate=oracle.GATE_BATCH)
    np.testing.assert_array_equal(r.eigenvalues, cells["n8_b64/ascending/evals"])
    np.testing.assert_allclose(r.eigenvectors, cells["n8_b64/ascending/evecs"], atol=1e-12)


def test_known_answers(known):
    r = oracle.forward(known["diag123/a"], deflation_tol=1e-5, max_double_steps=6)
    np.testing.assert_array_equal(r.eigenvalues, known["diag123/evals"])
    np.testing.assert_array_equal(r.eigenvectors, known["diag123/evecs"])
    r = oracle.forward(known["classic2x2/a"], deflation_tol=1e-5, max_double_steps=4)
    np.testing.assert_allclose(r.eigenvalues, known["classic2x2/evals"], rtol=1e-15)
    np.testing.assert_allclose(r.eigenvectors, known["classic2x2/evecs"], rtol=1e-15)
    for abd, (lo, hi) in zip(known["wilkinson/abd"], known["wilkinson/lo_hi"]):
        got = oracle.wilkinson(*abd)
        assert got[0] == lo and got[1] == hi
    for name in ("hh345", "hhm345", "ones4"):
        w, vec = oracle.tridiagonalize(known[f"{name}/a"])
        np.testing.assert_allclose(vec[:, 0], known[f"{name}/u"], atol=1e-15)
        if name != "ones4":
            # one reflection of a 3x3 is the whole reduction
            np.testing.assert_allclose(w, known[f"{name}/after"], atol=1e-14)


def test_validation_statuses():
    a = np.stack([np.eye(3), np.eye(3), np.eye(3)])
    a[1, 0, 1] = np.nan
    a[2, 0, 1] = 1.0  # asymmetric
    r = oracle.forward(a)
    assert list(r.status) == [0, 2, 3]


def test_gen_spd_restatement_is_seeded_and_spd():
    a = oracle.gen_spd(16, 5, 3)
    b = oracle.gen_spd(16, 5, 3)
    assert np.array_equal(a, b)
    assert np.array_equal(a, a.transpose(0, 2, 1))
    assert np.linalg.eigvalsh(a).min() > 0
