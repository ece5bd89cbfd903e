"""CPU checks of the float64 spectral-power restatement oracle.matrix_power
(reference matrix_power, solver.py:115-143) on the reference's own known
answers (pkg/tests/test_solver.py:139-225)."""

import numpy as np

import oracle


def test_identity_and_diagonal_roots():
    out, bad = oracle.matrix_power(np.eye(4)[None], np.ones((1, 4)), -0.5)
    np.testing.assert_allclose(out[0], np.eye(4), atol=1e-14)
    assert not bad.any()
    out, _ = oracle.matrix_power(np.eye(2)[None], np.array([[4.0, 9.0]]), 0.5)
    np.testing.assert_allclose(out[0], np.diag([2.0, 3.0]), atol=1e-14)


def test_floors_and_positivity():
    v = np.eye(2)[None].repeat(2, axis=0)
    w = np.array([[1.0, 1e-30], [2.0, -1.0]])
    out, bad = oracle.matrix_power(v, w, -0.5)  # default floor 1e-12 * lambda_max
    assert np.isfinite(out[0]).all() and out[0, 1, 1] == 1e6
    _, bad = oracle.matrix_power(v, w, -0.5, floor=0.0)
    assert bad.tolist() == [False, True]
    out, bad = oracle.matrix_power(v, w, 2.0, floor=0.0)  # integer power: no check
    assert not bad.any()
    np.testing.assert_allclose(out[1], np.diag([4.0, 0.0]))


def test_reconstruction_and_symmetry():
    rng = np.random.default_rng(7)
    raw = rng.standard_normal((8, 5, 5))
    spd = raw @ raw.transpose(0, 2, 1) + 5 * np.eye(5)
    w, v = np.linalg.eigh(spd)
    out, _ = oracle.matrix_power(v, w, 1.0)
    np.testing.assert_allclose(out, spd, rtol=1e-12, atol=1e-12)
    half, _ = oracle.matrix_power(v, w, 0.5)
    np.testing.assert_array_equal(half, half.transpose(0, 2, 1))
    np.testing.assert_allclose(half @ half, spd, rtol=1e-10, atol=1e-10)
