"""CPU tests pinning the backward checker ``oracle.taylor_backward`` (the
reference package has no backward, pkg/README.md:116-117, so the restatement
of PAPER.md:668/:700 is pinned by the known-answer properties of SURVEY.md
8(c) instead):

  (i)   degree -> inf reproduces exact float64 ``torch.linalg.eigh`` autograd
        for well-separated spectra;
  (ii)  linearity in (gV, gLambda);
  (iii) gA is symmetric;
  (iv)  with gV = 0, gA = V diag(gLambda) V^T;
  (v)   equal eigenvalues give the finite F = (K+1)/lambda;
plus the domain rule for spectra the series does not converge on.
"""

import numpy as np
import pytest
import torch

import oracle

NS = [4, 16, 64]


def _spd_geometric(b, n, ratio, seed):
    """Q diag(lam) Q^T with lam_k = 4 * ratio^k: adjacent ratios are `ratio`."""
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((b, n, n)))
    lam = 4.0 * ratio ** np.arange(n)
    a = (q * lam[None, None, :]) @ q.transpose(0, 2, 1)
    return (a + a.transpose(0, 2, 1)) / 2


def _decompose(a):
    lam, v = np.linalg.eigh(a)
    return lam[:, ::-1].copy(), v[:, :, ::-1].copy()  # descending, like the solver


def _eigh_autograd(a, v_ref, gv, gl):
    """float64 torch.linalg.eigh autograd of <V, gV> + <lambda, gL>, with V's
    columns sign-aligned to v_ref and ordered descending."""
    at = torch.tensor(a, dtype=torch.float64, requires_grad=True)
    le, ve = torch.linalg.eigh(at)
    le, ve = le.flip(-1), ve.flip(-1)
    sign = torch.sign((ve.detach() * torch.from_numpy(v_ref)).sum(1, keepdim=True))
    loss = ((ve * sign) * torch.from_numpy(gv)).sum() + (le * torch.from_numpy(gl)).sum()
    loss.backward()
    return at.grad.numpy()


def _rel(x, y):
    return np.linalg.norm(x - y, axis=(1, 2)) / np.linalg.norm(y, axis=(1, 2))


@pytest.mark.parametrize("n", NS)
def test_large_degree_is_exact_eigh_autograd(n):
    b = 8
    ratio = 0.8 if n < 64 else 0.93  # keeps 4 * ratio^(n-1) well above f64 noise
    a = _spd_geometric(b, n, ratio, seed=n)
    lam, v = _decompose(a)
    rng = np.random.default_rng(100 + n)
    gv = rng.standard_normal((b, n, n))
    gl = rng.standard_normal((b, n))
    # the series' tail after K terms is ratio^(K+1) / (1 - ratio)
    degree = int(np.ceil(np.log(1e-14 * (1 - ratio)) / np.log(ratio)))
    got = oracle.taylor_backward(v, lam, gv, gl, degree)
    want = _eigh_autograd(a, v, gv, gl)
    assert _rel(got, want).max() <= 1e-8


@pytest.mark.parametrize("n", NS)
def test_degree_nine_differs_from_exact_as_intended(n):
    """The paper's K = 9 is an approximation: adjacent ratios near 1 are
    truncated (median 4e-4 at n=4 up to 0.21 at n=64)."""
    a = _spd_geometric(4, n, 0.9, seed=7 * n)
    lam, v = _decompose(a)
    rng = np.random.default_rng(n)
    gv = rng.standard_normal((4, n, n))
    err = _rel(oracle.taylor_backward(v, lam, gv, None, 9), _eigh_autograd(a, v, gv, np.zeros((4, n))))
    assert err.min() > 1e-3


@pytest.mark.parametrize("n", NS)
def test_linear_in_cotangents(n):
    b = 6
    lam, v = _decompose(_spd_geometric(b, n, 0.85, seed=2 * n))
    rng = np.random.default_rng(n)
    gv1, gv2 = rng.standard_normal((2, b, n, n))
    gl1, gl2 = rng.standard_normal((2, b, n))
    al, be = 1.75, -0.5
    lhs = oracle.taylor_backward(v, lam, al * gv1 + be * gv2, al * gl1 + be * gl2)
    rhs = al * oracle.taylor_backward(v, lam, gv1, gl1) + be * oracle.taylor_backward(v, lam, gv2, gl2)
    assert _rel(lhs, rhs).max() <= 1e-12


@pytest.mark.parametrize("n", NS)
def test_gradient_is_symmetric(n):
    lam, v = _decompose(_spd_geometric(5, n, 0.9, seed=3 * n))
    rng = np.random.default_rng(n)
    g = oracle.taylor_backward(v, lam, rng.standard_normal((5, n, n)), rng.standard_normal((5, n)))
    np.testing.assert_array_equal(g, g.transpose(0, 2, 1))


@pytest.mark.parametrize("n", NS)
def test_eigenvalue_cotangent_only(n):
    lam, v = _decompose(_spd_geometric(5, n, 0.9, seed=4 * n))
    gl = np.random.default_rng(n).standard_normal((5, n))
    got = oracle.taylor_backward(v, lam, None, gl)
    want = v @ (gl[:, :, None] * v.transpose(0, 2, 1))
    assert _rel(got, want).max() <= 1e-13
    # an all-zero gV contributes nothing either
    got0 = oracle.taylor_backward(v, lam, np.zeros((5, n, n)), gl)
    assert _rel(got0, want).max() <= 1e-13


@pytest.mark.parametrize("degree", [0, 3, 9, 20])
def test_equal_eigenvalues_give_finite_k(degree):
    lam = np.array([[2.0, 2.0, 1.0, 0.5]])
    f = oracle.taylor_k(lam, degree)
    assert np.isfinite(f).all()
    # pair (0, 1): tie, row 0 first by index -> F_01 = -(K+1)/2, F_10 = +(K+1)/2
    assert f[0, 0, 1] == pytest.approx(-(degree + 1) / 2.0, rel=1e-15)
    assert f[0, 1, 0] == pytest.approx((degree + 1) / 2.0, rel=1e-15)
    # separated pair (0, 2): -(1/2) sum_k (1/2)^k
    want = -0.5 * sum(0.5 ** k for k in range(degree + 1))
    assert f[0, 0, 2] == pytest.approx(want, rel=1e-15)
    assert np.all(np.diagonal(f, axis1=1, axis2=2) == 0)


def test_k_is_antisymmetric_and_approximates_inverse_gaps():
    lam = np.array([[5.0, 3.0, 1.0, 0.25]])
    f = oracle.taylor_k(lam, 200)
    np.testing.assert_allclose(f, -f.transpose(0, 2, 1), rtol=0, atol=0)
    gaps = lam[:, None, :] - lam[:, :, None]
    with np.errstate(divide="ignore"):
        exact = np.where(gaps != 0, 1.0 / gaps, 0.0)
    np.testing.assert_allclose(f, exact, rtol=1e-12, atol=0)


def test_outside_the_domain_takes_the_exact_inverse_gap():
    # (-1, -2): l_big <= 0; (3, -4): l_small <= -l_big; (0, 0): zeros; (-1, -1): tie
    lam = np.array([[-1.0, -2.0, 0.5, 0.25], [3.0, -4.0, 1.0, 0.5], [0.0, 0.0, 1.0, 0.5],
                    [2.0, 1.0, 0.5, -0.25], [-1.0, -1.0, -0.5, -3.0]])
    f = oracle.taylor_k(lam, 9)
    assert f[0, 0, 1] == pytest.approx(1.0 / (-2.0 - -1.0))
    assert f[1, 0, 1] == pytest.approx(1.0 / (-4.0 - 3.0))
    assert f[2, 0, 1] == 0.0
    assert f[4, 0, 1] == 0.0
    # (2, -0.25) is inside: |ratio| = 1/8 < 1, the series converges
    assert f[3, 0, 3] == pytest.approx(-(1 / 2.0) * sum((-0.125) ** k for k in range(10)))
    np.testing.assert_array_equal(oracle.taylor_domain(lam), [False, False, True, True, False])
