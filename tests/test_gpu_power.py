"""GPU parity of the spectral power (bed_matrix_power_f32) and ZCA whitening
 against the float64 restatement oracle.matrix_power
of the reference matrix_power (solver.py:115-143), plus the reference's own
known answers for matrix_power / zca_whiten (pkg/tests/test_solver.py:139-260)
at FP32 tolerances."""

import numpy as np
import pytest
import torch

import oracle
import parity as P

pytestmark = pytest.mark.gpu

ROOT_HALF = np.sqrt(0.5)


@pytest.fixture(scope="module")
def bed():
    import paper_2207_04228_b200 as bed

    return bed


def _cov(b, n, m, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((b, n, m))
    x = x - x.mean(axis=2, keepdims=True)
    c = x @ x.transpose(0, 2, 1) / m + 1e-3 * np.eye(n)
    return ((c + c.transpose(0, 2, 1)) / 2).astype(np.float32)


@pytest.mark.parametrize("n", [2, 3, 4, 5, 8, 12, 16, 24, 32, 40, 64])
@pytest.mark.parametrize("p", [-0.5, 0.5, 1.0, 2.0, -1.0, 0.3])
def test_power_matches_oracle_on_same_decomposition(bed, n, p):
    a = _cov(37, n, 4 * n, 100 + n)
    e = bed.batched_eig(torch.from_numpy(a).cuda(), bed.SolverConfig(deflation_tol=3e-12))
    out = bed.matrix_power(e, p).data.cpu().numpy().astype(np.float64)
    ref, bad = oracle.matrix_power(e.eigenvectors.cpu().numpy(), e.eigenvalues.cpu().numpy(), p)
    assert not bad.any()
    err = np.linalg.norm(out - ref, axis=(1, 2)) / np.linalg.norm(ref, axis=(1, 2))
    assert err.max() <= 1e-5, err.max()
    np.testing.assert_array_equal(out, out.transpose(0, 2, 1))  # symmetrised (solver.py:141)


def test_power_default_and_explicit_floor(bed):
    lam = torch.tensor([[1.0, 1e-30], [4.0, -2.0]], device="cuda")
    V = torch.eye(2, device="cuda").expand(2, 2, 2).contiguous()
    e = bed.EigenResult(lam, V, bed.SolveDiagnostics(0, -1.0, -1, -1, None))
    out = bed.matrix_power(e, -0.5).data.cpu().numpy()  # floor 1e-12 * lambda_max
    assert np.isfinite(out).all()
    assert out[0, 1, 1] == pytest.approx(1e6, rel=1e-6)
    assert out[1, 1, 1] == pytest.approx((4e-12) ** -0.5, rel=1e-6)
    with pytest.raises(bed.NonPositiveSpectrum) as err:
        bed.matrix_power(e, -0.5, floor=0.0)
    assert err.value.batch_index == 1
    assert err.value.min_eigenvalue == pytest.approx(-2.0)
    sq = bed.matrix_power(e, 2.0, floor=0.0).data.cpu().numpy()  # integer powers: no check
    np.testing.assert_allclose(sq[1], np.diag([16.0, 0.0]), rtol=1e-6)  # max(-2, 0)^2


# ---- the reference's known answers (pkg/tests/test_solver.py), FP32 tolerances


def test_identity_inverse_root(bed):
    e = bed.batched_eig(bed.BatchedSymmetric(np.eye(4)[None]))
    np.testing.assert_allclose(bed.matrix_power(e, -0.5).data[0], np.eye(4), atol=1e-6)


def test_square_root_of_diagonal(bed):
    e = bed.batched_eig(bed.BatchedSymmetric(np.diag([4.0, 9.0])[None]))
    np.testing.assert_allclose(bed.matrix_power(e, 0.5).data[0], np.diag([2.0, 3.0]), atol=1e-6)


def test_inverse_root_identity_check(bed):
    rng = np.random.default_rng(6)
    raw = rng.standard_normal((16, 6, 6))
    spd = raw @ raw.transpose(0, 2, 1) + 6 * np.eye(6)
    e = bed.batched_eig(bed.BatchedSymmetric(spd), bed.SolverConfig(deflation_tol=3e-12))
    r = bed.matrix_power(e, -0.5).data
    resid = np.linalg.norm(r @ spd @ r - np.eye(6), axis=(1, 2))
    assert resid.max() <= 1e-5


def test_first_power_reproduces(bed):
    rng = np.random.default_rng(7)
    raw = rng.standard_normal((8, 5, 5))
    spd = raw @ raw.transpose(0, 2, 1) + 5 * np.eye(5)
    e = bed.batched_eig(bed.BatchedSymmetric(spd), bed.SolverConfig(deflation_tol=3e-12))
    out = bed.matrix_power(e, 1.0).data
    resid = np.linalg.norm(out - spd, axis=(1, 2)) / np.linalg.norm(spd, axis=(1, 2))
    assert resid.max() <= 1e-5


def test_square_root_consistency(bed):
    rng = np.random.default_rng(8)
    raw = rng.standard_normal((8, 7, 7))
    spd = raw @ raw.transpose(0, 2, 1) + 7 * np.eye(7)
    e = bed.batched_eig(bed.BatchedSymmetric(spd), bed.SolverConfig(deflation_tol=3e-12))
    half = bed.matrix_power(e, 0.5).data
    resid = np.linalg.norm(half @ half - spd, axis=(1, 2)) / np.linalg.norm(spd, axis=(1, 2))
    assert resid.max() <= 1e-5


def test_requires_vectors_and_valid_floor(bed):
    e = bed.batched_eig(bed.BatchedSymmetric(np.eye(3)[None]), bed.SolverConfig(compute_vectors=False))
    with pytest.raises(ValueError):
        bed.matrix_power(e, 0.5)
    e = bed.batched_eig(bed.BatchedSymmetric(np.eye(2)[None]))
    with pytest.raises(ValueError):
        bed.matrix_power(e, 0.5, floor=-1.0)


def test_zca_single_channel_unit_variance(bed):
    out = bed.zca_whiten(bed.BatchedMatrix(np.array([[[1.0, -1.0]]])), 0.0)
    np.testing.assert_allclose(out.data[0, 0], [ROOT_HALF, -ROOT_HALF], rtol=1e-6)


def test_zca_recomputed_covariance_is_identity(bed):
    rng = np.random.default_rng(11)
    x = bed.BatchedMatrix(rng.standard_normal((4, 8, 256)))
    out = bed.zca_whiten(x, 1e-5)
    centered = out.data - out.data.mean(axis=2, keepdims=True)
    cov = centered @ centered.transpose(0, 2, 1)
    assert np.abs(cov - np.eye(8)).max() <= 1e-4


def test_zca_device_tensor_stays_on_device(bed):
    x = torch.randn(16, 16, 64, device="cuda")
    out = bed.zca_whiten(x, 1e-3).data
    assert out.is_cuda and out.shape == x.shape
    c = out - out.mean(dim=2, keepdim=True)
    cov = (c @ c.transpose(1, 2)).cpu().numpy()
    # eps_reg shrinks the whitened scatter slightly below I
    assert np.abs(cov - np.eye(16)).max() <= 1e-2


# ---- covariance producer (bed_scatter_f32)


@pytest.mark.parametrize("n,m", [(1, 5), (3, 7), (4, 64), (7, 33), (16, 64), (24, 100), (32, 31),
                                 (40, 256), (64, 256), (64, 70)])
@pytest.mark.parametrize("eps", [0.0, 1e-3])
def test_scatter_matches_float64(bed, n, m, eps):
    rng = np.random.default_rng(n * 1000 + m)
    x = (rng.standard_normal((9, n, m)) * 3.0 + rng.standard_normal((9, n, 1)) * 10.0).astype(np.float32)
    out = bed.scatter_matrices(torch.from_numpy(x).cuda(), eps).cpu().numpy().astype(np.float64)
    xc = x.astype(np.float64) - x.astype(np.float64).mean(axis=2, keepdims=True)
    ref = xc @ xc.transpose(0, 2, 1)
    ref = (ref + ref.transpose(0, 2, 1)) / 2 + eps * np.eye(n)
    err = np.linalg.norm(out - ref, axis=(1, 2)) / np.linalg.norm(ref, axis=(1, 2))
    assert err.max() <= 1e-5, err.max()
    np.testing.assert_array_equal(out, out.transpose(0, 2, 1))


@pytest.mark.parametrize("n", [1, 3, 4, 5, 8, 12, 16, 32, 64])
def test_scatter_full_ctas(bed, n):
    """Batches that fill every matrix slot of the producer's CTAs (128 / (n/4)^2
    matrices per CTA for n <= 32) -- each (matrix, channel) row sum has an owner."""
    m = 2 * n + 3
    b = 1024 if n <= 32 else 300
    rng = np.random.default_rng(n)
    x = (rng.standard_normal((b, n, m)) * 2.0 + rng.standard_normal((b, n, 1)) * 5.0).astype(np.float32)
    out = bed.scatter_matrices(torch.from_numpy(x).cuda(), 1e-3).cpu().numpy().astype(np.float64)
    xc = x.astype(np.float64) - x.astype(np.float64).mean(axis=2, keepdims=True)
    ref = xc @ xc.transpose(0, 2, 1)
    ref = (ref + ref.transpose(0, 2, 1)) / 2 + 1e-3 * np.eye(n)
    err = np.linalg.norm(out - ref, axis=(1, 2)) / np.linalg.norm(ref, axis=(1, 2))
    assert err.max() <= 1e-5, (err.max(), int(err.argmax()))


@pytest.mark.parametrize("n", [4, 8, 16])
def test_zca_large_batch(bed, n):
    b, m = 2048, 8 * n
    x = torch.randn(b, n, m, device="cuda", generator=torch.Generator(device="cuda").manual_seed(n))
    out = bed.zca_whiten(x, 1e-4).data
    c = out.double() - out.double().mean(dim=2, keepdim=True)
    cov = c @ c.transpose(1, 2)
    # eps_reg shrinks the whitened scatter slightly below I
    assert float((cov - torch.eye(n, device="cuda", dtype=torch.float64)).abs().max()) <= 2e-2


# ---- backward through f(lambda) (SpectralPowerFn)


def _sep_spd(b, n, ratio, seed):
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((b, n, n)))
    lam = 2.0 * ratio ** np.arange(n)
    a = (q * lam[None, None, :]) @ q.transpose(0, 2, 1)
    return ((a + a.transpose(0, 2, 1)) / 2).astype(np.float32)


@pytest.mark.parametrize("n,p", [(4, -0.5), (8, 0.5), (16, -0.5), (16, 2.0), (32, -1.0)])
def test_spectral_power_gradient_matches_exact_autograd_at_large_degree(bed, n, p):
    """Degree -> large: the Taylor-K chain equals exact float64 autograd of
    V diag(lambda^p) V^T through torch.linalg.eigh."""
    b = 24
    a = _sep_spd(b, n, 0.8 if n <= 16 else 0.9, n)  # condition <= ~30: FP32 error x cond^|p| stays small
    at = torch.from_numpy(a).cuda().requires_grad_(True)
    y = bed.spectral_power(at, p, bed.SolverConfig(deflation_tol=3e-12), floor=0.0, degree=300)
    gy = torch.randn_like(y)
    (y * gy).sum().backward()
    ad = torch.from_numpy(a.astype(np.float64)).requires_grad_(True)
    lam, v = torch.linalg.eigh(ad)
    yd = (v * lam.pow(p)[:, None, :]) @ v.transpose(1, 2)
    np.testing.assert_allclose(y.detach().cpu().numpy(), yd.detach().numpy(), rtol=0, atol=1e-4 * float(yd.abs().max()))
    (yd * gy.double().cpu()).sum().backward()
    err = P.grad_err(at.grad.cpu().numpy(), ad.grad.numpy())
    assert err.max() <= 1e-3, err.max()


@pytest.mark.parametrize("n", [4, 16, 64])
def test_spectral_power_gradient_matches_oracle_chain(bed, n):
    """Degree 9 (the paper's): the same chain restated in float64 --
    gV = (gY + gY^T) V f, gLambda = f' o diag(V^T gY V), then
    oracle.taylor_backward."""
    b, p = 33, -0.5
    rng = np.random.default_rng(n)
    x = rng.standard_normal((b, n, 4 * n))
    x = x - x.mean(axis=2, keepdims=True)
    a = (x @ x.transpose(0, 2, 1) / (4 * n) + 1e-3 * np.eye(n)).astype(np.float32)
    a = (a + a.transpose(0, 2, 1)) / 2
    at = torch.from_numpy(a).cuda().requires_grad_(True)
    y = bed.spectral_power(at, p, bed.SolverConfig(deflation_tol=3e-12), floor=0.0)
    gy = torch.randn_like(y)
    (y * gy).sum().backward()
    r = bed.batched_eig(torch.from_numpy(a).cuda(), bed.SolverConfig(deflation_tol=3e-12))
    v = r.eigenvectors.cpu().numpy().astype(np.float64)
    lam = r.eigenvalues.cpu().numpy().astype(np.float64)
    g = gy.cpu().numpy().astype(np.float64)
    f, df = lam ** p, p * lam ** (p - 1)
    gv = ((g + g.transpose(0, 2, 1)) @ v) * f[:, None, :]
    gl = np.diagonal(v.transpose(0, 2, 1) @ g @ v, axis1=1, axis2=2) * df
    ref = oracle.taylor_backward(v, lam, gv, gl)
    assert P.grad_err(at.grad.cpu().numpy(), ref).max() <= 1e-4


# ---- eigenvalues + spectral power in one call (bed_forward_power_f32; fused for n <= 8)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 8, 9, 16, 24, 40])
@pytest.mark.parametrize("p", [-0.5, 0.5, 2.0, -1.0, 0.3])
def test_power_of_matches_two_step_path(bed, n, p):
    a = torch.from_numpy(_cov(300, n, 4 * n, 300 + n)).cuda()
    cfg = bed.SolverConfig(deflation_tol=3e-12)
    got = bed.power_of(a, p, cfg).cpu().numpy().astype(np.float64)
    e = bed.batched_eig(a, cfg)
    ref, bad = oracle.matrix_power(e.eigenvectors.cpu().numpy(), e.eigenvalues.cpu().numpy(), p)
    assert not bad.any()
    err = np.linalg.norm(got - ref, axis=(1, 2)) / np.linalg.norm(ref, axis=(1, 2))
    assert err.max() <= 1e-5, err.max()
    np.testing.assert_array_equal(got, got.transpose(0, 2, 1))


@pytest.mark.parametrize("n", [4, 16])
def test_power_of_errors_and_default_floor(bed, n):
    a = np.stack([np.eye(n, dtype=np.float32)] * 5)
    a[3] *= -1.0  # negative spectrum
    at = torch.from_numpy(a).cuda()
    with pytest.raises(bed.NonPositiveSpectrum) as err:
        bed.power_of(at, -0.5, floor=0.0)
    assert err.value.batch_index == 3
    sq = bed.power_of(at, 2.0, floor=0.0).cpu().numpy()  # integer power: no check
    np.testing.assert_allclose(sq[3], np.zeros((n, n)), atol=0)  # max(-1, 0)^2
    bad = a.copy()
    bad[1, 0, 1] = np.nan
    with pytest.raises(bed.NonFinite):
        bed.power_of(torch.from_numpy(bad).cuda(), 0.5)
    # the differentiable entry takes the fused path when no gradient is needed
    x = torch.from_numpy(_cov(64, n, 4 * n, 5)).cuda()
    with torch.no_grad():
        y = bed.spectral_power(x, -0.5)
    np.testing.assert_allclose(y.cpu().numpy(), bed.power_of(x, -0.5).cpu().numpy(), rtol=0, atol=0)


# ---- covariance -> ED [-> power] in one call (bed_scatter_forward_f32; one kernel for n <= 8)


def _samples(b, n, m, seed):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((b, n, m)) * 2.0 + rng.standard_normal((b, n, 1)) * 5.0).astype(np.float32)


def _scatter64(x, eps):
    xc = x.astype(np.float64) - x.astype(np.float64).mean(axis=2, keepdims=True)
    s = xc @ xc.transpose(0, 2, 1)
    return (s + s.transpose(0, 2, 1)) / 2 + eps * np.eye(x.shape[1])


@pytest.mark.parametrize("n,m", [(1, 1), (1, 6), (2, 3), (3, 12), (4, 16), (4, 17), (5, 20), (6, 8),
                                 (7, 29), (8, 32), (8, 5), (9, 36), (16, 64), (24, 50), (40, 160)])
def test_scatter_eig_matches_float64(bed, n, m):
    b, eps = 333, 1e-2  # 333: a partial last CTA
    x = _samples(b, n, m, 7 * n + m)
    cfg = bed.SolverConfig(deflation_tol=3e-12, max_double_steps=4 * n)
    lam, v = bed.scatter_eig(torch.from_numpy(x).cuda(), eps, cfg)
    lam, v = lam.cpu().numpy().astype(np.float64), v.cpu().numpy().astype(np.float64)
    s = _scatter64(x, eps)
    ref = np.linalg.eigvalsh(s)[:, ::-1]
    scale = np.linalg.norm(s, axis=(1, 2))
    assert (np.abs(lam - ref).max(axis=1) / scale).max() <= 1e-5
    rec = (v * lam[:, None, :]) @ v.transpose(0, 2, 1)
    assert (np.linalg.norm(rec - s, axis=(1, 2)) / scale).max() <= 2e-5
    eye = np.eye(n)
    assert np.abs(v.transpose(0, 2, 1) @ v - eye).max() <= 1e-5
    # evals-only and the A-input path agree with the fused one on the same X
    cfg = bed.SolverConfig(deflation_tol=3e-12, max_double_steps=4 * n, compute_vectors=False)
    lam2, v2 = bed.scatter_eig(torch.from_numpy(x).cuda(), eps, cfg)
    assert v2 is None
    np.testing.assert_allclose(lam2.cpu().numpy(), lam, rtol=0, atol=1e-5 * scale.max())


@pytest.mark.parametrize("n,m", [(1, 4), (2, 9), (3, 12), (4, 16), (4, 31), (6, 24), (8, 32),
                                 (8, 64), (12, 48), (16, 64), (32, 128), (48, 192)])
@pytest.mark.parametrize("p", [-0.5, 0.5, -1.0])
def test_scatter_power_matches_float64(bed, n, m, p):
    b, eps = 200, 1e-1
    x = _samples(b, n, m, 11 * n + m)
    cfg = bed.SolverConfig(deflation_tol=3e-12, max_double_steps=4 * n)
    got = bed.scatter_power(torch.from_numpy(x).cuda(), p, eps, cfg, floor=0.0).cpu().numpy()
    s = _scatter64(x, eps)
    w, q = np.linalg.eigh(s)
    ref = (q * w[:, None, :] ** p) @ q.transpose(0, 2, 1)
    err = np.linalg.norm(got.astype(np.float64) - ref, axis=(1, 2)) / np.linalg.norm(ref, axis=(1, 2))
    cond = w[:, -1] / w[:, 0]
    # FP32 (3xTF32 products for n > 32): input rounding of S amplified by the
    # condition number (to the |p|-ish power)
    assert (err / (1.0 + cond) ** max(abs(p), 0.5)).max() <= 5e-6, (err.max(), cond.max())
    np.testing.assert_array_equal(got, got.transpose(0, 2, 1))


@pytest.mark.parametrize("n", [3, 4, 8, 16])
def test_scatter_power_equals_composed_path(bed, n):
    """The fused call and scatter_matrices -> power_of on the same X: same
    matrix up to the producer's rounding (both shift by the first sample).
    Budget 4n (the reference's verify profile, bench.py:227-228): under the
    default 2n a few of these scatters need 7 double steps at n = 3 -- the
    float64 oracle too (oracle.forward(max_double_steps=6) reports them)."""
    x = torch.from_numpy(_samples(500, n, 8 * n, n)).cuda()
    cfg = bed.SolverConfig(deflation_tol=3e-12, max_double_steps=4 * n)
    fused = bed.scatter_power(x, -0.5, 1e-2, cfg, floor=0.0)
    composed = bed.power_of(bed.scatter_matrices(x, 1e-2), -0.5, cfg, floor=0.0)
    err = torch.linalg.matrix_norm((fused - composed).double()) / torch.linalg.matrix_norm(composed.double())
    assert float(err.max()) <= 1e-4


@pytest.mark.parametrize("n", [4, 7, 16])
def test_scatter_forward_layouts_and_errors(bed, n):
    m = 4 * n
    base = torch.from_numpy(_samples(65, n, m + 1, n)).cuda()
    # misaligned, non-multiple-of-4 rows: X a view one float in (the scalar load path)
    flat = torch.empty(65 * n * m + 1, device="cuda")
    flat[1:] = base[:, :, :m].reshape(-1)
    xm = flat[1:].view(65, n, m)
    cfg = bed.SolverConfig(deflation_tol=3e-12, max_double_steps=4 * n)
    a, _ = bed.scatter_eig(xm, 1e-2, cfg)
    b_, _ = bed.scatter_eig(base[:, :, :m].contiguous(), 1e-2, cfg)
    torch.testing.assert_close(a, b_, rtol=0, atol=1e-5 * float(b_.abs().max()))
    # empty batch
    lam, v = bed.scatter_eig(torch.empty(0, n, m, device="cuda"), 0.0)
    assert lam.shape == (0, n) and v.shape == (0, n, n)
    # a NaN sample: NonFinite at its (channel, sample) position, first bad matrix
    bad = base[:, :, :m].contiguous()
    bad[40, n - 1, 3] = float("nan")
    bad[50, 0, 0] = float("inf")
    with pytest.raises(bed.NonFinite) as err:
        bed.scatter_power(bad, -0.5, 1e-2)
    assert err.value.batch_index == 40 and tuple(err.value.position) == (n - 1, 3)
    # one sample, eps = 0: the scatter is exactly zero -- no positive spectrum for the inverse root
    with pytest.raises(bed.NonPositiveSpectrum):
        bed.scatter_power(base[:, :, :1].contiguous(), -0.5, 0.0, floor=0.0)
    with pytest.raises(ValueError):
        bed.scatter_eig(base, -1.0)
