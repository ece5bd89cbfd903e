"""GPU parity of the Taylor-polynomial ED backward (bed_backward_f32) against
the float64 numpy restatement oracle.taylor_backward, fed the same V,
Lambda and cotangents; plus autograd wiring through BatchedEigFn."""

import numpy as np
import pytest
import torch

import oracle
import parity as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bed():
    import paper_2207_04228_b200 as bed

    return bed


def _cov(b, n, m, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((b, n, m))
    x = x - x.mean(axis=2, keepdims=True)
    c = x @ x.transpose(0, 2, 1) / m + 1e-5 * np.eye(n)
    return ((c + c.transpose(0, 2, 1)) / 2).astype(np.float32)


@pytest.mark.parametrize("n", [2, 3, 4, 7, 8, 12, 16, 24, 32, 40, 64])
@pytest.mark.parametrize("degree", [9, 3])
def test_backward_matches_oracle(bed, n, degree):
    b = 67
    a = _cov(b, n, 4 * n, n)
    r = bed.batched_eig(torch.from_numpy(a).cuda(), bed.SolverConfig(deflation_tol=3e-12))
    lam, v = r.eigenvalues, r.eigenvectors
    rng = np.random.default_rng(17)
    gv = torch.from_numpy(rng.standard_normal((b, n, n)).astype(np.float32)).cuda()
    gl = torch.from_numpy(rng.standard_normal((b, n)).astype(np.float32)).cuda()
    ga = bed.taylor_backward(v, lam, gv, gl, degree).cpu().numpy()
    ref = oracle.taylor_backward(v.cpu().numpy(), lam.cpu().numpy(), gv.cpu().numpy(),
                                 gl.cpu().numpy(), degree)
    err = P.grad_err(ga, ref)
    assert err.max() <= P.GRAD_TOL, err.max()
    np.testing.assert_array_equal(ga, ga.transpose(0, 2, 1))  # symmetric by construction


def test_backward_null_cotangents(bed):
    a = _cov(16, 16, 64, 1)
    r = bed.batched_eig(torch.from_numpy(a).cuda())
    lam, v = r.eigenvalues, r.eigenvectors
    gl = torch.randn(16, 16, device="cuda")
    ga = bed.taylor_backward(v, lam, None, gl).cpu().numpy()
    vn = v.cpu().numpy().astype(np.float64)
    ref = vn @ (gl.cpu().numpy()[:, :, None] * vn.transpose(0, 2, 1))  # V diag(gL) V^T
    assert P.grad_err(ga, ref).max() <= P.GRAD_TOL
    gv = torch.randn(16, 16, 16, device="cuda")
    ga = bed.taylor_backward(v, lam, gv, None).cpu().numpy()
    ref = oracle.taylor_backward(vn, lam.cpu().numpy(), gv.cpu().numpy(), None)
    assert P.grad_err(ga, ref).max() <= P.GRAD_TOL


def test_autograd_through_eigh(bed):
    n, b = 16, 128
    a = torch.from_numpy(_cov(b, n, 64, 3)).cuda().requires_grad_(True)
    lam, v = bed.eigh(a)
    w = torch.randn(b, n, n, device="cuda")
    loss = (v * w).sum() + (lam ** 2).sum()
    loss.backward()
    ref = oracle.taylor_backward(v.detach().cpu().numpy(), lam.detach().cpu().numpy(),
                                 w.cpu().numpy(), (2 * lam).detach().cpu().numpy())
    assert P.grad_err(a.grad.cpu().numpy(), ref).max() <= P.GRAD_TOL


def test_large_degree_approaches_exact_gradient(bed):
    """Well-separated spectrum: degree -> large converges to exact eigh autograd."""
    n, b = 4, 64
    rng = np.random.default_rng(5)
    q, _ = np.linalg.qr(rng.standard_normal((b, n, n)))
    lam = np.tile(np.array([8.0, 4.0, 2.0, 1.0]), (b, 1))
    a = ((q * lam[:, None, :]) @ q.transpose(0, 2, 1)).astype(np.float32)
    a = (a + a.transpose(0, 2, 1)) / 2
    at = torch.from_numpy(a).cuda()
    r = bed.batched_eig(at, bed.SolverConfig(deflation_tol=3e-12))
    gv = torch.randn(b, n, n, device="cuda")
    g200 = bed.taylor_backward(r.eigenvectors, r.eigenvalues, gv, None, 200)
    ad = at.double().requires_grad_(True)
    le, ve = torch.linalg.eigh(ad)  # ascending; flip to descending + same signs
    ve = ve.flip(-1)
    sign = torch.sign((ve * r.eigenvectors.double()).sum(1, keepdim=True))
    ((ve * sign) * gv.double()).sum().backward()
    assert P.grad_err(g200.cpu().numpy(), ad.grad.cpu().numpy()).max() <= 1e-4


@pytest.mark.parametrize("n,b,m", [(16, 65536, 64), (64, 8192, 256)])
def test_backward_full_size_configs(bed, n, b, m):
    """C4 (16 x 16, 65536) and C5 (64 x 64, 8192) at full size: the covariance
    inputs of SURVEY 8(d); the oracle on a sample, symmetry on all."""
    from paper_2207_04228_b200.datagen import covariance_device

    a = covariance_device(b, n, m, n)
    r = bed.batched_eig(a, bed.SolverConfig(deflation_tol=3e-12, max_double_steps=4 * n))
    g = torch.Generator(device="cuda").manual_seed(17)
    gv = torch.randn((b, n, n), device="cuda", generator=g)
    gl = torch.randn((b, n), device="cuda", generator=g)
    ga = bed.taylor_backward(r.eigenvectors, r.eigenvalues, gv, gl, check=True)
    assert torch.equal(ga, ga.transpose(1, 2))
    idx = torch.randperm(b, generator=torch.Generator().manual_seed(2))[:128].cuda()
    ref = oracle.taylor_backward(r.eigenvectors[idx].cpu().numpy(), r.eigenvalues[idx].cpu().numpy(),
                                 gv[idx].cpu().numpy(), gl[idx].cpu().numpy())
    assert P.grad_err(ga[idx].cpu().numpy(), ref).max() <= P.GRAD_TOL


def test_backward_outside_taylor_domain(bed):
    """Indefinite / non-positive spectra: pairs outside the series' domain take
    the exact 1/(l_j - l_i) and the matrix is flagged (NonPositiveSpectrum
    with check=True); the oracle applies the same rule."""
    n, b = 6, 40
    rng = np.random.default_rng(9)
    q, _ = np.linalg.qr(rng.standard_normal((b, n, n)))
    lam = np.sort(rng.uniform(-3.0, 3.0, (b, n)), axis=1)[:, ::-1]
    lam[:4] = np.abs(lam[:4]) + 0.5  # the first four are SPD
    a = ((q * lam[:, None, :]) @ q.transpose(0, 2, 1)).astype(np.float32)
    a = (a + a.transpose(0, 2, 1)) / 2
    r = bed.batched_eig(torch.from_numpy(a).cuda(), bed.SolverConfig(deflation_tol=3e-12))
    gv = torch.from_numpy(rng.standard_normal((b, n, n)).astype(np.float32)).cuda()
    ga = bed.taylor_backward(r.eigenvectors, r.eigenvalues, gv, None)
    ref = oracle.taylor_backward(r.eigenvectors.cpu().numpy(), r.eigenvalues.cpu().numpy(),
                                 gv.cpu().numpy(), None)
    assert P.grad_err(ga.cpu().numpy(), ref).max() <= P.GRAD_TOL
    inside = oracle.taylor_domain(r.eigenvalues.cpu().numpy())
    assert inside[:4].all() and not inside.all()
    with pytest.raises(bed.NonPositiveSpectrum) as err:
        bed.taylor_backward(r.eigenvectors, r.eigenvalues, gv, None, check=True)
    assert err.value.batch_index == int(np.nonzero(~inside)[0][0])
    # SPD only: no error with check
    bed.taylor_backward(r.eigenvectors[:4].contiguous(), r.eigenvalues[:4].contiguous(), gv[:4].contiguous(),
                        None, check=True)
    # through autograd with check=True
    at = torch.from_numpy(a).cuda().requires_grad_(True)
    lam_t, v_t = bed.eigh(at, bed.SolverConfig(deflation_tol=3e-12), check=True)
    with pytest.raises(bed.NonPositiveSpectrum):
        (v_t * gv).sum().backward()


# ---- the tcgen05 tier (33 <= n <= 64, bed_backward_tc.cuh): ragged n and
# batches, null cotangents, the domain rule and the large-degree limit


@pytest.mark.parametrize("n,b", [(33, 1), (47, 5), (57, 333), (64, 2)])
def test_tensor_core_backward_ragged(bed, n, b):
    rng = np.random.default_rng(n + b)
    q, _ = np.linalg.qr(rng.standard_normal((b, n, n)))
    lam = np.sort(rng.uniform(0.1, 4.0, (b, n)), axis=1)[:, ::-1].copy()
    v = q.astype(np.float32)
    vt, lt = torch.from_numpy(v).cuda(), torch.from_numpy(lam.astype(np.float32)).cuda()
    gv = rng.standard_normal((b, n, n)).astype(np.float32)
    gl = rng.standard_normal((b, n)).astype(np.float32)
    for g_v, g_l in ((gv, gl), (None, gl), (gv, None)):
        ga = bed.taylor_backward(vt, lt, None if g_v is None else torch.from_numpy(g_v).cuda(),
                                 None if g_l is None else torch.from_numpy(g_l).cuda()).cpu().numpy()
        ref = oracle.taylor_backward(v.astype(np.float64), lam.astype(np.float32).astype(np.float64), g_v, g_l)
        assert P.grad_err(ga, ref).max() <= P.GRAD_TOL
        np.testing.assert_array_equal(ga, ga.transpose(0, 2, 1))


def test_tensor_core_backward_domain_and_degree(bed):
    n, b = 40, 24
    rng = np.random.default_rng(3)
    q, _ = np.linalg.qr(rng.standard_normal((b, n, n)))
    lam = np.sort(rng.uniform(-2.0, 3.0, (b, n)), axis=1)[:, ::-1].copy()
    lam[:8] = np.abs(lam[:8]) + 0.5  # SPD rows
    vt = torch.from_numpy(q.astype(np.float32)).cuda()
    lt = torch.from_numpy(lam.astype(np.float32)).cuda()
    gv = torch.from_numpy(rng.standard_normal((b, n, n)).astype(np.float32)).cuda()
    ga = bed.taylor_backward(vt, lt, gv, None).cpu().numpy()
    ref = oracle.taylor_backward(vt.cpu().numpy(), lt.cpu().numpy(), gv.cpu().numpy(), None)
    assert P.grad_err(ga, ref).max() <= P.GRAD_TOL
    inside = oracle.taylor_domain(lt.cpu().numpy())
    with pytest.raises(bed.NonPositiveSpectrum) as err:
        bed.taylor_backward(vt, lt, gv, None, check=True)
    assert err.value.batch_index == int(np.nonzero(~inside)[0][0])
    # large degree on a geometric SPD spectrum (neighbour ratio 0.9: 0.9^300 ~ 2e-14)
    # -> the exact 1/(l_j - l_i)
    lg = np.tile(3.0 * 0.9 ** np.arange(n), (8, 1))
    spd = torch.from_numpy(lg.astype(np.float32)).cuda()
    v8 = vt[:8].contiguous()
    g300 = bed.taylor_backward(v8, spd, gv[:8].contiguous(), None, 300).cpu().numpy()
    l64 = spd.cpu().numpy().astype(np.float64)
    vv = v8.cpu().numpy().astype(np.float64)
    diff = l64[:, None, :] - l64[:, :, None]
    fexact = np.where(np.eye(n, dtype=bool), 0.0, 1.0 / np.where(np.eye(n, dtype=bool), 1.0, diff))
    m = vv.transpose(0, 2, 1) @ gv[:8].cpu().numpy().astype(np.float64)
    gex = vv @ (fexact * m) @ vv.transpose(0, 2, 1)
    gex = (gex + gex.transpose(0, 2, 1)) / 2
    assert P.grad_err(g300, gex).max() <= 1e-3
