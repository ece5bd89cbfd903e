"""GPU parity tests of the forward ED against the reference (golden fixtures)
and the C oracle.  Every solve goes through the C ABI (libbed200.so)."""

import ctypes

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


def _cell_names():
    import os

    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "cells.npz"))
    return sorted({k.split("/")[0] for k in z.files if k.endswith("/a")})


def _solve(bed, a32, **kw):
    cfg = bed.SolverConfig(max_double_steps=4 * a32.shape[1], **kw)
    r = bed.batched_eig(torch.from_numpy(a32).cuda(), cfg)
    v = None if r.eigenvectors is None else r.eigenvectors.cpu().numpy()
    return r.eigenvalues.cpu().numpy(), v, r


@pytest.mark.parametrize("name", _cell_names())
@pytest.mark.parametrize("tol", [3e-12, 1e-5])
def test_golden_cells(bed, cells, name, tol):
    a32 = cells[f"{name}/a"]
    a = a32.astype(np.float64)
    ref_l = cells[f"{name}/verify/evals"]
    ref_v = cells[f"{name}/verify/evecs"]
    lam, vec, _ = _solve(bed, a32, deflation_tol=tol)
    # the reference's fast profile (1e-5) locks couplings up to 1e-5 of the
    # matrix scale, so its residual is bounded by the threshold, not by FP32
    recon_tol = max(P.RECON_TOL, 4 * tol)
    assert np.all(P.eig_err(lam, ref_l) <= P.EIG_TOL), P.eig_err(lam, ref_l).max()
    assert np.all(P.recon_err(a, lam, vec) <= recon_tol), P.recon_err(a, lam, vec).max()
    assert np.all(P.orth_err(vec) <= P.ORTH_TOL), P.orth_err(vec).max()
    if not name.startswith("edge") and tol < 1e-6:
        assert np.all(P.vector_err(vec, ref_v, ref_l) <= 1.0), P.vector_err(vec, ref_v, ref_l).max()
    # descending order, sign convention
    assert np.all(np.diff(lam, axis=1) <= 0)
    lead = np.take_along_axis(vec, np.argmax(np.abs(vec), axis=1)[:, None, :], axis=1)
    assert lead.min() >= 0.0


def test_known_answers(bed, known):
    lam, vec, _ = _solve(bed, known["diag123/a"].astype(np.float32))
    np.testing.assert_array_equal(lam, known["diag123/evals"])
    np.testing.assert_array_equal(vec, known["diag123/evecs"])
    lam, vec, _ = _solve(bed, known["classic2x2/a"].astype(np.float32))
    np.testing.assert_allclose(lam, known["classic2x2/evals"], rtol=2e-7)
    np.testing.assert_allclose(vec, known["classic2x2/evecs"], rtol=2e-7)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 7, 8, 9, 12, 13, 16, 17, 20, 23, 24, 25, 31, 32, 33, 40, 48, 57, 64])
def test_every_size_against_oracle(bed, n):
    b = 37 if n > 8 else 301  # ragged: not a multiple of any CTA tile
    a = oracle.gen_spd(b, n, 1000 + n).astype(np.float32)
    lam, vec, r = _solve(bed, a, **VERIFY)
    o = oracle.forward(a.astype(np.float64))
    assert np.all(P.eig_err(lam, o.eigenvalues) <= P.EIG_TOL)
    assert np.all(P.recon_err(a.astype(np.float64), lam, vec) <= P.RECON_TOL)
    assert np.all(P.orth_err(vec) <= P.ORTH_TOL)
    assert np.all(P.vector_err(vec, o.eigenvectors, o.eigenvalues) <= 1.0)
    steps = r.diagnostics.converged_steps.cpu().numpy()
    assert steps.max() <= 4 * n


@pytest.mark.parametrize("n", [4, 16, 32, 64])
def test_values_only_matches_full(bed, n):
    a = oracle.gen_spd(64, n, 7).astype(np.float32)
    full, _, _ = _solve(bed, a, **VERIFY)
    vals, vec, _ = _solve(bed, a, compute_vectors=False, **VERIFY)
    assert vec is None
    # same band arithmetic; only FMA contraction may differ between the two
    # compiled variants (solver.py:79-85 reference test uses atol 1e-12 in f64)
    assert np.all(P.eig_err(vals, full) <= 1e-6)


@pytest.mark.parametrize("n", [4, 16, 48])
def test_sort_orders(bed, n):
    a = oracle.gen_spd(40, n, 3).astype(np.float32)
    desc, vd, _ = _solve(bed, a, **VERIFY)
    asc, va, _ = _solve(bed, a, sort="ascending", **VERIFY)
    none, vn, _ = _solve(bed, a, sort="none", **VERIFY)
    np.testing.assert_array_equal(asc, desc[:, ::-1])
    np.testing.assert_array_equal(va, vd[:, :, ::-1])
    np.testing.assert_array_equal(np.sort(none, axis=1), np.sort(desc, axis=1))


@pytest.mark.parametrize("n", [4, 16, 64])
def test_partition_independence_bitwise(bed, n):
    """Per-matrix deflation: a matrix's result does not depend on its batch."""
    a = oracle.gen_spd(96, n, 11).astype(np.float32)
    full, vf, _ = _solve(bed, a, **VERIFY)
    for lo, hi in ((0, 1), (5, 40), (40, 96)):
        part, vp, _ = _solve(bed, np.ascontiguousarray(a[lo:hi]), **VERIFY)
        np.testing.assert_array_equal(part, full[lo:hi])
        np.testing.assert_array_equal(vp, vf[lo:hi])


def test_scale_equivariance(bed):
    a = oracle.gen_spd(16, 8, 4).astype(np.float32)
    base, vb, _ = _solve(bed, a, **VERIFY)
    # even powers of two: every scaled quantity, including the square roots in
    # the reflector norms, scales exactly, so the FP32 problems are identical
    for c in (2.0 ** -10, 4.0, 2.0 ** 10):
        s, vs, _ = _solve(bed, (a * np.float32(c)).astype(np.float32), **VERIFY)
        np.testing.assert_array_equal(s, base * np.float32(c))
        np.testing.assert_array_equal(vs, vb)


def test_errors(bed):
    a = np.stack([np.eye(4, dtype=np.float32)] * 3)
    bad = a.copy()
    bad[1, 2, 3] = np.nan
    with pytest.raises(bed.NonFinite) as e:
        bed.batched_eig(torch.from_numpy(bad).cuda())
    assert e.value.batch_index == 1 and e.value.position == (2, 3)
    asym = a.copy()
    asym[2, 0, 1] = 1.0
    with pytest.raises(bed.NonSymmetric) as e:
        bed.batched_eig(torch.from_numpy(asym).cuda())
    assert e.value.batch_index == 2
    hard = oracle.gen_spd(64, 16, 5).astype(np.float32)
    with pytest.raises(bed.NoConvergence):
        bed.batched_eig(torch.from_numpy(hard).cuda(),
                        bed.SolverConfig(deflation_tol=3e-12, max_double_steps=1))
    # fixed schedule: no error, diagonal locked
    r = bed.batched_eig(torch.from_numpy(hard).cuda(),
                        bed.SolverConfig(deflation_tol=3e-12, max_double_steps=1,
                                         strict_convergence=False))
    assert r.eigenvalues.shape == (64, 16)


def test_numpy_host_path_and_batched_symmetric(bed, cells):
    a32 = cells["c1_n4_b512/a"]
    r = bed.batched_eig(bed.BatchedSymmetric(a32.astype(np.float64)),
                        bed.SolverConfig(**VERIFY, max_double_steps=16))
    assert isinstance(r.eigenvalues, np.ndarray) and r.eigenvalues.dtype == np.float64
    assert np.all(P.eig_err(r.eigenvalues, cells["c1_n4_b512/verify/evals"]) <= P.EIG_TOL)


def test_c_abi_host_entry(bed):
    """bed_forward_host_f32 on plain numpy buffers -- the call a non-torch FFI makes."""
    from paper_2207_04228_b200 import _native

    for n, b in ((4, 5000), (24, 300)):
        a = oracle.gen_spd(b, n, 21).astype(np.float32)
        lam = np.zeros((b, n), np.float32)
        vec = np.zeros((b, n, n), np.float32)
        st = np.zeros(b, np.int32)
        k = np.zeros(b, np.int32)
        cfg = _native.make_config(bed.SolverConfig(max_double_steps=4 * n, **VERIFY), n)
        _native.forward_host_f32(a.ctypes.data, b, n, lam.ctypes.data, vec.ctypes.data,
                                 st.ctypes.data, k.ctypes.data, cfg, 0)
        dev, vdev, _ = _solve(bed, a, **VERIFY)
        np.testing.assert_array_equal(lam, dev)
        np.testing.assert_array_equal(vec, vdev)
        assert st.max() == 0 and k.min() >= 1


def test_c_abi_rejects_bad_arguments(bed):
    from paper_2207_04228_b200 import _native

    L = _native.lib()
    cfg = _native.make_config(bed.SolverConfig(), 4)
    x = torch.zeros((2, 4, 4), device="cuda")
    y = torch.zeros((2, 4), device="cuda")
    assert L.bed_forward_f32(x.data_ptr(), 2, 65, y.data_ptr(), x.data_ptr(), None, None, None,
                             ctypes.byref(cfg), None) == 1
    assert L.bed_forward_f32(x.data_ptr(), 2, 4, None, x.data_ptr(), None, None, None,
                             ctypes.byref(cfg), None) == 1
    assert L.bed_forward_f32(x.data_ptr() + 2, 2, 4, y.data_ptr(), x.data_ptr(), None, None, None,
                             ctypes.byref(cfg), None) == 2
    assert L.bed_forward_f32(x.data_ptr(), 0, 4, y.data_ptr(), x.data_ptr(), None, None, None,
                             ctypes.byref(cfg), None) == 0


@pytest.mark.parametrize("n,b", [(4, 1 << 20), (16, 65536), (64, 2048)])
def test_large_batch_properties(bed, n, b):
    """Full-size batches: invariants on every matrix, oracle on a sample."""
    g = torch.Generator(device="cuda").manual_seed(n)
    x = torch.randn((b, n, n), device="cuda", generator=g)
    a = x @ x.transpose(1, 2) / n + 1e-3 * torch.eye(n, device="cuda")
    a = 0.5 * (a + a.transpose(1, 2))
    r = bed.batched_eig(a, bed.SolverConfig(**VERIFY, max_double_steps=4 * n))
    lam, v = r.eigenvalues, r.eigenvectors
    ad = a.double()
    rec = torch.linalg.matrix_norm(ad @ v.double() - v.double() * lam.double()[:, None, :])
    rec = rec / torch.linalg.matrix_norm(ad)
    orth = torch.linalg.matrix_norm(v.double().transpose(1, 2) @ v.double() - torch.eye(n, device="cuda", dtype=torch.float64)) / n
    assert float(rec.max()) <= P.RECON_TOL
    assert float(orth.max()) <= P.ORTH_TOL
    assert bool((lam[:, 1:] <= lam[:, :-1]).all())
    idx = torch.randperm(b, generator=torch.Generator().manual_seed(0))[:64]
    o = oracle.forward(a[idx.cuda()].double().cpu().numpy())
    assert np.all(P.eig_err(lam[idx.cuda()].cpu().numpy(), o.eigenvalues) <= P.EIG_TOL)


def test_values_only_matches_reference_fixture(bed, cells):
    """The reference's own values-only output (solver.py:94-109, written by
    tests/golden/make_golden.py with tol 3e-12, budget 32)."""
    vals, vec, _ = _solve(bed, cells["n8_b64/a"], compute_vectors=False, **VERIFY)
    assert vec is None
    assert np.all(P.eig_err(vals, cells["n8_b64/values_only/evals"]) <= P.EIG_TOL)
    full, _, _ = _solve(bed, cells["n8_b64/a"], **VERIFY)
    assert np.all(P.eig_err(full, cells["n8_b64/values_only/evals"]) <= P.EIG_TOL)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7, 8, 9, 12, 16, 17, 20, 24, 25, 31, 32, 33, 48, 64])
@pytest.mark.parametrize("sort", ["descending", "ascending", "none"])
def test_values_only_against_oracle(bed, n, sort):
    b = 37 if n > 8 else 301
    a = oracle.gen_spd(b, n, 2000 + n).astype(np.float32)
    vals, vec, _ = _solve(bed, a, compute_vectors=False, sort=sort, **VERIFY)
    o = oracle.forward(a.astype(np.float64), compute_vectors=False, sort=sort)
    if sort == "none":  # unsorted order is the band order of each implementation
        vals, ref = np.sort(vals, axis=1), np.sort(o.eigenvalues, axis=1)
    else:
        ref = o.eigenvalues
    assert np.all(P.eig_err(vals, ref) <= P.EIG_TOL)


@pytest.mark.parametrize("n,b", [(12, 3001), (16, 5000), (24, 3000), (32, 2000), (40, 700), (64, 300)])
@pytest.mark.parametrize("vectors", [True, False])
def test_chunked_workspace_is_bitwise_identical(bed, n, b, vectors):
    """A workspace smaller than the batch needs (bed_forward_workspace_bytes)
    solves it in chunks; results must not depend on the chunking."""
    from paper_2207_04228_b200 import _native

    a = torch.from_numpy(oracle.gen_spd(b, n, 31).astype(np.float32)).cuda()
    cfg = bed.SolverConfig(max_double_steps=4 * n, compute_vectors=vectors, **VERIFY)
    c = _native.make_config(cfg, n)
    full = _native.workspace_bytes(b, n, c)
    smallest = _native.workspace_bytes(32, n, c)
    assert 0 < smallest < full

    def run(ws):
        lam = torch.empty((b, n), device="cuda")
        vec = torch.empty((b, n, n), device="cuda") if vectors else None
        st = torch.empty((b,), device="cuda", dtype=torch.int32)
        k = torch.empty((b,), device="cuda", dtype=torch.int32)
        bed.forward_into(a, cfg, lam, vec, st, k, ws=ws)
        return [t.cpu() for t in (lam, vec, st, k) if t is not None]

    ref = run(bed.workspace(a, cfg))
    for cap in (full // 3, smallest, smallest + 1000):
        got = run(bed.workspace(a, cfg, max_bytes=cap))
        for x, y in zip(got, ref):
            assert torch.equal(x, y)
    # below the 32-matrix minimum the call is rejected, nothing launched
    with pytest.raises(_native.NativeError):
        tiny = torch.empty((smallest // 2,), dtype=torch.uint8, device="cuda")
        lam = torch.empty((b, n), device="cuda")
        vec = torch.empty((b, n, n), device="cuda")
        bed.forward_into(a, cfg, lam, vec, ws=tiny)


def test_workspace_sizes(bed):
    """Values-only: the band and status, 4 (2n + 1) bytes per matrix.  With
    vectors: plus P (4 n^2) and the rotation record of every sweep the budget
    allows (2 * budget + 1 sweeps of the tier's NMAX - 1 positions, 8 bytes
    each, plus a 4-byte extent per warp-sweep and a 1-byte size per lane)."""
    from paper_2207_04228_b200 import _native

    b = 65536
    for n, nmax in ((9, 16), (16, 16), (20, 24), (24, 24), (32, 32), (40, 64), (64, 64)):
        cv = _native.make_config(bed.SolverConfig(max_double_steps=4 * n, compute_vectors=False), n)
        assert b * 4 * (2 * n + 1) <= _native.workspace_bytes(b, n, cv) <= b * 4 * (2 * n + 1) + 4 * 256
        c = _native.make_config(bed.SolverConfig(max_double_steps=4 * n), n)
        smax = 8 * n + 1
        want = b * (4 * (n * n + 3 * n + 1) + smax * (nmax - 1) * 8 + smax) + (b // 32) * (4 * smax + 4)
        assert want <= _native.workspace_bytes(b, n, c) <= want + 9 * 256
    assert _native.workspace_bytes(1000, 8, _native.make_config(bed.SolverConfig(), 8)) == 0


def test_headline_inputs_c2(bed):
    """The bench's headline workload exactly: 4,194,304 gen_spd_device 4x4
    matrices, verify profile.  Invariants on every matrix, the oracle on a
    sample (the same call bench.py times)."""
    from paper_2207_04228_b200.datagen import gen_spd_device

    b, n = 1 << 22, 4
    a = gen_spd_device(b, n, 0)
    r = bed.batched_eig(a, bed.SolverConfig(deflation_tol=3e-12, max_double_steps=16))
    lam, v = r.eigenvalues, r.eigenvectors
    eye = torch.eye(n, device="cuda", dtype=torch.float64)
    for lo in range(0, b, 1 << 20):
        ad, vd, ld = a[lo:lo + (1 << 20)].double(), v[lo:lo + (1 << 20)].double(), lam[lo:lo + (1 << 20)].double()
        rec = torch.linalg.matrix_norm(ad @ vd - vd * ld[:, None, :]) / torch.linalg.matrix_norm(ad)
        orth = torch.linalg.matrix_norm(vd.transpose(1, 2) @ vd - eye) / n
        assert float(rec.max()) <= P.RECON_TOL
        assert float(orth.max()) <= P.ORTH_TOL
    assert bool((lam[:, 1:] <= lam[:, :-1]).all())
    lead = torch.gather(v, 1, v.abs().argmax(dim=1, keepdim=True))
    assert float(lead.min()) >= 0.0
    assert int(r.diagnostics.converged_steps.max()) <= 16
    idx = torch.randperm(b, generator=torch.Generator().manual_seed(1))[:256].cuda()
    o = oracle.forward(a[idx].double().cpu().numpy())
    assert np.all(P.eig_err(lam[idx].cpu().numpy(), o.eigenvalues) <= P.EIG_TOL)
    assert np.all(P.vector_err(v[idx].cpu().numpy(), o.eigenvectors, o.eigenvalues) <= 1.0)


def test_float64_host_input_validated_before_the_fp32_cast(bed):
    """A float64 batch symmetric to ~1e-16 (accepted by the reference) can
    round a_ij and a_ji to adjacent FP32 values: it is symmetrised in float64
    first, so it solves; a real asymmetry is still rejected with the
    reference's fields (core.py:286-309)."""
    a = oracle.gen_spd(64, 6, 6)
    # put a_01 / a_10 on either side of an FP32 rounding midpoint: a float64
    # asymmetry of ~1e-16 relative that rounds to two adjacent FP32 values
    x = a[:, 0, 1].astype(np.float32)
    mid = (x.astype(np.float64) + np.nextafter(x, np.float32(np.inf)).astype(np.float64)) / 2
    a[:, 0, 1] = mid * (1 - 1e-15)
    a[:, 1, 0] = mid * (1 + 1e-15)
    assert np.abs(a - a.transpose(0, 2, 1)).max() < 1e-12
    assert np.abs(a.astype(np.float32) - a.astype(np.float32).transpose(0, 2, 1)).max() > 0
    r = bed.batched_eig(bed.BatchedSymmetric(a), bed.SolverConfig(**VERIFY, max_double_steps=24))
    o = oracle.forward((a + a.transpose(0, 2, 1)) / 2)
    assert np.all(P.eig_err(r.eigenvalues, o.eigenvalues) <= P.EIG_TOL)
    bad = a.copy()
    bad[5, 0, 3] += 1e-3
    with pytest.raises(bed.NonSymmetric) as err:
        bed.batched_eig(bed.BatchedSymmetric(bad))
    assert err.value.batch_index == 5
    bad = a.copy()
    bad[9, 2, 1] = np.inf
    with pytest.raises(bed.NonFinite) as err:
        bed.batched_eig(bed.BatchedSymmetric(bad))
    assert err.value.batch_index == 9 and err.value.position == (2, 1)


@pytest.mark.parametrize("n", [4, 6, 12, 16, 24, 40])
def test_diagnostics_match_the_per_matrix_reference_loop(bed, n):
    """Per-matrix SolveDiagnostics counters (qr.py:101-118) against the
    oracle's restatement of the reference loop gated per matrix, at the
    reference's default tolerance (1e-5, above the FP32 floor)."""
    b = 96
    a = oracle.gen_spd(b, n, 500 + n).astype(np.float32)
    cfg = bed.SolverConfig(deflation_tol=1e-5, max_double_steps=4 * n)
    r = bed.batched_eig(torch.from_numpy(a).cuda(), cfg)
    d = r.diagnostics
    o = oracle.forward(a.astype(np.float64), deflation_tol=1e-5, max_double_steps=4 * n)
    steps = d.converged_steps.cpu().numpy()
    rots = d.rotations.cpu().numpy()
    reds = d.reduction_counts.cpu().numpy()
    # FP32 vs float64 can move a deflation by one sweep on a few matrices
    assert np.mean(steps == o.double_steps) >= 0.9
    assert np.mean(rots == o.rotations) >= 0.9
    assert np.all(reds == n - 2)  # every matrix converged down to its closing 2x2
    assert d.rotation_count == int(rots.sum()) and d.reduction_events == int(reds.sum())
    assert d.double_steps == int(steps.max())
    assert 0.0 < d.reductions < n - 2


def test_no_convergence_reports_the_residual(bed):
    hard = oracle.gen_spd(64, 16, 5).astype(np.float32)
    with pytest.raises(bed.NoConvergence) as err:
        bed.batched_eig(torch.from_numpy(hard).cuda(),
                        bed.SolverConfig(deflation_tol=3e-12, max_double_steps=1))
    res = err.value.residual_offdiag_max
    assert np.isfinite(res) and res >= 2.0 ** -22
    assert len(err.value.batch_indices) > 0
