"""Generate the golden fixtures in tests/golden/ by running the REFERENCE
package (``/root/reference/pkg/src/batchedeig``) in this container.

The reference is CPU/numba Python and cannot travel to the GPU box, so its
outputs are committed here as small .npz fixtures.  Run from the repo root:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every input is FP32-representable (generated in float64, cast to float32 and
upcast again) so the same values feed the CUDA path (FP32) and the reference
(float64).  Fixtures:

``known_answers.npz``  reference known-answer cases (test_solver.py:29-45,
                       test_qr.py:45-114, test_householder.py:33-69).
``cells.npz``          reference ``batched_eig`` (batch-wide gate) on seeded
                       ``gen_spd`` batches plus edge-case batches, in the
                       default (1e-5, 2n) and verify (3e-12, 4n) profiles,
                       and the same solver applied matrix by matrix (batch of
                       one) for the per-matrix-gate comparison.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from batchedeig import (  # noqa: E402
    BatchedSymmetric,
    SolverConfig,
    batched_eig,
    gen_spd,
    givens_coeffs,
    householder_vector,
    rank2_update,
    wilkinson_shifts,
)

HERE = os.path.dirname(os.path.abspath(__file__))


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)


def covariance(rng, batch, n, m, eps=1e-5):
    x = rng.standard_normal((batch, n, m))
    x = x - x.mean(axis=2, keepdims=True)
    c = x @ x.transpose(0, 2, 1) / m + eps * np.eye(n)
    return (c + c.transpose(0, 2, 1)) / 2.0


def cells():
    rng = np.random.default_rng(20261017)
    out = {}
    # name -> float64 FP32-representable input batch
    batches = {
        "c1_n4_b512": gen_spd(512, 4, 0).data,
        "psd_n4_b64": (lambda r: r @ r.transpose(0, 2, 1))(rng.standard_normal((64, 4, 4))),
        "n1_b4": rng.standard_normal((4, 1, 1)),
        "n2_b16": gen_spd(16, 2, 2).data,
        "n3_b32": gen_spd(32, 3, 3).data,
        "n5_b32": gen_spd(32, 5, 5).data,
        "n7_b32": gen_spd(32, 7, 7).data,
        "n8_b64": gen_spd(64, 8, 8).data,
        "n12_b32": gen_spd(32, 12, 12).data,
        "n16_b64": gen_spd(64, 16, 16).data,
        "cov_n16_b32": covariance(rng, 32, 16, 64),
        "n24_b32": gen_spd(32, 24, 24).data,
        "n32_b32": gen_spd(32, 32, 32).data,
        "n40_b8": gen_spd(8, 40, 40).data,
        "n64_b8": gen_spd(8, 64, 64).data,
        "cov_n64_b4": covariance(rng, 4, 64, 256),
        # edge cases: exact diagonal, repeated eigenvalues, zero, rank one,
        # indefinite, tiny and huge scales, mixed in one batch
        "edge_n4": np.stack([
            np.diag([1.0, 2.0, 3.0, 4.0]),
            np.eye(4),
            np.zeros((4, 4)),
            np.outer([1.0, 2.0, 3.0, 4.0], [1.0, 2.0, 3.0, 4.0]),
            (lambda r: (r + r.T) / 2)(rng.standard_normal((4, 4))),
            1e-20 * gen_spd(1, 4, 11).data[0],
            1e20 * gen_spd(1, 4, 12).data[0],
            np.diag([5.0, 5.0, 1.0, 1.0]),
        ]),
        "edge_n16": np.stack([
            np.eye(16),
            np.diag(np.arange(16.0)),
            (lambda r: (r + r.T) / 2)(rng.standard_normal((16, 16))),
            np.ones((16, 16)),
        ]),
    }
    profiles = {"default": (1e-5, None), "verify": (3e-12, "4n")}
    for name, a in batches.items():
        a = f32(a)
        b, n, _ = a.shape
        out[f"{name}/a"] = a.astype(np.float32)
        for pname, (tol, steps) in profiles.items():
            ms = 4 * n if steps == "4n" else None
            cfg = SolverConfig(deflation_tol=tol, max_double_steps=ms, strict_convergence=False)
            res = batched_eig(BatchedSymmetric(a), cfg)
            out[f"{name}/{pname}/evals"] = res.eigenvalues
            if pname == "verify" or n <= 8:
                out[f"{name}/{pname}/evecs"] = res.eigenvectors
            out[f"{name}/{pname}/double_steps"] = np.int64(res.diagnostics.double_steps)
            out[f"{name}/{pname}/rotations"] = np.int64(res.diagnostics.rotation_count)
            out[f"{name}/{pname}/converged"] = res.diagnostics.converged_steps.astype(np.int64)
            # the same solver run matrix by matrix (per-matrix gate)
            solo_l, solo_v, solo_k = [], [], []
            for k in range(min(b, 8)):
                r1 = batched_eig(BatchedSymmetric(a[k : k + 1]), cfg)
                solo_l.append(r1.eigenvalues[0])
                solo_v.append(r1.eigenvectors[0])
                solo_k.append(r1.diagnostics.double_steps)
            out[f"{name}/{pname}/solo_evals"] = np.array(solo_l)
            if pname == "verify":
                out[f"{name}/{pname}/solo_evecs"] = np.array(solo_v)
            out[f"{name}/{pname}/solo_steps"] = np.array(solo_k, np.int64)
    # values-only and ascending-sort variants on one cell
    a = f32(gen_spd(64, 8, 8).data)
    cfg = SolverConfig(deflation_tol=3e-12, max_double_steps=32, compute_vectors=False)
    out["n8_b64/values_only/evals"] = batched_eig(BatchedSymmetric(a), cfg).eigenvalues
    cfg = SolverConfig(deflation_tol=3e-12, max_double_steps=32, sort="ascending")
    r = batched_eig(BatchedSymmetric(a), cfg)
    out["n8_b64/ascending/evals"] = r.eigenvalues
    out["n8_b64/ascending/evecs"] = r.eigenvectors
    np.savez_compressed(os.path.join(HERE, "cells.npz"), **out)
    return out


def known_answers():
    out = {}
    # test_solver.py:29-34
    r = batched_eig(BatchedSymmetric(np.diag([1.0, 2.0, 3.0])[None]))
    out["diag123/a"] = np.diag([1.0, 2.0, 3.0])[None]
    out["diag123/evals"] = r.eigenvalues
    out["diag123/evecs"] = r.eigenvectors
    # test_solver.py:37-45
    a = np.array([[[2.0, 1.0], [1.0, 2.0]]])
    r = batched_eig(BatchedSymmetric(a))
    out["classic2x2/a"] = a
    out["classic2x2/evals"] = r.eigenvalues
    out["classic2x2/evecs"] = r.eigenvectors
    # test_qr.py:45-50 givens (3, 4)
    g = givens_coeffs([3.0], [4.0])
    out["givens34/cs"] = np.array([g.c[0], g.s[0]])
    # test_qr.py:90-94, :77-87, :109-114 wilkinson pairs
    abd = np.array([[5.0, 2.0, 1.0], [2.0, 1.0, 2.0], [4.0, 0.0, 9.0], [2.0, 1e-300, 1.0]])
    pairs = [wilkinson_shifts([x[0]], [x[1]], [x[2]]) for x in abd]
    out["wilkinson/abd"] = abd
    out["wilkinson/lo_hi"] = np.array([[p.mu_lo[0], p.mu_hi[0]] for p in pairs])
    # test_householder.py:33-69: 3-4-5 tail, sign rule, all-ones 4x4
    for name, tail in (("hh345", [3.0, 4.0]), ("hhm345", [-3.0, 4.0])):
        n = len(tail) + 1
        m = np.zeros((n, n))
        m[0, 0] = 1.0
        m[1:, 0] = tail
        m[0, 1:] = tail
        m[1:, 1:] = np.eye(n - 1) * 2.0
        a = BatchedSymmetric(m[None])
        u, sigma = householder_vector(a, 0)
        out[f"{name}/a"] = m[None]
        out[f"{name}/u"] = u
        out[f"{name}/after"] = rank2_update(a, u, sigma).data
    a = BatchedSymmetric(np.ones((1, 4, 4)))
    u, sigma = householder_vector(a, 0)
    out["ones4/a"] = np.ones((1, 4, 4))
    out["ones4/u"] = u
    out["ones4/after"] = rank2_update(a, u, sigma).data
    np.savez_compressed(os.path.join(HERE, "known_answers.npz"), **out)
    return out


if __name__ == "__main__":
    c = cells()
    k = known_answers()
    print(f"cells: {len(c)} arrays; known answers: {len(k)} arrays")
