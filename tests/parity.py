"""Shared parity metrics for the GPU tests (test infrastructure).

Tolerances (north star, BASELINE.json):
* eigenvalues: |lam - lam_ref| <= 1e-5 * rho, rho = max|lam_ref| (the
  reference's own convention, oracle.py:34, :232)
* reconstruction ||A V - V Lambda||_F / ||A||_F <= 1e-5
* orthogonality ||V^T V - I||_F / n <= 1e-5 (normalised by n as the
  reference's verify does, bench.py:261-268)
* eigenvectors, up to sign, for well separated eigenvalues:
  ||v - s v_ref|| <= 64 eps32 rho / gap  (first-order perturbation bound)
* gradients: ||gA - gA_ref||_F <= 1e-4 ||gA_ref||_F
"""

from __future__ import annotations

import numpy as np

EIG_TOL = 1e-5
RECON_TOL = 1e-5
ORTH_TOL = 1e-5
GRAD_TOL = 1e-4
EPS32 = float(np.finfo(np.float32).eps)


def eig_err(vals, ref_vals):
    vals = np.asarray(vals, np.float64)
    ref = np.asarray(ref_vals, np.float64)
    rho = np.maximum(np.abs(ref).max(axis=1), np.finfo(np.float64).tiny)
    return np.abs(vals - ref).max(axis=1) / rho


def recon_err(a, vals, vecs):
    a = np.asarray(a, np.float64)
    v = np.asarray(vecs, np.float64)
    lam = np.asarray(vals, np.float64)
    res = a @ v - v * lam[:, None, :]
    den = np.maximum(np.linalg.norm(a, axis=(1, 2)), np.finfo(np.float64).tiny)
    return np.linalg.norm(res, axis=(1, 2)) / den


def orth_err(vecs):
    v = np.asarray(vecs, np.float64)
    n = v.shape[1]
    return np.linalg.norm(v.transpose(0, 2, 1) @ v - np.eye(n), axis=(1, 2)) / n


def vector_err(vecs, ref_vecs, ref_vals, gap_floor=1e-3):
    """Max over well-separated columns of ||v - s v_ref|| / (64 eps rho / gap)
    (<= 1 passes).  Columns whose gap to a neighbour is below
    gap_floor * rho are skipped (their subspace is covered by recon/orth)."""
    v = np.asarray(vecs, np.float64)
    vr = np.asarray(ref_vecs, np.float64)
    lam = np.asarray(ref_vals, np.float64)
    b, n = lam.shape
    worst = np.zeros(b)
    for k in range(b):
        rho = max(np.abs(lam[k]).max(), 1e-300)
        for j in range(n):
            others = np.delete(lam[k], j)
            gap = np.abs(others - lam[k, j]).min() if n > 1 else rho
            if gap < gap_floor * rho:
                continue
            s = 1.0 if v[k, :, j] @ vr[k, :, j] >= 0 else -1.0
            err = np.linalg.norm(v[k, :, j] - s * vr[k, :, j])
            worst[k] = max(worst[k], err / (64 * EPS32 * rho / gap))
    return worst


def grad_err(g, g_ref):
    g = np.asarray(g, np.float64)
    g_ref = np.asarray(g_ref, np.float64)
    den = np.maximum(np.linalg.norm(g_ref, axis=(1, 2)), 1e-300)
    return np.linalg.norm(g - g_ref, axis=(1, 2)) / den
