"""Synthetic input batches generated on the device (benchmark harness).

``gen_spd_device`` draws from the same distribution as the reference
generator ``gen_spd`` (/root/reference/pkg/src/batchedeig/bench.py:112-134):
A = Q diag(lam) Q^T with Q a product of n random Householder reflectors and
lam log-uniform over ``condition_decades`` decades below a per-matrix scale
10^U(-0.5, 0.5).  It uses torch's CUDA generator, so the values differ from
the numpy stream; ``oracle.gen_spd`` is the bit-exact restatement used by
the parity tests.  ``covariance_device`` is the decorrelated-BN / GCP shape
(X - mu)(X - mu)^T / m + eps I.
"""

from __future__ import annotations

import torch


def gen_spd_device(batch: int, n: int, seed: int, condition_decades: float = 3.0,
                   device: str | torch.device = "cuda", chunk: int = 1 << 20) -> torch.Tensor:
    g = torch.Generator(device=device).manual_seed(seed)
    out = torch.empty((batch, n, n), device=device, dtype=torch.float32)
    eye = torch.eye(n, device=device, dtype=torch.float32)
    for lo in range(0, batch, chunk):
        b = min(chunk, batch - lo)
        exps = torch.rand((b, n), device=device, generator=g) * condition_decades
        scale = 10.0 ** (torch.rand((b,), device=device, generator=g) - 0.5)
        lam = scale[:, None] * 10.0 ** (-exps)
        q = eye.expand(b, n, n).clone()
        for _ in range(n):
            v = torch.randn((b, n), device=device, generator=g)
            v = v / v.norm(dim=1, keepdim=True)
            q -= 2.0 * (q @ v[:, :, None]) * v[:, None, :]
        a = (q * lam[:, None, :]) @ q.transpose(1, 2)
        out[lo : lo + b] = 0.5 * (a + a.transpose(1, 2))
    return out


def covariance_device(batch: int, n: int, m: int, seed: int, eps: float = 1e-5,
                      device: str | torch.device = "cuda", chunk: int = 1 << 16) -> torch.Tensor:
    g = torch.Generator(device=device).manual_seed(seed)
    out = torch.empty((batch, n, n), device=device, dtype=torch.float32)
    eye = torch.eye(n, device=device, dtype=torch.float32)
    for lo in range(0, batch, chunk):
        b = min(chunk, batch - lo)
        x = torch.randn((b, n, m), device=device, generator=g)
        x = x - x.mean(dim=2, keepdim=True)
        c = x @ x.transpose(1, 2) / m + eps * eye
        out[lo : lo + b] = 0.5 * (c + c.transpose(1, 2))
    return out
