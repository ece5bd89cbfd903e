"""Tensor-core spectral power (bed_power_tc.cuh) against the float64 oracle,
then the power kernel's device time at n = 64, 8192 matrices (dev tool, GPU).
BED_TC=0 runs the FFMA2 kernel."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402  (test infrastructure: the float64 checker)
import paper_2207_04228_b200 as bed  # noqa: E402

for n, b, p in ((64, 5, -0.5), (40, 33, 0.5), (33, 16, -1.0), (64, 300, 2.0), (48, 77, 0.3)):
    x = np.random.default_rng(n + b).standard_normal((b, n, 4 * n))
    a = x @ x.transpose(0, 2, 1) / (4 * n) + 1e-2 * np.eye(n)
    lam, v = np.linalg.eigh(a)
    V = torch.from_numpy(v.astype(np.float32)).cuda()
    L = torch.from_numpy(lam.astype(np.float32)).cuda()
    got = bed.matrix_power(bed.EigenResult(L, V, None), p).data.cpu().numpy().astype(np.float64)
    ref, bad = oracle.matrix_power(V.cpu().numpy().astype(np.float64), L.cpu().numpy().astype(np.float64), p)
    err = np.linalg.norm(got - ref, axis=(1, 2)) / np.linalg.norm(ref, axis=(1, 2))
    sym = np.abs(got - got.transpose(0, 2, 1)).max()
    print(f"n={n} b={b} p={p}: rel err max {err.max():.3e}, asym {sym}", flush=True)

n, b = 64, 8192
V, _ = torch.linalg.qr(torch.randn(b, n, n, device="cuda"))
L = torch.rand(b, n, device="cuda") + 0.5
e = bed.EigenResult(L, V, None)
for _ in range(3):
    bed.matrix_power(e, -0.5)
s0, s1 = torch.cuda.Event(True), torch.cuda.Event(True)
torch.cuda.synchronize()
s0.record()
for _ in range(20):
    bed.matrix_power(e, -0.5)
s1.record()
torch.cuda.synchronize()
print(f"matrix_power n=64 b=8192 ({'tensor cores' if os.environ.get('BED_TC', '1') != '0' else 'FFMA2'}): "
      f"{s0.elapsed_time(s1) / 20 * 1e3:.1f} us (incl. the host check)", flush=True)
