"""Tensor-core backward (bed_backward_tc.cuh) against the float64 oracle and
the FFMA2 kernel: relative gradient error per matrix, then device time at C5
(dev tool, GPU).  BED_TC=0 runs the FFMA2 kernel for comparison."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402  (test infrastructure: the float64 checker)
import paper_2207_04228_b200 as bed  # noqa: E402

torch.manual_seed(0)
for n, b in ((64, 2), (64, 7), (40, 33), (33, 16), (64, 300)):
    x = np.random.default_rng(n + b).standard_normal((b, n, 4 * n))
    a = x @ x.transpose(0, 2, 1) / (4 * n) + 1e-3 * np.eye(n)
    lam64, v64 = np.linalg.eigh(a)
    lam64, v64 = lam64[:, ::-1].copy(), v64[:, :, ::-1].copy()
    gv = np.random.default_rng(1).standard_normal((b, n, n))
    gl = np.random.default_rng(2).standard_normal((b, n))
    V = torch.from_numpy(v64.astype(np.float32)).cuda()
    L = torch.from_numpy(lam64.astype(np.float32)).cuda()
    g = bed.taylor_backward(V, L, torch.from_numpy(gv.astype(np.float32)).cuda(),
                            torch.from_numpy(gl.astype(np.float32)).cuda()).cpu().numpy()
    ref = oracle.taylor_backward(V.cpu().numpy().astype(np.float64), L.cpu().numpy().astype(np.float64), gv, gl)
    err = np.linalg.norm(g - ref, axis=(1, 2)) / np.linalg.norm(ref, axis=(1, 2))
    print(f"n={n} b={b}: rel err max {err.max():.3e} median {np.median(err):.3e}", flush=True)

n, b = 64, 8192
x = torch.randn(b, n, n, device="cuda")
V, _ = torch.linalg.qr(x)
L = torch.rand(b, n, device="cuda") + 0.5
gv = torch.randn(b, n, n, device="cuda")
gl = torch.randn(b, n, device="cuda")
f = lambda: bed.taylor_backward(V, L, gv, gl)  # noqa: E731
for _ in range(3):
    f()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
torch.cuda.synchronize()
s.record()
for _ in range(20):
    f()
e.record()
torch.cuda.synchronize()
print(f"C5 backward n=64 b=8192 ({'tensor cores' if os.environ.get('BED_TC', '1') != '0' else 'FFMA2'}): "
      f"{s.elapsed_time(e) / 20 * 1e3:.1f} us", flush=True)
