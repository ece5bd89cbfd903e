"""Accuracy of the backward's three products on tensor cores (dev tool).

gA = sym(V (F o (V^T gV) + diag gL) V^T) with the products in single-pass
TF32 (torch.backends.cuda.matmul.allow_tf32, i.e. cuBLAS TF32 tensor-core
GEMMs), in 3xTF32 (each operand split into a TF32 head and a TF32 tail,
three products), and in FP32 (the FFMA path), each against float64.  The
gradient gate of the parity tests is 1e-4 relative (Frobenius).  Prints one
line per (n, precision) with the median and max relative error over the batch.
Run on a GPU: python tools/tf32_accuracy.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402  (test infrastructure: the float64 checker)

torch.manual_seed(0)
dev = "cuda"


def tf32(x):
    return (x.view(torch.int32) & ~0x1FFF).view(torch.float32)  # truncate to 10 mantissa bits


def mm(a, b, mode):
    if mode == "fp32":
        torch.backends.cuda.matmul.allow_tf32 = False
        return a @ b
    if mode == "tf32":
        torch.backends.cuda.matmul.allow_tf32 = True
        return a @ b
    torch.backends.cuda.matmul.allow_tf32 = True  # 3xTF32: hi*hi + hi*lo + lo*hi
    ah, bh = tf32(a), tf32(b)
    al, bl = a - ah, b - bh
    return ah @ bh + (ah @ bl + al @ bh)


for n, m in ((16, 64), (32, 128), (64, 256)):
    b = 2048
    x = torch.randn(b, n, m, device=dev, dtype=torch.float64)
    x = x - x.mean(dim=2, keepdim=True)
    a = x @ x.transpose(1, 2) / m + 1e-5 * torch.eye(n, device=dev, dtype=torch.float64)
    lam, v = torch.linalg.eigh(a)
    lam, v = lam.flip(-1), v.flip(-1)
    gv = torch.randn(b, n, n, device=dev, dtype=torch.float64)
    gl = torch.randn(b, n, device=dev, dtype=torch.float64)
    ref = torch.from_numpy(oracle.taylor_backward(v.cpu().numpy(), lam.cpu().numpy(), gv.cpu().numpy(),
                                                  gl.cpu().numpy())).to(dev)
    f = torch.from_numpy(oracle.taylor_k(lam.cpu().numpy())).to(dev).float()
    v32, gv32, gl32 = v.float(), gv.float(), gl.float()
    for mode in ("fp32", "tf32", "3xtf32"):
        mmat = mm(v32.transpose(1, 2), gv32, mode)
        mp = f * mmat + torch.diag_embed(gl32)
        g = mm(mm(v32, mp, mode), v32.transpose(1, 2), mode)
        g = 0.5 * (g + g.transpose(1, 2))
        err = (torch.linalg.matrix_norm(g.double() - ref) / torch.linalg.matrix_norm(ref)).cpu().numpy()
        print(f"n={n:2d} {mode:7s} rel err median {np.median(err):.2e} max {err.max():.2e} "
              f"(gate 1e-4: {'pass' if err.max() <= 1e-4 else 'FAIL'})")
torch.backends.cuda.matmul.allow_tf32 = False
