"""One C5-sized Taylor backward launch (n = 64, 8192 matrices) for ncu
captures of bed_backward_tc_kernel / bed_backward_kernel (BED_TC=0)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2207_04228_b200 as bed  # noqa: E402

n, b = 64, 8192
V, _ = torch.linalg.qr(torch.randn(b, n, n, device="cuda"))
L = torch.rand(b, n, device="cuda") + 0.5
gv = torch.randn(b, n, n, device="cuda")
gl = torch.randn(b, n, device="cuda")
bed.taylor_backward(V, L, gv, gl)
torch.cuda.synchronize()
