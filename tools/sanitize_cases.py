"""Small ragged-batch solves of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck) runs."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2207_04228_b200 as bed  # noqa: E402

torch.cuda.set_device(0)
for n, b in ((3, 130), (4, 131), (8, 129), (9, 37), (13, 41), (16, 161), (24, 70), (32, 33), (40, 19), (64, 35)):
    a = torch.from_numpy(oracle.gen_spd(b, n, n).astype(np.float32)).cuda().requires_grad_(True)
    lam, v = bed.eigh(a, bed.SolverConfig(deflation_tol=3e-12, max_double_steps=4 * n))
    (v.sum() + lam.sum()).backward()
    bed.batched_eig(a.detach(), bed.SolverConfig(compute_vectors=False, max_double_steps=4 * n))
    bed.matrix_power(bed.EigenResult(lam.detach(), v.detach(), None), -0.5)
    bed.scatter_matrices(torch.randn(7, n, 2 * n + 3, device="cuda"), 1e-3)
    bed.spectral_power(a.detach().clone().requires_grad_(True), -0.5).sum().backward()
# full scatter CTAs, a chunked medium-path workspace, diagnostics outputs
bed.scatter_matrices(torch.randn(200, 4, 9, device="cuda"), 0.0)
a = torch.from_numpy(oracle.gen_spd(300, 20, 2).astype(np.float32)).cuda()
cfg = bed.SolverConfig(deflation_tol=3e-12, max_double_steps=80)
lam = torch.empty((300, 20), device="cuda")
vec = torch.empty((300, 20, 20), device="cuda")
bed.forward_into(a, cfg, lam, vec, ws=bed.workspace(a, cfg, max_bytes=1))
bed.batched_eig(a, cfg)
# chunked host path and a batch above the medium path's sub-warp tails
x = oracle.gen_spd(3000, 4, 1).astype(np.float32)
bed.batched_eig(x, bed.SolverConfig(deflation_tol=3e-12))
# float64 host entry (host-thread validation, one stream per staging slot)
bed.batched_eig(oracle.gen_spd(2100, 6, 3), bed.SolverConfig(deflation_tol=3e-12, max_double_steps=24))
bed.batched_eig(oracle.gen_spd(70, 36, 3), bed.SolverConfig(deflation_tol=3e-12, max_double_steps=144))
# fused power and covariance paths (one kernel for n <= 8), ragged m
for n, m in ((3, 7), (4, 16), (8, 33), (12, 48), (40, 130), (64, 65)):
    xs = torch.randn(67, n, m, device="cuda")
    bed.scatter_power(xs, -0.5, 1e-2, check=False)
    bed.scatter_eig(xs, 1e-2, check=False)
    bed.power_of(bed.scatter_matrices(xs, 1e-2), 0.5, check=False)
torch.cuda.synchronize()
print("sanitize cases done")
