"""One launch of each main kernel configuration, for ncu captures."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2207_04228_b200 as bed  # noqa: E402
from paper_2207_04228_b200.datagen import covariance_device, gen_spd_device  # noqa: E402

torch.cuda.set_device(0)
cases = [(4, 1 << 22, False), (8, 1 << 20, False), (16, 65536, True), (24, 65536, False), (32, 65536, False),
         (64, 8192, True)]
which = [x for x in sys.argv[1:] if x.isdigit()] or None
power = "pow" in sys.argv
if "scat" in sys.argv:  # covariance producer only
    for n, m, b in ((16, 64, 65536), (64, 256, 8192)):
        x = torch.randn((b, n, m), device="cuda")
        bed.scatter_matrices(x, 1e-5)
    torch.cuda.synchronize()
    print("done")
    sys.exit(0)
if "powf" in sys.argv or "scatpow" in sys.argv:  # the fused power / covariance paths
    for n, b, _ in cases:
        if which and str(n) not in which:
            continue
        if "powf" in sys.argv:
            a = covariance_device(b, n, 4 * n, 0)
            bed.power_of(a, -0.5, check=False)
        else:
            x = torch.randn((b // 4, n, 4 * n), device="cuda")
            bed.scatter_power(x, -0.5, 1e-3, check=False)
            bed.scatter_matrices(x, 1e-3)
    torch.cuda.synchronize()
    print("done")
    sys.exit(0)
for n, b, bwd in cases:
    if which and str(n) not in which:
        continue
    a = covariance_device(b, n, 4 * n, 0) if n == 16 else gen_spd_device(b, n, 0)
    cfg = bed.SolverConfig(deflation_tol=3e-12, max_double_steps=4 * n)
    lam = torch.empty((b, n), device="cuda")
    vec = torch.empty((b, n, n), device="cuda")
    bed.forward_into(a, cfg, lam, vec)
    if power:
        bed.matrix_power(bed.EigenResult(lam, vec, None), -0.5)
    if bwd:
        gv = torch.randn_like(vec)
        gl = torch.randn_like(lam)
        bed.taylor_backward(vec, lam, gv, gl)
    torch.cuda.synchronize()
print("done")
