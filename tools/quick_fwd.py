"""Device time of forward_into at a few (n, batch) points (dev tool, GPU):
python tools/quick_fwd.py n:batch [n:batch ...]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2207_04228_b200 as bed  # noqa: E402
from paper_2207_04228_b200.datagen import gen_spd_device  # noqa: E402

for arg in sys.argv[1:] or ["8:1048576", "7:1048576", "4:4194304"]:
    n, b = (int(x) for x in arg.split(":"))
    a = gen_spd_device(b, n, 0)
    cfg = bed.SolverConfig(deflation_tol=3e-12, max_double_steps=4 * n)
    lam = torch.empty((b, n), device="cuda")
    vec = torch.empty((b, n, n), device="cuda")
    ws = bed.workspace(a, cfg)
    f = lambda: bed.forward_into(a, cfg, lam, vec, ws=ws)  # noqa: E731
    for _ in range(5):
        f()
    best = 1e9
    for _ in range(3):
        s0, s1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda.synchronize()
        s0.record()
        for _ in range(20):
            f()
        s1.record()
        torch.cuda.synchronize()
        best = min(best, s0.elapsed_time(s1) / 20)
    print(f"n={n} b={b}: {best:.4f} ms", flush=True)
