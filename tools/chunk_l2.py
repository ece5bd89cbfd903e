"""Medium-path chunk size vs device time (dev tool, GPU): smaller chunks keep a
chunk's P and rotation records L2-resident between the H, Q and F kernels."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2207_04228_b200 as bed  # noqa: E402
from paper_2207_04228_b200 import _native  # noqa: E402
from paper_2207_04228_b200.datagen import covariance_device, gen_spd_device  # noqa: E402

for n, b in ((16, 65536), (16, 262144), (24, 131072), (32, 65536), (64, 8192)):
    a = covariance_device(b, n, 4 * n, 0) if n == 16 else gen_spd_device(b, n, 0)
    cfg = bed.SolverConfig(deflation_tol=3e-12, max_double_steps=4 * n)
    lam = torch.empty((b, n), device="cuda")
    vec = torch.empty((b, n, n), device="cuda")
    c = _native.make_config(cfg, n)
    for chunk in (b, 32768, 16384, 8192, 4096):
        if chunk > b:
            continue
        wb = _native.workspace_bytes(chunk, n, c)
        ws = torch.empty((wb + 256,), dtype=torch.uint8, device="cuda")
        f = lambda: bed.forward_into(a, cfg, lam, vec, ws=ws)  # noqa: E731
        for _ in range(3):
            f()
        best = 1e9
        for _ in range(3):
            s0, s1 = torch.cuda.Event(True), torch.cuda.Event(True)
            torch.cuda.synchronize()
            s0.record()
            for _ in range(10):
                f()
            s1.record()
            torch.cuda.synchronize()
            best = min(best, s0.elapsed_time(s1) / 10)
        print(f"n={n} b={b} chunk={chunk}: {best:.4f} ms (workspace {wb / 2**20:.0f} MiB)", flush=True)
