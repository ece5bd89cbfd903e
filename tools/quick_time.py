"""Quick device timing of the forward/backward kernels (dev tool, not the bench)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2207_04228_b200 as bed  # noqa: E402

torch.cuda.set_device(0)
PEAK_HBM = 6538.6e9
PEAK_F32 = 74.4e12


def spd(b, n, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn((b, n, n), device="cuda", generator=g)
    a = x @ x.transpose(1, 2) / n + 1e-3 * torch.eye(n, device="cuda")
    return 0.5 * (a + a.transpose(1, 2))


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


CASES = [(4, 1 << 22, 1e-5), (4, 1 << 22, 3e-12), (8, 1 << 20, 3e-12), (16, 65536, 3e-12),
         (24, 65536, 3e-12), (32, 65536, 3e-12), (64, 8192, 3e-12)]
ONLY = [int(x) for x in sys.argv[1:] if x.isdigit()]
EIGH = "--eigh" in sys.argv
for n, b, tol in CASES:
    if ONLY and n not in ONLY:
        continue
    a = spd(b, n)
    cfg = bed.SolverConfig(deflation_tol=tol, max_double_steps=4 * n)
    L = torch.empty((b, n), device="cuda")
    V = torch.empty((b, n, n), device="cuda")
    st = torch.empty((b,), device="cuda", dtype=torch.int32)
    k = torch.empty((b,), device="cuda", dtype=torch.int32)
    t = timeit(lambda: bed.forward_into(a, cfg, L, V, st, k))
    F = (8 / 3) * n ** 3 + (6 * n + 24) * n * (n - 1)
    B = 4 * (2 * n * n + n)
    roof = max(B / PEAK_HBM, F / PEAK_F32)
    steps = k.float().mean().item()
    print(f"fwd n={n:2d} b={b:8d} tol={tol:.0e}: {t*1e3:8.3f} ms  {b/t/1e6:9.2f} M mat/s  "
          f"roof frac {roof*b/t:.3f}  mean steps {steps:.2f} max {int(k.max())} status {int(st.max())}")
    cfgv = bed.SolverConfig(deflation_tol=tol, max_double_steps=4 * n, compute_vectors=False)
    t = timeit(lambda: bed.forward_into(a, cfgv, L, None, st, k))
    print(f"   values-only: {t*1e3:8.3f} ms  {b/t/1e6:9.2f} M mat/s")
    if n in (16, 64, 32):
        gv = torch.randn_like(V)
        gl = torch.randn_like(L)
        t = timeit(lambda: bed.taylor_backward(V, L, gv, gl))
        Fb = 6 * n ** 3 + 22 * n * n
        Bb = 4 * (3 * n * n + 2 * n)
        roof = max(Bb / PEAK_HBM, Fb / PEAK_F32)
        print(f"   bwd: {t*1e3:8.3f} ms  {b/t/1e6:9.2f} M mat/s  roof frac {roof*b/t:.3f}")
    if not EIGH:
        continue
    try:
        sub = a[: min(b, 16384)].contiguous()
        te = timeit(lambda: torch.linalg.eigh(sub), reps=3, warm=1)
        print(f"   torch.linalg.eigh on {sub.shape[0]}: {te*1e3:.2f} ms -> {sub.shape[0]/te/1e6:.3f} M mat/s")
    except Exception as exc:  # noqa: BLE001
        print("   torch.linalg.eigh failed:", str(exc)[:80])
