"""Fused covariance -> ED -> power (scatter_power) against the composed
scatter_matrices -> power_of path, and the producer alone (dev tool, GPU)."""
import torch, sys
sys.path.insert(0, ".")
import paper_2207_04228_b200 as bed
for n, b in ((4, 1 << 20), (8, 1 << 18), (16, 1 << 16)):
    m = 4 * n
    x = torch.randn(b, n, m, device="cuda")
    cfg = bed.SolverConfig()
    def fused(): return bed.scatter_power(x, -0.5, 1e-2, cfg, floor=0.0, check=False)
    def comp(): return bed.power_of(bed.scatter_matrices(x, 1e-2), -0.5, cfg, floor=0.0, check=False)
    for name, f in (("fused", fused), ("composed", comp)):
        for _ in range(3): f()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda.synchronize(); s.record()
        for _ in range(10): f()
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 10
        gb = b * 4 * (n * m + n * n + n) / ms / 1e6
        print(f"n={n} b={b} m={m} {name}: {ms:.3f} ms  ({gb:.0f} GB/s of X+out+evals)")
# the producer alone (scatter_matrices / bed_scatter_f32)
for n, b, m in ((4, 1 << 20, 16), (8, 1 << 18, 32), (16, 1 << 16, 64), (32, 1 << 14, 128), (64, 4096, 256)):
    x = torch.randn(b, n, m, device="cuda")
    f = lambda: bed.scatter_matrices(x, 1e-2)
    for _ in range(3): f()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); s.record()
    for _ in range(10): f()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"scatter n={n} b={b} m={m}: {ms:.3f} ms ({b * 4 * (n * m + n * n) / ms / 1e6:.0f} GB/s)")
