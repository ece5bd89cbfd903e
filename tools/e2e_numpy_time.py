"""batched_eig(BatchedSymmetric(float64 numpy)) end to end (the reference
user's call, now through bed_forward_host_f64), n = 4 / 16 / 64 (dev tool, GPU)."""
import sys
import time

sys.path.insert(0, ".")
import oracle  # noqa: E402  (test infrastructure: input generator only)
import paper_2207_04228_b200 as bed  # noqa: E402

for n, b in ((4, 1 << 20), (4, 1 << 22), (16, 1 << 16), (64, 4096)):
    a = oracle.gen_spd(b, n, 7)
    cfg = bed.SolverConfig(deflation_tol=3e-12, max_double_steps=4 * n)
    bed.batched_eig(bed.BatchedSymmetric(a), cfg)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        bed.batched_eig(bed.BatchedSymmetric(a), cfg)
        ts.append(time.perf_counter() - t0)
    t = sorted(ts)[1]
    print(f"n={n} b={b}: {t * 1e3:.1f} ms, {b / t / 1e6:.1f} M matrices/s")
