"""Replays bench.py's other_configs sequence case by case (dev tool):
per-case event time, plus a second pass of the same case, to expose
state-dependent slowdowns (allocator / pool effects)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2207_04228_b200 as bed  # noqa: E402

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
cases = [(4, 512, "fwd"), (8, 512, "fwd"), (16, 512, "fwd"), (24, 512, "fwd"), (32, 512, "fwd"),
         (8, 1 << 20, "fwd"), (16, 1 << 18, "fwd"), (24, 1 << 17, "fwd"), (32, 1 << 16, "fwd"),
         (64, 8192, "fwd"), (16, 65536, "fwdbwd"), (64, 8192, "fwdbwd")]
only = [int(x) for x in sys.argv[1:]]
for i, (n, b, mode) in enumerate(cases):
    if only and i not in only:
        continue
    st = bench.Step(torch, bed, n, b, mode, dev, seed=n)
    for rep in range(2):
        reps = 10
        t0 = time.perf_counter()
        sec = bench.time_steps(torch, st, reps, 3) / reps
        wall = (time.perf_counter() - t0) / (reps + 3)
        print(f"case {i} n={n} b={b} {mode} pass {rep}: {sec*1e3:.3f} ms event, {wall*1e3:.3f} ms wall/call",
              flush=True)
