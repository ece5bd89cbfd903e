#!/usr/bin/env python
"""Benchmark: batched symmetric ED (arXiv 2207.04228) on B200.

Headline (BASELINE.json configs[1]): 4x4 ED forward, 4,194,304 matrices per
GPU (weak scaling across ranks), matrices/second over the whole job.  A step
is one forward pass over the resident batch (one kernel launch); inputs are
generated on the device before timing and the 576 MB working set exceeds the
126 MB L2, so no flush is needed between steps.

Run:  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
Multi-GPU: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
Prints ONE JSON line (rank 0).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "batched ED matrices/sec (fwd, fwd+bwd) vs n, batch; frac of HBM/FP32 roofline"
UNIT = "matrices/s"
HEADLINE = dict(name="c2_fwd_n4", n=4, batch=4194304, mode="fwd")
# accuracy profile of every timed run: the reference verify profile
# (bench.py:40, bench.py:227-228): tol 3e-12 (the kernels floor it at the FP32
# limit 2^-22) and a 4n double-step budget -- the profile whose results pass
# the parity gates (tests/parity.py).
TOL = 3e-12
# FP32 FMA-pipe peak measured on B200 with tools/ubench/ffma_peak.cu (FFMA2,
# profiles/r01_fp32_peak.md); nominal 148 SM x 128 x 2 x 1.965 GHz = 74.4 TFLOP/s
FP32_PEAK = 73.7e12


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]) * 1e9, "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return 6.65e12, "fallback (B200_PROFILING.md)"


def work_per_matrix(n: int, mode: str):
    """algorithmic flops and bytes per matrix."""
    f_fwd = (8.0 / 3.0) * n ** 3 + (6 * n + 24) * n * (n - 1)
    b_fwd = 4 * (2 * n * n + n)
    if mode == "fwd":
        return f_fwd, b_fwd
    if mode == "val":  # eigenvalues only (solver.py:94-109): no P, no fold
        return (4.0 / 3.0) * n ** 3 + 24 * n * (n - 1), 4 * (n * n + n)
    if mode == "fwdpow":  # + spectral power V diag(f) V^T: one n^3 product
        return f_fwd + 2 * n ** 3, b_fwd + 4 * (2 * n * n + n)
    if mode == "powf":  # eigenvalues + A^p in one call: V never returned (bed_forward_power_f32)
        return f_fwd + 2 * n ** 3, b_fwd
    if mode == "scatpow":  # X (n x 4n samples) -> S^p and eigenvalues (bed_scatter_forward_f32)
        m = 4 * n
        return n * (n + 1) * m + f_fwd + 2 * n ** 3, 4 * (n * m + n * n + n)
    f_bwd = 6 * n ** 3 + 22 * n * n
    b_bwd = 4 * (3 * n * n + 2 * n)
    return f_fwd + f_bwd, b_fwd + b_bwd


def roofline(n, mode, batch, seconds, hbm_peak):
    flops, nbytes = work_per_matrix(n, mode)
    t_hbm = batch * nbytes / hbm_peak
    t_f32 = batch * flops / FP32_PEAK
    bound = "hbm" if t_hbm >= t_f32 else "fp32"
    return bound, max(t_hbm, t_f32) / seconds, flops * batch, nbytes * batch


class ClockSampler:
    """NVML poller (5 ms) of SM clock and throttle reasons during a region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001
            pass
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def make_inputs(torch, n, batch, mode, seed, dev):
    from paper_2207_04228_b200.datagen import covariance_device, gen_spd_device

    if mode in ("fwdbwd", "fwdpow") and n <= 16:
        a = covariance_device(batch, n, 4 * n, seed, device=dev)
    else:
        a = gen_spd_device(batch, n, seed, device=dev)
    return a


class Step:
    """One step of a workload on preallocated device buffers."""

    def __init__(self, torch, bed, n, batch, mode, dev, seed):
        self.torch, self.bed, self.n, self.batch, self.mode = torch, bed, n, batch, mode
        if mode == "scatpow":  # samples, not matrices: the covariance is formed inside
            g = torch.Generator(device=dev).manual_seed(seed)
            self.a = torch.randn((batch, n, 4 * n), device=dev, generator=g)
        else:
            self.a = make_inputs(torch, n, batch, mode, seed, dev)
        self.cfg = bed.SolverConfig(deflation_tol=TOL, max_double_steps=4 * n,
                                    compute_vectors=mode != "val")
        self.lam = torch.empty((batch, n), device=dev)
        self.vec = torch.empty((batch, n, n), device=dev)
        self.status = torch.empty((batch,), device=dev, dtype=torch.int32)
        self.steps = torch.empty((batch,), device=dev, dtype=torch.int32)
        if mode == "fwdpow":
            self.pw = torch.empty_like(self.vec)
            self.pst = torch.empty((batch,), device=dev, dtype=torch.int32)
        if mode == "fwdbwd":
            g = torch.Generator(device=dev).manual_seed(seed + 1)
            self.gv = torch.randn((batch, n, n), device=dev, generator=g)
            self.gl = torch.randn((batch, n), device=dev, generator=g)
        # n >= 9: allocated once, outside the timed steps
        self.ws = bed.workspace(self.a, self.cfg) if mode != "scatpow" else None
        if mode == "scatpow":
            from paper_2207_04228_b200 import _native

            self.pws_bytes = _native.scatter_forward_workspace_bytes(batch, n, 4 * n,
                                                                     _native.make_config(self.cfg, n), 1)
            self.pws = torch.empty((self.pws_bytes + 256,), dtype=torch.uint8, device=dev)
            self.pws_ptr = (self.pws.data_ptr() + 255) & ~255 if self.pws_bytes else None
            self.steps.zero_()
        if mode == "powf":
            from paper_2207_04228_b200 import _native

            self.pws_bytes = _native.power_workspace_bytes(batch, n, _native.make_config(self.cfg, n))
            self.pws = torch.empty((self.pws_bytes + 256,), dtype=torch.uint8, device=dev)
            self.pws_ptr = (self.pws.data_ptr() + 255) & ~255 if self.pws_bytes else None
            self.steps.zero_()
        self.launches = 1 if mode in ("fwd", "val") or (mode in ("powf", "scatpow") and n <= 8) else 2
        if mode == "scatpow" and n > 8:
            self.launches = 3 if n > 24 else 2  # scatter, forward (+ power kernel above n = 24)

    def __call__(self):
        if self.mode == "scatpow":  # S^(-1/2) of the samples' scatter: the whitening matrix
            from paper_2207_04228_b200 import _native

            c = _native.make_config(self.cfg, self.n)
            _native.scatter_forward_f32(self.a.data_ptr(), self.batch, self.n, 4 * self.n, 1e-3,
                                        self.lam.data_ptr(), self.vec.data_ptr(),
                                        self.status.data_ptr(), None, c, 1, -0.5, -1.0,
                                        self.pws_ptr, self.pws_bytes,
                                        self.torch.cuda.current_stream().cuda_stream)
            return
        if self.mode == "powf":
            from paper_2207_04228_b200 import _native

            c = _native.make_config(self.cfg, self.n)
            _native.forward_power_f32(self.a.data_ptr(), self.batch, self.n, self.lam.data_ptr(),
                                      self.vec.data_ptr(), self.status.data_ptr(), None, c, -0.5, -1.0,
                                      self.pws_ptr, self.pws_bytes,
                                      self.torch.cuda.current_stream().cuda_stream)
            return
        self.bed.forward_into(self.a, self.cfg, self.lam, self.vec, self.status, self.steps,
                              ws=self.ws)
        if self.mode == "fwdpow":  # A^(-1/2), the decorrelated-BN / ZCA consumer
            from paper_2207_04228_b200 import _native

            _native.matrix_power_f32(self.vec.data_ptr(), self.lam.data_ptr(), self.pw.data_ptr(),
                                     self.pst.data_ptr(), None, self.batch, self.n, -0.5, -1.0,
                                     self.torch.cuda.current_stream().cuda_stream)
        if self.mode == "fwdbwd":
            self.ga = self.bed.taylor_backward(self.vec, self.lam, self.gv, self.gl)


def time_steps(torch, step, k, w, dist=None):
    for _ in range(w):
        step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        step()
    e1.record()
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) * 1e-3
    if dist is not None:
        t = torch.tensor([sec], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        sec = float(t.item())
    return sec


def cpu_oracle_rate(n, sample, threads, mode="fwd", a=None):
    """Matrices/s of the reference algorithm's C restatement (oracle/) on
    host cores: per-matrix gating, same tolerance/budget as the GPU run.
    `a`: the inputs, generated here when not given (generation is untimed)."""
    import oracle

    if a is None:
        a = oracle.gen_spd(sample, n, 12345)
    t0 = time.perf_counter()
    r = oracle.forward(a, deflation_tol=TOL, max_double_steps=4 * n, gate=oracle.GATE_MATRIX,
                       threads=threads, chunk=max(64, sample // (8 * threads)))
    t1 = time.perf_counter()
    sec = t1 - t0
    if mode == "fwdbwd":
        rng = np.random.default_rng(1)
        gv = rng.standard_normal((sample, n, n))
        t0 = time.perf_counter()
        oracle.taylor_backward(r.eigenvectors, r.eigenvalues, gv, None)
        sec += time.perf_counter() - t0
    return sample / sec, sec


def calibrated_sample(n, threads, target_s, cap):
    rate, _ = cpu_oracle_rate(n, 2048 if n <= 16 else 256, threads)
    return int(max(256, min(cap, rate * target_s)))


def e2e_host(torch, bed, n, batch, steps, dev_index):
    """Same metric through the C ABI host-buffer entry bed_forward_host_f32
    (the reference-facing call on numpy-side buffers): per step the H2D copy
    of A from page-locked memory, the solve, and the D2H copy of eigenvalues,
    eigenvectors and per-matrix status, all inside the timed region."""
    from paper_2207_04228_b200 import _native

    a = bed.datagen.gen_spd_device(batch, n, 7, device=f"cuda:{dev_index}").cpu().pin_memory()
    lam = torch.empty((batch, n), dtype=torch.float32).pin_memory()
    vec = torch.empty((batch, n, n), dtype=torch.float32).pin_memory()
    st = torch.empty((batch,), dtype=torch.int32).pin_memory()
    cfg = _native.make_config(bed.SolverConfig(deflation_tol=TOL, max_double_steps=4 * n), n)
    call = lambda: _native.forward_host_f32(a.data_ptr(), batch, n, lam.data_ptr(),  # noqa: E731
                                            vec.data_ptr(), st.data_ptr(), None, cfg, dev_index)
    call()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        call()
        times.append(time.perf_counter() - t0)
    assert int(st.max()) == 0, "e2e solve reported a nonzero status"
    sec = statistics.median(times)
    return {"value": batch / sec, "unit": UNIT, "h2d_bytes_per_step": 4 * batch * n * n,
            "d2h_bytes_per_step": 4 * batch * (n * n + n) + 4 * batch,
            "path": "C ABI bed_forward_host_f32, page-locked host buffers, median of "
                    f"{steps} calls (chunked 3-stream copy/compute overlap)"}


def e2e_numpy_api(bed, n, batch, steps):
    """The reference-facing Python call exactly as a reference user makes it:
    batched_eig(BatchedSymmetric(float64 numpy)) -> float64 numpy results
    (solver.py:79-112) -> bed_forward_host_f64: float64 validation +
    symmetrisation and the FP32 cast on host threads into page-locked staging,
    H2D, solve, D2H, float64 results -- all timed, chunks overlapped."""
    from paper_2207_04228_b200.datagen import gen_spd_device

    # the same distribution, generated by the package (oracle/ stays the
    # checker); float64 on the host, as a reference user holds it
    a = gen_spd_device(min(batch, 1 << 20), n, 7).double().cpu().numpy()
    cfg = bed.SolverConfig(deflation_tol=TOL, max_double_steps=4 * n)
    bed.batched_eig(bed.BatchedSymmetric(a), cfg)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        bed.batched_eig(bed.BatchedSymmetric(a), cfg)
        times.append(time.perf_counter() - t0)
    sec = statistics.median(times)
    b = a.shape[0]
    return {"value": b / sec, "unit": UNIT, "batch": b, "h2d_bytes_per_step": 4 * b * n * n,
            "d2h_bytes_per_step": 4 * b * (n * n + n) + 24 * b,
            "host_threads": min(os.cpu_count() or 1, 64),
            "path": "batched_eig(BatchedSymmetric(float64 numpy)) -> C ABI bed_forward_host_f64 "
                    f"(host-thread float64 validate/cast overlapped with PCIe and the solve), median of "
                    f"{steps} calls"}


def load_traffic(name):
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(name, {}).get("dram_bytes_per_launch")
    except Exception:  # noqa: BLE001
        return None


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2207_04228_b200 as bed
    import paper_2207_04228_b200.datagen  # noqa: F401

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        pg = dist
    hbm_peak, peak_src = peaks()
    n, batch = HEADLINE["n"], HEADLINE["batch"]
    step = Step(torch, bed, n, batch, "fwd", dev, seed=100 + rank)
    with ClockSampler(local) as clk:
        sec = time_steps(torch, step, args.steps, args.warmup, pg)
    per_step = sec / args.steps
    value = world * batch / per_step
    bound, frac, flops, nbytes = roofline(n, "fwd", batch, per_step, hbm_peak)
    achieved = nbytes / per_step / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: Q diag(lam) Q^T, lam log-uniform over 3 decades (reference gen_spd "
                "distribution), generated on device",
        "config": {"workload": "c2: 4x4 ED forward, 4194304 matrices per GPU", "n": n,
                   "batch_per_gpu": batch, "global_batch": world * batch,
                   "deflation_tol": TOL, "effective_deflation_tol": 2.0 ** -22,
                   "max_double_steps": 4 * n, "gating": "per-matrix",
                   "l2": "no flush: 576 MB working set per step > 126 MB L2",
                   "parallelism": f"batch sharded, {world} rank(s), no collective"},
        "gpu_launches": args.steps * step.launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak / 1e9,
                     "unit": "GB/s", "frac": achieved / (hbm_peak / 1e9),
                     "traffic": load_traffic("bed_small_kernel<4,1>"),
                     "kernel": "bed_small_kernel<4, true>", "peak_source": peak_src,
                     "bytes_per_matrix": work_per_matrix(n, "fwd")[1],
                     "fp32_frac": flops / per_step / FP32_PEAK,
                     "fp32_peak": "73.7 TFLOP/s measured (profiles/r01_fp32_peak.md)"},
        "clocks": clk.summary(),
    }
    mean_steps = float(step.steps.float().mean())
    line["config"]["mean_double_steps"] = mean_steps
    line["config"]["qr_useful_lane_frac"] = float(
        mean_steps / step.steps.float().view(-1, 32).max(dim=1).values.mean())
    line["config"]["max_double_steps_used"] = int(step.steps.max())
    if world > 1:
        dist.barrier()
    if rank == 0:
        t0 = time.perf_counter()

        def lap(what):  # wall time of each section, on stderr (the JSON line stays on stdout)
            nonlocal t0
            t1 = time.perf_counter()
            print(f"[bench] {what}: {t1 - t0:.1f} s", file=sys.stderr, flush=True)
            t0 = t1

        line["e2e"] = e2e_host(torch, bed, n, batch, max(3, min(args.steps, 10)), local)
        lap("e2e (C ABI host path)")
        line["e2e_numpy_api"] = e2e_numpy_api(bed, n, batch, 3)
        lap("e2e (float64 numpy API)")
        if not args.quick:
            line["other_configs"] = other_configs(torch, bed, dev, hbm_peak)
            lap("other_configs")
        threads = os.cpu_count() or 1
        # a bounded sample (~10 s of host work): repeated solves of one batch
        # of up to 2^20 matrices, so memory stays small
        sample = calibrated_sample(n, threads, 3.0, 1 << 20)
        import oracle

        a_cpu = oracle.gen_spd(sample, n, 12345)  # generated once, solved repeatedly
        total, secs, reps = 0, 0.0, 0
        while secs < 10.0 and reps < 1000:
            _, dt = cpu_oracle_rate(n, sample, threads, a=a_cpu)
            total += sample
            secs += dt
            reps += 1
        rate = total / secs
        lap("cpu_baseline")
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": f"{reps} x {sample} 4x4 matrices (same distribution), oracle/ "
                                          "C restatement of the reference solver, per-matrix gate, "
                                          f"tol {TOL:g}, budget 16, {threads} threads, {secs:.1f} s"}
        te = torch_eigh_ms(torch, step.a)
        lap("torch.linalg.eigh baseline")
        line["torch_eigh_baseline"] = (
            {"value": batch / (te * 1e-3), "unit": UNIT, "batch": batch, "ms": te,
             "what": "torch.linalg.eigh fp32 on the same resident batch, 1 B200, CUDA events"}
            if te else {"unavailable": "torch.linalg.eigh failed"})
        if not args.quick:
            try:
                line["reference_numba"] = reference_numba(n)
            except Exception as exc:  # noqa: BLE001
                line["reference_numba"] = {"unavailable": str(exc)[:160]}
            lap("reference_numba")
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def torch_eigh_ms(torch, a, reps=3):
    """torch.linalg.eigh (cuSOLVER batched syevj, FP32) on the same resident
    batch, CUDA-event time per full pass (best of `reps`; one pass when a
    pass takes over half a second).  Batches cuSOLVER rejects whole are
    passed in chunks (16384, else 4096 matrices; cusolverDnXsyevBatched rejects
    32768 and up) inside the timed region."""

    def run(chunk):
        if not chunk:
            torch.linalg.eigh(a)
            return
        for lo in range(0, a.shape[0], chunk):
            torch.linalg.eigh(a[lo:lo + chunk])

    try:  # cuSOLVER handle creation and workspace queries happen on the first call
        torch.linalg.eigh(a[: min(a.shape[0], 64)])
        torch.cuda.synchronize()
    except Exception:  # noqa: BLE001
        pass
    # cusolverDnXsyevBatched rejects whole batches of 32768 and up: go straight to chunks
    for chunked in ((0,) if a.shape[0] < 32768 else ()) + (1 << 14, 1 << 12):
        try:
            best = float("inf")
            for r in range(reps + 1):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                run(chunked)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1)
                if r > 0 or ms > 500.0:
                    best = min(best, ms)
                if ms > 500.0:
                    break
            return best
        except Exception as e:  # noqa: BLE001
            print(f"torch.linalg.eigh chunk={chunked} on {tuple(a.shape)}: {type(e).__name__}: "
                  f"{str(e)[:200]}", file=sys.stderr)
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
    return None


def other_configs(torch, bed, dev, hbm_peak):
    """C1/C3 (b=512, launch-bound), C4 (n=16 fwd+bwd), C5 (n=64 fwd+bwd),
    and the n sweep at large batch -- reported beside the headline, each with
    torch.linalg.eigh on the same tensors (forward rows)."""
    rows = []
    cases = [(4, 512, "fwd"), (8, 512, "fwd"), (16, 512, "fwd"), (24, 512, "fwd"), (32, 512, "fwd"),
             (8, 1 << 20, "fwd"), (16, 1 << 18, "fwd"), (24, 1 << 17, "fwd"), (32, 1 << 16, "fwd"),
             (64, 8192, "fwd"), (16, 65536, "fwdbwd"), (64, 8192, "fwdbwd"),
             (16, 65536, "fwdpow"), (64, 8192, "fwdpow"),
             (4, 1 << 22, "val"), (16, 1 << 18, "val"), (32, 1 << 16, "val"), (64, 8192, "val"),
             (4, 1 << 22, "fwdpow"), (4, 1 << 22, "powf"), (16, 65536, "powf"),
             (4, 1 << 20, "scatpow"), (8, 1 << 18, "scatpow"), (16, 65536, "scatpow")]
    for n, b, mode in cases:
        t_row = time.perf_counter()
        st = Step(torch, bed, n, b, mode, dev, seed=n)
        reps = 50 if b <= 4096 else 10
        # best of three timed blocks after warm-up: the first calls at a new
        # size can pay one-off costs (module load, workspace pool growth)
        sec = min(time_steps(torch, st, reps, 5) for _ in range(3)) / reps
        bound, frac, _, _ = roofline(n, mode, b, sec, hbm_peak)
        stp = st.steps.float()
        wmax = stp[: b // 32 * 32].view(-1, 32).max(dim=1).values.mean() if b >= 32 else stp.max()
        row = {"n": n, "batch": b, "mode": mode, "ms": sec * 1e3, "value": b / sec,
               "roofline_bound": bound, "roofline_frac": frac,
               "mean_double_steps": float(stp.mean()),
               # warp-synchronous QR: lanes idle once their matrix is done
               "qr_useful_lane_frac": float(stp.mean() / wmax) if float(wmax) > 0 else None}
        if mode == "fwd":
            te = torch_eigh_ms(torch, st.a)
            row["torch_eigh_ms"] = te
            row["speedup_vs_torch_eigh"] = (te / (sec * 1e3)) if te else None
        rows.append(row)
        print(f"[bench]   row n={n} b={b} {mode}: {time.perf_counter() - t_row:.1f} s", file=sys.stderr, flush=True)
        del st
        torch.cuda.empty_cache()
    return rows


REF_PATH = os.path.join(ROOT, "baseline", "_ref")


_NUMBA_CHUNK = {}


def _numba_chunk(key):
    """One chunk through the unmodified reference (baseline/_ref) in a forked
    pool worker; the chunk itself was inherited through fork (no pickling)."""
    import batchedeig as ref

    a, n = _NUMBA_CHUNK[key]
    cfg = ref.SolverConfig(deflation_tol=TOL, max_double_steps=4 * n)
    ref.batched_eig(ref.BatchedSymmetric(a), cfg)
    return a.shape[0]


def reference_numba(n, target_s=6.0):
    """The UNMODIFIED reference package (pip-installed into baseline/_ref)
    through its own public API: batchedeig.batched_eig on host arrays from
    its own gen_spd, verify profile (bench.py:40, :227-228).  (i) as shipped,
    one process on one batch; (ii) sharded over every host core (fork pool,
    chunks of 4096 / 2048 / 256 matrices for n = 4 / 16 / 64).
    None if baseline/_ref is absent."""
    if not os.path.isdir(os.path.join(REF_PATH, "batchedeig")):
        return None
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    import multiprocessing as mproc

    import batchedeig as ref
    from batchedeig.bench import gen_spd

    cfg = ref.SolverConfig(deflation_tol=TOL, max_double_steps=4 * n)
    warm = gen_spd(64, n, 1, 3.0).data
    ref.batched_eig(ref.BatchedSymmetric(warm), cfg)  # numba JIT / cache load
    chunk = 4096 if n <= 4 else (2048 if n <= 16 else 256)
    a = gen_spd(chunk, n, 2, 3.0).data
    t0 = time.perf_counter()
    ref.batched_eig(ref.BatchedSymmetric(a), cfg)
    one = time.perf_counter() - t0
    reps = max(1, int(target_s / 2 / max(one, 1e-6)))
    t0 = time.perf_counter()
    for _ in range(reps):
        ref.batched_eig(ref.BatchedSymmetric(a), cfg)
    single = chunk * reps / (time.perf_counter() - t0)
    procs = os.cpu_count() or 1
    jobs = ["run"] * max(procs, int(procs * single * target_s / 2 / chunk))
    _NUMBA_CHUNK["warm"] = (warm, n)
    _NUMBA_CHUNK["run"] = (a, n)
    ctx = mproc.get_context("fork")
    with ctx.Pool(procs) as pool:
        pool.map(_numba_chunk, ["warm"] * procs)  # JIT / cache load in every worker
        t0 = time.perf_counter()
        done = sum(pool.map(_numba_chunk, jobs))
        multi = done / (time.perf_counter() - t0)
    return {"as_shipped": {"value": single, "unit": UNIT, "cores": 1,
                           "sample": f"{reps} x batched_eig on {chunk} {n}x{n} gen_spd matrices"},
            "all_cores": {"value": multi, "unit": UNIT, "cores": procs,
                          "sample": f"{len(jobs)} chunks of {chunk} over a {procs}-process fork pool"},
            "kind": "reference", "path": "baseline/_ref batchedeig.batched_eig (numba "
                                         "kernels, batch-wide deflation gate), verify profile"}


def run_reference(args):
    """The reference algorithm on the host cores (oracle/ C restatement:
    the reference is numba Python that cannot travel to the GPU box), same
    config, metric and unit; each step a bounded sample of the workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = HEADLINE["n"]
    threads = os.cpu_count() or 1
    budget = 60.0 / max(1, args.steps + args.warmup)
    sample = calibrated_sample(n, threads, budget, HEADLINE["batch"])
    import oracle

    a = oracle.gen_spd(sample, n, 12345)  # generated once (untimed), solved every step
    for _ in range(args.warmup):
        cpu_oracle_rate(n, sample, threads, a=a)
    secs = [cpu_oracle_rate(n, sample, threads, a=a)[1] for _ in range(args.steps)]
    sec = statistics.median(secs)
    value = sample / sec
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "impl": "reference",
        "data": "synthetic: reference gen_spd restatement (oracle.gen_spd)",
        "config": {"workload": "c2: 4x4 ED forward (bounded host sample per step)", "n": n,
                   "batch_per_step": sample, "deflation_tol": TOL, "max_double_steps": 4 * n,
                   "gating": "per-matrix"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{sample} matrices per step, oracle/bed_oracle.c (float64 "
                                   f"restatement of batchedeig.batched_eig), {threads} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    try:
        line["reference_numba"] = reference_numba(n, target_s=4.0)
    except Exception as exc:  # noqa: BLE001
        line["reference_numba"] = {"unavailable": str(exc)[:160]}
    print(json.dumps(line), flush=True)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--quick", action="store_true", help="skip the other_configs sweep")
    args = p.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
