"""Per-config roofline table from a bench JSON line (and the ncu summary for
per-kernel traffic): python tools/roofline_table.py <bench.json> [round] >
profiles/<round>_roofline.md

Work model (the formulas bench.py uses):
  forward  F = (8/3) n^3 + (6n + 24) n (n - 1) flops, B = 4 (2 n^2 + n) bytes
  backward F = 6 n^3 + 22 n^2,                          B = 4 (3 n^2 + 2 n)
  power    F = 2 n^3,                                    B = 4 (2 n^2 + n)
  modes: fwd, val (eigenvalues only), fwdbwd, fwdpow (forward + power kernel), powf
  (eigenvalues + A^p in one call), scatpow (X of 4n samples -> S^p in one call,
  + n (n + 1) 4n scatter flops, B = 4 (4 n^2 + n^2 + n)) -- bench.work_per_matrix
Roofline time = max(B / HBM, F / FP32) with HBM from MEASURED_PEAKS.json and
FP32 = 73.7 TFLOP/s (measured FFMA2 peak, profiles/r01_fp32_peak.md)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import FP32_PEAK, peaks, work_per_matrix  # noqa: E402


def main(path, tag="r02"):
    line = json.loads(open(path).read().strip().splitlines()[-1])
    hbm, src = peaks()
    rows = [dict(n=line["config"]["n"], batch=line["config"]["batch_per_gpu"], mode="fwd",
                 ms=line["ms_per_step"], mean_double_steps=line["config"].get("mean_double_steps"),
                 qr_useful_lane_frac=line["config"].get("qr_useful_lane_frac"))]
    rows += line.get("other_configs", [])
    out = [f"# Roofline per configuration, {tag}", "",
           f"Source: `{os.path.relpath(path, ROOT)}` (CUDA-event device time, inputs resident).  "
           f"HBM peak {hbm / 1e9:.1f} GB/s ({src}); FP32 peak {FP32_PEAK / 1e12:.1f} TFLOP/s "
           "(measured FFMA2).  Work model: SURVEY.md 8(d).", "",
           "| n | batch | mode | ms | matrices/s | GB/s (alg.) | TFLOP/s (alg.) | bound | frac | "
           "mean steps | QR useful lanes | torch.linalg.eigh ms | speed-up |",
           "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        f, b = work_per_matrix(r["n"], r["mode"])
        sec = r["ms"] * 1e-3
        t_h, t_f = r["batch"] * b / hbm, r["batch"] * f / FP32_PEAK
        bound = "HBM" if t_h >= t_f else "FP32"
        frac = max(t_h, t_f) / sec
        te = r.get("torch_eigh_ms")
        sp = f"{te / r['ms']:.1f}x" if te else "-"
        ul = r.get("qr_useful_lane_frac")
        ms = r.get("mean_double_steps")
        out.append(f"| {r['n']} | {r['batch']} | {r['mode']} | {r['ms']:.4f} | {r['batch'] / sec:.4g} | "
                   f"{r['batch'] * b / sec / 1e9:.0f} | {r['batch'] * f / sec / 1e12:.2f} | {bound} | "
                   f"{frac:.3f} | {ms:.2f} | {ul:.2f} | {te if te is None else round(te, 3)} | {sp} |"
                   if ms is not None and ul is not None else
                   f"| {r['n']} | {r['batch']} | {r['mode']} | {r['ms']:.4f} | {r['batch'] / sec:.4g} | "
                   f"{r['batch'] * b / sec / 1e9:.0f} | {r['batch'] * f / sec / 1e12:.2f} | {bound} | "
                   f"{frac:.3f} | - | - | {te if te is None else round(te, 3)} | {sp} |")
    out.append("")
    out.append("`QR useful lanes` = mean double steps per matrix / mean over warps of the warp's "
               "largest step count: the share of the warp-synchronous band-QR loop's lane-steps "
               "that advance an unfinished matrix (the rest are exact no-op sweeps).")
    print("\n".join(out))


if __name__ == "__main__":
    main(*sys.argv[1:])
