"""Command-line harness on the GPU path, mirroring the
reference ``batchedeig`` CLI (/root/reference/pkg/src/batchedeig/cli.py):

  solve   decompose a BED1 batch file -> <out>.values.bed, <out>.vectors.bed
  gen     write a random SPD batch (reference gen_spd distribution) as BED1
  bench   time GPU solves over a (dims x batches) grid, CSV to stdout in the
          reference schema (bench.py:42)
  verify  solve >= count matrices per grid cell on the GPU and check them on
          the host in float64 (cli.py:107-127, bench.py:222-376): eigenvalues
          against LAPACK (numpy.linalg.eigvalsh, the checker here where the
          reference uses its Jacobi oracle), reconstruction and
          orthogonality residuals, batch-vs-single agreement; the reference's
          table / CSV columns and exit status (1 if any cell fails)

Exit codes as the reference: 0 success, 1 solve failure, 2 usage error,
3 I/O or file-format error.

Run: ``python -m paper_2207_04228_b200.cli <command> ...``
"""

from __future__ import annotations

import argparse
import sys

import numpy as np

from .bed_io import read_batch, write_batch
from .core import (
    BadMagic,
    BatchedEigError,
    BatchedMatrix,
    DimMismatch,
    SolverConfig,
    TruncatedPayload,
)

EXIT_OK, EXIT_FAIL, EXIT_USAGE, EXIT_IO = 0, 1, 2, 3
CSV_HEADER = "dim,batch,mode,median_wall_s,per_matrix_s,mean_r,mean_k,rotations,max_eig_err"


def _ints(text: str) -> tuple[int, ...]:
    try:
        vals = tuple(int(p) for p in text.split(",") if p)
    except ValueError:
        raise argparse.ArgumentTypeError(f"expected comma-separated integers, got {text!r}")
    if not vals:
        raise argparse.ArgumentTypeError("expected at least one integer")
    return vals


def _parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="bed200", description="Batched symmetric ED on B200.")
    sub = p.add_subparsers(dest="command", required=True)
    grid = argparse.ArgumentParser(add_help=False)
    grid.add_argument("--dims", type=_ints, default=(4, 8, 16))
    grid.add_argument("--batches", type=_ints, default=(1, 64))
    grid.add_argument("--seed", type=int, default=0)
    grid.add_argument("--decades", type=float, default=3.0)
    s = sub.add_parser("solve", help="decompose a BED1 batch file")
    s.add_argument("input")
    s.add_argument("--out", required=True, help="writes <out>.values.bed and <out>.vectors.bed")
    s.add_argument("--no-vectors", action="store_true")
    s.add_argument("--tol", type=float, default=None)
    g = sub.add_parser("gen", parents=[grid], help="random SPD batch as BED1")
    g.add_argument("--out", required=True)
    b = sub.add_parser("bench", parents=[grid], help="time GPU solves, CSV to stdout")
    b.add_argument("--reps", type=int, default=5)
    b.add_argument("--mode", choices=("values", "full"), default="full")
    b.add_argument("--tol", type=float, default=None)
    v = sub.add_parser("verify", parents=[grid], help="run the invariant suite over a grid")
    v.add_argument("--count", type=int, default=256, help="minimum matrices per cell")
    # the reference gates float64 at 1e-8; this path computes in FP32 (north star: 1e-5)
    v.add_argument("--tol", type=float, default=1e-5,
                   help="eigenvalue / residual gate, scaled by the spectral radius")
    v.add_argument("--deflation-tol", type=float, default=3e-12,
                   help="deflation threshold of the verification solves (bench.py:40)")
    v.add_argument("--csv", action="store_true", help="per-cell CSV instead of the table")
    return p


def _cfg(tol, vectors: bool) -> SolverConfig:
    return SolverConfig(compute_vectors=vectors) if tol is None else \
        SolverConfig(compute_vectors=vectors, deflation_tol=tol)


def _cmd_solve(args) -> int:
    from .solver import batched_eig

    batch = read_batch(args.input)
    res = batched_eig(batch, _cfg(args.tol, not args.no_vectors))
    write_batch(BatchedMatrix(np.asarray(res.eigenvalues)[:, :, None]), f"{args.out}.values.bed")
    if not args.no_vectors:
        write_batch(BatchedMatrix(np.asarray(res.eigenvectors)), f"{args.out}.vectors.bed")
    d = res.diagnostics
    print(f"solved batch={batch.data.shape[0]} dim={batch.data.shape[1]}: "
          f"double_steps={d.double_steps} mean_reductions={d.reductions:.3f} "
          f"rotations={d.rotation_count}", file=sys.stderr)
    return EXIT_OK


def _cmd_gen(args) -> int:
    if len(args.dims) != 1 or len(args.batches) != 1:
        print("gen needs exactly one value in --dims and --batches", file=sys.stderr)
        return EXIT_USAGE
    from .datagen import gen_spd_device

    a = gen_spd_device(args.batches[0], args.dims[0], args.seed, args.decades)
    write_batch(a, args.out)
    print(f"wrote batch={args.batches[0]} dim={args.dims[0]} to {args.out}", file=sys.stderr)
    return EXIT_OK


def _cmd_bench(args) -> int:
    import torch

    from .datagen import gen_spd_device
    from .solver import forward_into

    out = [CSV_HEADER]
    for n in args.dims:
        for b in args.batches:
            a = gen_spd_device(b, n, args.seed, args.decades)
            cfg = _cfg(args.tol, args.mode == "full")
            lam = torch.empty((b, n), device=a.device)
            vec = torch.empty((b, n, n), device=a.device) if cfg.compute_vectors else None
            steps = torch.empty((b,), device=a.device, dtype=torch.int32)
            diag = torch.empty((b, 3), device=a.device, dtype=torch.int32)
            forward_into(a, cfg, lam, vec, None, steps, diag=diag)  # warm-up (and counters)
            times = []
            for _ in range(max(1, args.reps)):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                forward_into(a, cfg, lam, vec, None, steps)
                e1.record()
                e1.synchronize()
                times.append(e0.elapsed_time(e1) * 1e-3)
            med = float(np.median(times))
            k = float(steps.float().mean())
            tot = diag.long().sum(dim=0).tolist()
            nsteps = int(steps.long().sum())
            mean_r = tot[2] / nsteps if nsteps else 0.0
            # max_eig_err stays empty outside verify runs, as in the reference
            out.append(f"{n},{b},{args.mode},{med:.9e},{med / b:.9e},{mean_r:.6f},{k:.3f},{tot[0]},")
    sys.stdout.write("\n".join(out) + "\n")
    return EXIT_OK


def _verify_cell(n: int, b: int, args):
    """One grid cell of the verify sweep (reference bench.py:222-300)."""
    import torch

    from .datagen import gen_spd_device
    from .solver import batched_eig

    cfg = SolverConfig(deflation_tol=args.deflation_tol, max_double_steps=4 * n)
    cell = dict(dim=n, batch=b, count=0, eig=0.0, recon=0.0, orth=0.0, single=0.0, r=[], k=0,
                fails=0)
    solves = max(1, -(-args.count // b))
    eye = np.eye(n)
    for s in range(solves):
        a = gen_spd_device(b, n, args.seed * 7919 + n * 131 + b * 17 + s, args.decades)
        res = batched_eig(a, cfg)
        lam = res.eigenvalues.double().cpu().numpy()
        v = res.eigenvectors.double().cpu().numpy()
        ad = a.double().cpu().numpy()
        ref = np.linalg.eigvalsh(ad)[:, ::-1]
        rho = np.maximum(np.abs(ref).max(axis=1), 1e-300)
        eig = np.abs(lam - ref).max(axis=1) / rho
        recon = np.linalg.norm(ad @ v - v * lam[:, None, :], axis=(1, 2)) / np.maximum(
            np.linalg.norm(ad, axis=(1, 2)), 1e-300)
        orth = np.linalg.norm(v.transpose(0, 2, 1) @ v - eye, axis=(1, 2)) / n
        cell["fails"] += int(np.sum((eig > args.tol) | (recon > args.tol) | (orth > args.tol)))
        cell["eig"] = max(cell["eig"], float(eig.max()))
        cell["recon"] = max(cell["recon"], float(recon.max()))
        cell["orth"] = max(cell["orth"], float(orth.max()))
        d = res.diagnostics
        cell["r"].append(d.reductions)
        cell["k"] = max(cell["k"], d.double_steps)
        cell["count"] += b
        if b > 1 and s == 0:  # batch-vs-single: per-matrix deflation makes them identical
            for j in range(min(b, 16)):
                one = batched_eig(a[j:j + 1].contiguous(), cfg).eigenvalues
                dev = float((one[0] - res.eigenvalues[j]).abs().max())
                cell["single"] = max(cell["single"], dev)
                cell["fails"] += int(dev > args.tol * float(rho[j]))
        del a, res
        torch.cuda.empty_cache()
    cell["passed"] = cell["fails"] == 0
    return cell


def _cmd_verify(args) -> int:
    cells = [_verify_cell(n, b, args) for n in args.dims for b in args.batches]
    if args.csv:
        print("dim,batch,count,max_eig_err,max_recon,max_orth,max_single_dev,r_median,passed")
        for c in cells:
            print(f"{c['dim']},{c['batch']},{c['count']},{c['eig']:.3e},{c['recon']:.3e},"
                  f"{c['orth']:.3e},{c['single']:.3e},{float(np.median(c['r'])):.3f},{int(c['passed'])}")
    else:
        print(f"{'dim':>4} {'batch':>6} {'count':>6} {'eig_err':>10} {'recon':>10} {'orth':>10} "
              f"{'single':>10} {'r_median':>9} {'k_max':>6} {'status':>7}")
        for c in cells:
            print(f"{c['dim']:>4} {c['batch']:>6} {c['count']:>6} {c['eig']:>10.3e} {c['recon']:>10.3e} "
                  f"{c['orth']:>10.3e} {c['single']:>10.3e} {float(np.median(c['r'])):>9.3f} "
                  f"{c['k']:>6} {'pass' if c['passed'] else 'FAIL':>7}")
    return EXIT_OK if all(c["passed"] for c in cells) else EXIT_FAIL


def main(argv=None) -> int:
    args = _parser().parse_args(argv)
    handler = {"solve": _cmd_solve, "gen": _cmd_gen, "bench": _cmd_bench,
               "verify": _cmd_verify}[args.command]
    try:
        return handler(args)
    except (OSError, BadMagic, TruncatedPayload, DimMismatch) as err:
        print(f"error: {err}", file=sys.stderr)
        return EXIT_IO
    except BatchedEigError as err:
        print(f"error: {err}", file=sys.stderr)
        return EXIT_FAIL
    except ValueError as err:
        print(f"error: {err}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
