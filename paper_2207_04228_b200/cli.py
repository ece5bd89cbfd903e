"""Command-line harness on the GPU path, mirroring the
reference ``batchedeig`` CLI (/root/reference/pkg/src/batchedeig/cli.py):

  solve   decompose a BED1 batch file -> <out>.values.bed, <out>.vectors.bed
  gen     write a random SPD batch (reference gen_spd distribution) as BED1
  bench   time GPU solves over a (dims x batches) grid, CSV to stdout in the
          reference schema (bench.py:42)

Exit codes as the reference: 0 success, 1 solve failure, 2 usage error,
3 I/O or file-format error.  The reference's ``verify`` (a Jacobi-oracle
sweep) is test infrastructure here: ``tests/`` with the oracle in
``oracle/``, not part of the product.

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
    print(f"solved batch={batch.data.shape[0]} dim={batch.data.shape[1]}: "
          f"double_steps={res.diagnostics.double_steps}", file=sys.stderr)
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
            forward_into(a, cfg, lam, vec, None, steps)  # warm-up
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
            # mean_r / rotations are batch-gate counters of the reference loop
            # (not kept per matrix on the device); max_eig_err is left empty
            out.append(f"{n},{b},{args.mode},{med:.9e},{med / b:.9e},-1,{k:.3f},-1,")
    sys.stdout.write("\n".join(out) + "\n")
    return EXIT_OK


def main(argv=None) -> int:
    args = _parser().parse_args(argv)
    handler = {"solve": _cmd_solve, "gen": _cmd_gen, "bench": _cmd_bench}[args.command]
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
