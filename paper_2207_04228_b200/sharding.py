"""Host-side batch sharding across GPUs (north-star subsystem 5).

The reference solves one batch in one process (its only coupling between
matrices is the batch-wide deflation gate, _kernels.py:303-318, which the
device path replaces with per-matrix gating).  With per-matrix gating every
matrix is independent, so a batch shards into contiguous slices, one per GPU
(one process per GPU, ``torch.distributed``), with no collective on the hot
path.  Results are bit-identical for any number of shards.  A gather of the
outputs (NCCL all-gather over NVLink) is offered only for callers that need
the whole batch on every rank.
"""

from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist

from .core import SolverConfig

__all__ = ["shard_bounds", "shard_sizes", "solve_shard", "gather_shards", "batched_eig_devices"]


def shard_sizes(batch: int, world: int) -> list[int]:
    """Sizes of the contiguous slices: ceil(batch / world) each, the last
    ones shorter (possibly empty)."""
    if batch < 0 or world < 1:
        raise ValueError("batch must be >= 0 and world >= 1")
    per = -(-batch // world) if batch else 0
    return [max(0, min(per, batch - r * per)) for r in range(world)]


def shard_bounds(batch: int, world: int, rank: int) -> tuple[int, int]:
    """[start, stop) of rank's slice."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    per = -(-batch // world) if batch else 0
    start = min(batch, rank * per)
    return start, min(batch, start + per)


def solve_shard(a: torch.Tensor, cfg: SolverConfig | None = None, *, world: int | None = None,
                rank: int | None = None, presharded: bool = False,
                solve_fn: Callable | None = None):
    """Solve this rank's slice.

    ``a`` is either the full batch (every rank holds it; the rank slices its
    part) or, with ``presharded=True``, already this rank's slice.  Returns
    ``(start, stop, result)`` with ``result`` the ``EigenResult`` of the slice.
    ``solve_fn`` defaults to the device :func:`batched_eig`; tests inject a
    CPU solver to exercise the host logic without a GPU.
    """
    if solve_fn is None:
        from .solver import batched_eig as solve_fn  # noqa: N813
    world = dist.get_world_size() if world is None else world
    rank = dist.get_rank() if rank is None else rank
    if presharded:
        sizes = shard_sizes_global(a.shape[0], world)
        start = sum(sizes[:rank])
        stop = start + a.shape[0]
        local = a
    else:
        start, stop = shard_bounds(a.shape[0], world, rank)
        local = a[start:stop]
    if stop <= start:
        return start, stop, None
    return start, stop, solve_fn(local, cfg)


def shard_sizes_global(local_batch: int, world: int) -> list[int]:
    """Slice sizes when every rank holds ``local_batch`` matrices (weak scaling)."""
    return [local_batch] * world


def gather_shards(local: torch.Tensor, batch: int, group=None) -> torch.Tensor:
    """All-gather rank slices (as cut by :func:`shard_bounds`) into the full
    batch on every rank.  Uneven tails are padded for the collective and
    trimmed after."""
    world = dist.get_world_size(group)
    sizes = shard_sizes(batch, world)
    per = max(sizes) if sizes else 0
    pad = torch.zeros((per,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(out, pad, group=group)
    return torch.cat([o[:s] for o, s in zip(out, sizes)], dim=0)


def batched_eig_devices(a: torch.Tensor, cfg: SolverConfig | None = None,
                        devices: list[int] | None = None, out_device: int | str | None = None):
    """Single-process sharding: the batch is cut into ``len(devices)``
    contiguous slices (:func:`shard_bounds`), each solved on its own device
    and CUDA stream -- the H2D copy of the slice, the solve and the copy of
    its results into the output run on that stream, so the devices (or, with
    a device listed twice, two streams of one device) work concurrently.  No
    collective: every matrix is independent (per-matrix deflation).

    ``a`` is a (batch, n, n) float32 tensor on any device or the host (pin
    it for asynchronous copies).  Results land on ``out_device`` (default:
    the first listed device) and are bit-identical to one
    ``batched_eig`` call on the whole batch.  Raises like ``batched_eig``.
    """
    from . import solver
    from .core import EigenResult

    cfg = cfg or SolverConfig()
    devices = list(range(torch.cuda.device_count())) if devices is None else list(devices)
    if not devices:
        raise RuntimeError("batched_eig_devices needs at least one CUDA device")
    if a.ndim != 3 or a.shape[1] != a.shape[2]:
        raise ValueError(f"expected (batch, n, n), got {tuple(a.shape)}")
    b, n, _ = a.shape
    out_dev = torch.device("cuda", devices[0]) if out_device is None else torch.device(out_device)
    evals = torch.empty((b, n), device=out_dev, dtype=torch.float32)
    evecs = torch.empty((b, n, n), device=out_dev, dtype=torch.float32) if cfg.compute_vectors else None
    status = torch.empty((b,), device=out_dev, dtype=torch.int32)
    steps = torch.empty((b,), device=out_dev, dtype=torch.int32)
    diag = torch.empty((b, 3), device=out_dev, dtype=torch.int32)
    resid = torch.empty((b,), device=out_dev, dtype=torch.float32)
    producer = torch.cuda.current_stream(a.device) if a.is_cuda else None
    consumer = torch.cuda.current_stream(out_dev) if out_dev.type == "cuda" else None
    streams = []
    for r, d in enumerate(devices):
        lo, hi = shard_bounds(b, len(devices), r)
        if hi <= lo:
            continue
        dev = torch.device("cuda", d)
        st = torch.cuda.Stream(dev)
        streams.append(st)
        with torch.cuda.device(dev), torch.cuda.stream(st):
            if producer is not None:
                st.wait_stream(producer)
            local = a[lo:hi].to(dev, non_blocking=True).contiguous()
            if consumer is not None:
                st.wait_stream(consumer)  # the output buffers are ready
            le = torch.empty((hi - lo, n), device=dev, dtype=torch.float32)
            lv = torch.empty((hi - lo, n, n), device=dev, dtype=torch.float32) if evecs is not None else None
            ls = torch.empty((hi - lo,), device=dev, dtype=torch.int32)
            lk = torch.empty((hi - lo,), device=dev, dtype=torch.int32)
            ld = torch.empty((hi - lo, 3), device=dev, dtype=torch.int32)
            lr = torch.empty((hi - lo,), device=dev, dtype=torch.float32)
            solver.forward_into(local, cfg, le, lv, ls, lk, diag=ld, resid=lr)
            evals[lo:hi].copy_(le, non_blocking=True)
            if lv is not None:
                evecs[lo:hi].copy_(lv, non_blocking=True)
            status[lo:hi].copy_(ls, non_blocking=True)
            steps[lo:hi].copy_(lk, non_blocking=True)
            diag[lo:hi].copy_(ld, non_blocking=True)
            resid[lo:hi].copy_(lr, non_blocking=True)
            for t in (evals, evecs, status, steps, diag, resid):
                if t is not None and t.is_cuda:
                    t.record_stream(st)
    for st in streams:
        if consumer is not None:
            consumer.wait_stream(st)
        else:
            st.synchronize()
    flags = 0
    for code in torch.unique(status.cpu()).tolist():
        flags |= (1 << code) if code else 0
    solver._raise_for_status(a, status, flags, cfg, resid)
    return EigenResult(evals, evecs, solver._diagnostics(steps, diag))
