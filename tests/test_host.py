"""CPU tests: the C ABI library loads and exports every symbol the header
declares; host-side config/error/sharding logic; a world_size-2 gloo run of
the sharded solve (with the oracle injected as the per-rank solver)."""

import os
import re
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2207_04228_b200 as bed
from paper_2207_04228_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    header = open(os.path.join(ROOT, "include", "bed200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(bed_\w+)\s*\(", header, re.M))
    assert declared == set(_native.EXPORTS)
    L = _native.lib()
    for sym in declared:
        assert getattr(L, sym) is not None
    assert L.bed_abi_version() == 2
    assert b"invalid" in L.bed_error_string(1)


def test_abi_argument_checks_need_no_gpu():
    L = _native.lib()
    cfg = _native.make_config(bed.SolverConfig(), 4)
    import ctypes

    # n out of range / null output: rejected before any CUDA call
    assert L.bed_forward_f32(None, 1, 0, None, None, None, None, None, ctypes.byref(cfg), None) == 1
    assert L.bed_forward_f32(None, 1, 65, None, None, None, None, None, ctypes.byref(cfg), None) == 1
    assert L.bed_backward_f32(None, None, None, None, None, 1, 4, -1, None, None, None) == 1
    # workspace queries are host arithmetic: exact without a GPU
    c16 = _native.make_config(bed.SolverConfig(max_double_steps=64), 16)
    assert _native.workspace_bytes(0, 16, c16) == 0
    assert _native.workspace_bytes(1000, 4, c16) == 0
    w32 = _native.workspace_bytes(32, 16, c16)
    assert 0 < w32 < _native.workspace_bytes(64, 16, c16) < _native.workspace_bytes(1 << 20, 16, c16)
    # below the 32-matrix minimum: rejected before any CUDA call
    assert L.bed_forward_ws_f32(1 << 20, 100, 16, 1 << 20, 1 << 20, None, None, None, None, None, ctypes.byref(c16),
                                1 << 20, w32 - 1, None) == 1
    bad = _native.BedConfig(1e-5, 1e-12, 8, 7, 1, 0)  # bad sort code
    assert L.bed_forward_f32(None, 0, 4, None, None, None, None, None, ctypes.byref(bad), None) == 1


def test_solver_config_mirrors_reference():
    c = bed.SolverConfig()
    assert (c.deflation_tol, c.max_double_steps, c.compute_vectors, c.sort, c.wy_block,
            c.symmetry_tol, c.strict_convergence) == (1e-5, None, True, "descending", "auto",
                                                      1e-12, True)
    assert c.resolved_max_steps(16) == 32 and c.resolved_wy_block(16) == 4
    assert c.resolved_wy_block(8) is None
    for bad in (dict(deflation_tol=-1), dict(max_double_steps=0), dict(sort="up"),
                dict(wy_block="x"), dict(wy_block=0)):
        with pytest.raises(ValueError):
            bed.SolverConfig(**bad)
    cfg = _native.make_config(bed.SolverConfig(sort="ascending", compute_vectors=False), 5)
    assert (cfg.max_double_steps, cfg.sort, cfg.compute_vectors) == (10, 2, 0)


def test_shapes_rejected():
    with pytest.raises(bed.ShapeMismatch):
        bed.BatchedSymmetric(np.zeros((2, 3, 4)))
    with pytest.raises(bed.ShapeMismatch):
        bed.BatchedSymmetric(np.zeros((0, 3, 3)))


def test_errors_carry_reference_fields():
    e = bed.NoConvergence([3, 1], 0.5)
    assert e.batch_indices == [1, 3] and e.residual_offdiag_max == 0.5
    assert bed.NonFinite(2, (0, 1)).position == (0, 1)
    assert bed.NonSymmetric(4, 1e-3).batch_index == 4
    assert issubclass(bed.NoConvergence, bed.BatchedEigError)


@pytest.mark.parametrize("batch,world", [(0, 2), (1, 2), (7, 2), (8, 4), (9, 4), (4194304, 8), (5, 8)])
def test_shard_bounds_tile_the_batch(batch, world):
    sizes = bed.shard_sizes(batch, world)
    assert sum(sizes) == batch and len(sizes) == world
    pos = 0
    for r in range(world):
        lo, hi = bed.shard_bounds(batch, world, r)
        assert lo == pos and hi - lo == sizes[r]
        pos = hi


def _oracle_solve(a, cfg):
    """CPU stand-in for the device solve (test infrastructure only)."""
    cfg = cfg or bed.SolverConfig()
    a = a.numpy() if isinstance(a, torch.Tensor) else a
    r = oracle.forward(np.asarray(a, np.float64), deflation_tol=3e-12)
    return bed.EigenResult(torch.from_numpy(r.eigenvalues), torch.from_numpy(r.eigenvectors),
                           bed.SolveDiagnostics(int(r.double_steps.max()), -1.0, -1, -1,
                                                r.double_steps))


def _worker(rank, world, port, batch, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = torch.from_numpy(oracle.gen_spd(batch, 5, 9))
    lo, hi, res = bed.solve_shard(a, solve_fn=_oracle_solve)
    local = res.eigenvalues if res is not None else torch.zeros((0, 5), dtype=torch.float64)
    full = bed.gather_shards(local, batch)
    if rank == 0:
        out.put((lo, hi, full.numpy()))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("batch", [9, 10])
def test_gloo_two_rank_sharded_solve_matches_single(batch):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, batch, q)) for r in range(2)]
    for p in procs:
        p.start()
    lo, hi, full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    single = oracle.forward(oracle.gen_spd(batch, 5, 9), deflation_tol=3e-12).eigenvalues
    np.testing.assert_array_equal(full, single)
    assert (lo, hi) == (0, (batch + 1) // 2)
