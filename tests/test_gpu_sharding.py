"""Batch sharding with the GPU solve (north-star subsystem 5):
single-process shards on several streams (one device listed twice stands in
for two devices on a one-GPU box), and two ranks of torch.distributed each
solving its slice on the GPU (gloo for the gather, both ranks on cuda:0)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle

pytestmark = pytest.mark.gpu

VERIFY = dict(deflation_tol=3e-12)


@pytest.fixture(scope="module")
def bed():
    import paper_2207_04228_b200 as bed

    return bed


@pytest.mark.parametrize("n,b,shards", [(4, 100003, 2), (16, 4099, 3), (24, 1500, 2), (40, 333, 4)])
def test_devices_streams_bitwise_equal_single_call(bed, n, b, shards):
    a = torch.from_numpy(oracle.gen_spd(b, n, 70 + n).astype(np.float32))
    cfg = bed.SolverConfig(max_double_steps=4 * n, **VERIFY)
    ref = bed.batched_eig(a.cuda(), cfg)
    for src in (a.pin_memory(), a.cuda()):
        got = bed.batched_eig_devices(src, cfg, devices=[0] * shards)
        assert torch.equal(got.eigenvalues, ref.eigenvalues)
        assert torch.equal(got.eigenvectors, ref.eigenvectors)
        assert torch.equal(got.diagnostics.converged_steps, ref.diagnostics.converged_steps)


def test_devices_raises_like_batched_eig(bed):
    a = torch.eye(4).expand(10, 4, 4).contiguous()
    a[7, 1, 2] = float("nan")
    with pytest.raises(bed.NonFinite) as err:
        bed.batched_eig_devices(a.cuda(), devices=[0, 0])
    assert err.value.batch_index == 7


def _worker(rank, world, port, n, batch, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2207_04228_b200 as bed

    torch.cuda.set_device(0)
    a = torch.from_numpy(oracle.gen_spd(batch, n, 5).astype(np.float32)).cuda()
    cfg = bed.SolverConfig(max_double_steps=4 * n, **VERIFY)
    lo, hi, res = bed.solve_shard(a, cfg)  # the device batched_eig on this rank's slice
    local = res.eigenvectors.cpu() if res is not None else torch.zeros((0, n, n))
    full = bed.gather_shards(local, batch)
    if rank == 0:
        whole = bed.batched_eig(a, cfg).eigenvectors.cpu()
        out.put((lo, hi, bool(torch.equal(full, whole))))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("n,batch", [(4, 5001), (16, 777)])
def test_two_ranks_gpu_solve_gathered_bitwise(n, batch):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, batch, q)) for r in range(2)]
    for p in procs:
        p.start()
    lo, hi, same = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert (lo, hi) == (0, (batch + 1) // 2)
    assert same
