"""The slab-sharded driver with the real CUDA evaluator: two ranks (gloo,
both on cuda:0 -- the only GPU of the test box) split the lattice into
i-slabs, run the sm_100a kernels on their slab and all-reduce one packed
buffer.  Loss, gradients and the gathered grid must equal the
single-process device path (the per-slab split plans may reorder fp64
partial sums: agreement to 1e-9 relative).  This is the N>1 code path of
bench.py; real multi-GPU runs use NCCL instead of gloo."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

RES = (20, 18, 32)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    from paper_2407_11272_b200 import configs
    v, f = configs.torus_with_holes()
    grid = ((-1.0,) * 3, (1.0,) * 3, RES)
    n = int(np.prod(RES))
    target = (np.random.default_rng(5).random(n) > 0.7).astype(np.float32)
    return v, f, grid, target


def _worker(rank, world, port, outdir, mode, strip):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2407_11272_b200 import device
    if strip:  # strip forward / strip-pair backward on every slab
        device.STRIP_MIN_NODES = 0
    from paper_2407_11272_b200.distributed import CudaSlabEvaluator, SlabDriver
    v, f, grid, target = _problem()
    dm = device.DeviceMesh.from_numpy(v, f)
    n = int(np.prod(RES))
    drv = SlabDriver(CudaSlabEvaluator(dm, grid, mode=mode), n, rank, world)
    n0, cnt = drv.slab
    tg = torch.from_numpy(target[n0:n0 + cnt]).cuda()
    loss, grads, excl, _ = drv.loss_grad(tg)
    vals, flags = drv.forward(policy=1, gather=True)
    if rank == 0:
        np.savez(os.path.join(outdir, f"out_{mode}_{int(strip)}.npz"), loss=float(loss),
                 grads=grads.cpu().numpy(), excl=float(excl), vals=vals.cpu().numpy(),
                 flags=flags.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode,strip", [("exact", False), ("soft", False), ("exact", True)])
def test_two_rank_cuda_driver_matches_single_process(tmp_path, cuda_device, mode, strip,
                                                     monkeypatch):
    import torch
    from paper_2407_11272_b200 import _lib as L, device
    from paper_2407_11272_b200.grad import device_loss_grad
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), mode, strip), nprocs=2, join=True)
    out = np.load(tmp_path / f"out_{mode}_{int(strip)}.npz")
    if strip:
        monkeypatch.setattr(device, "STRIP_MIN_NODES", 0)
    v, f, grid, target = _problem()
    dm = device.DeviceMesh.from_numpy(v, f)
    sums, g = device_loss_grad(dm, grid, torch.from_numpy(target).cuda(), mode=mode,
                               precision="f32")
    s = sums.cpu().numpy()
    ref = g.cpu().numpy() / s[1]
    assert abs(float(out["loss"]) - s[4]) <= 1e-9 * abs(s[4])
    assert np.abs(out["grads"] - ref).max() <= 1e-9 * np.abs(ref).max()
    assert int(out["excl"]) == int(s[2])
    vals, flags = device.forward(dm, mode, "f32", grid=grid, policy=L.POLICY_HALF)
    assert np.abs(out["vals"] - vals.cpu().numpy()).max() <= 1e-6
    assert np.array_equal(out["flags"], flags.cpu().numpy())


def _mc_field():
    """A winding-number field with several components (two tori) on a grid
    whose i-extent does not split evenly over 3 ranks."""
    from paper_2407_11272_b200 import configs
    v1, f1 = configs.torus(0.55, 0.25, 40, 20)
    v2, f2 = configs.torus(0.3, 0.12, 30, 14)
    v = np.concatenate([v1, v2 * [1, 1, 1] + [0.1, 0.0, 0.3]])
    f = np.concatenate([f1, f2 + len(v1)])
    return v, f, ((-1.0,) * 3, (1.0,) * 3, (29, 24, 32))


def _mc_worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2407_11272_b200 import _lib as L, device
    from paper_2407_11272_b200.recon import slab_marching_cubes
    v, f, grid = _mc_field()
    rx, ry, rz = grid[2]
    per = -(-rx // world)
    i0, i1 = min(rx, rank * per), min(rx, (rank + 1) * per)
    dm = device.DeviceMesh.from_numpy(v, f)
    vals, _ = device.forward(dm, "exact", "f32", grid=grid, n0=i0 * ry * rz,
                             count=(i1 - i0) * ry * rz, policy=L.POLICY_HALF)
    mv, mf = slab_marching_cubes(vals, grid, i0, 0.5, rank=rank, world=world)
    if rank == 0:
        np.savez(os.path.join(outdir, f"mc_{world}.npz"), v=mv.cpu().numpy(), f=mf.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_marching_cubes_matches_single_gpu(tmp_path, cuda_device, world):
    """Slab-sharded marching cubes (1-row halo from the next rank, global
    vertex ids from all-gathered per-axis counts) over 2 and 3 ranks (29
    i-rows: uneven slabs) gives the one-GPU mesh bit for bit -- which is the
    reference's marching_cubes output (test_mc.py)."""
    from paper_2407_11272_b200 import _lib as L, device
    from paper_2407_11272_b200.recon import marching_cubes_device
    mp.spawn(_mc_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    out = np.load(tmp_path / f"mc_{world}.npz")
    v, f, grid = _mc_field()
    dm = device.DeviceMesh.from_numpy(v, f)
    vals, _ = device.forward(dm, "exact", "f32", grid=grid, policy=L.POLICY_HALF)
    rv, rf = marching_cubes_device(vals, grid, 0.5)
    assert rf.shape[0] > 1000
    assert out["v"].tobytes() == rv.cpu().numpy().tobytes()
    assert np.array_equal(out["f"], rf.cpu().numpy())
