"""Multi-process (gloo, world sizes 2 and 3, CPU) test of the slab-sharded driver.

The driver's sharding, all-gather and single packed all-reduce are the
product code; the per-slab compute is injected as an oracle evaluator
(CPU, f64) so the N>1 logic runs without a GPU.  The reduced loss and
gradient must equal the single-process reference computation (grad.py:71-127
restated by the oracle) to rounding.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import golden, grid_of


class OracleEvaluator:
    def __init__(self, vertices, faces, grid, mode="soft"):
        from oracle import oracle as orc
        self.orc = orc
        self.v, self.f = vertices, faces
        self.pts = orc.node_coordinates(*grid)
        self.mode = mode

    def forward(self, n0, count, policy):
        vals, flags = self.orc.winding_number_batch(self.v, self.f, self.pts[n0:n0 + count],
                                                    mode=self.mode, threads=1)
        if policy == 1:
            vals = np.where(flags, 0.5, vals)
        return torch.from_numpy(vals), torch.from_numpy(flags.astype(np.uint8))

    def loss_grad_partial(self, n0, count, targets, weights=None):
        pts = self.pts[n0:n0 + count]
        vals, flags = self.orc.winding_number_batch(self.v, self.f, pts, mode=self.mode,
                                                    threads=1)
        t = np.asarray(targets, dtype=np.float64)
        w = np.ones(count) if weights is None else np.asarray(weights, dtype=np.float64)
        r = np.where(flags, 0.0, vals - t)
        sums = torch.tensor([float((w * r * r).sum()), float(w[~flags].sum()),
                             float(flags.sum())], dtype=torch.float64)
        coefs = 2.0 * w * r
        gfn = self.orc.soft_grad if self.mode == "soft" else self.orc.exact_grad
        g = gfn(self.v, self.f, pts, coefs, threads=1)
        return sums, torch.from_numpy(g)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2407_11272_b200.distributed import SlabDriver
    g = golden("loss_grad")
    grid = grid_of(g)
    ev = OracleEvaluator(g["vertices"], g["faces"], grid)
    n_total = int(np.prod(grid[2]))
    drv = SlabDriver(ev, n_total, rank, world)
    n0, cnt = drv.slab
    loss, grads, excl, _ = drv.loss_grad(g["target"][n0:n0 + cnt])
    vals, flags = drv.forward(policy=1, gather=True)
    if rank == 0:
        np.savez(os.path.join(outdir, "out.npz"), loss=float(loss), grads=grads.numpy(),
                 excl=float(excl), vals=vals.numpy(), flags=flags.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_slab_ranges_cover_grid():
    from paper_2407_11272_b200.distributed import slab_range
    for n in (1, 7, 64, 4096, 32 ** 3):
        for world in (1, 2, 3, 4, 8):
            spans = [slab_range(n, r, world) for r in range(world)]
            covered = np.zeros(n, int)
            for n0, c in spans:
                covered[n0:n0 + c] += 1
            assert (covered == 1).all()


@pytest.mark.parametrize("world", [2, 3])
def test_multi_rank_loss_grad_matches_single_process(tmp_path, world):
    """world 2: equal slabs; world 3: uneven slabs (the node count is not a
    multiple of 3)."""
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    out = np.load(tmp_path / "out.npz")
    from oracle import oracle as orc
    g = golden("loss_grad")
    grid = grid_of(g)
    pts = orc.node_coordinates(*grid)
    loss, grads, excl = orc.occupancy_loss_grad(g["vertices"], g["faces"], pts, g["target"])
    assert abs(float(out["loss"]) - loss) <= 1e-14 * abs(loss)
    assert np.abs(out["grads"] - grads).max() <= 1e-12 * np.abs(grads).max()
    assert int(out["excl"]) == excl
    vals, flags = orc.voxelize(g["vertices"], g["faces"], pts, mode="soft")
    assert np.array_equal(out["vals"], vals)
    assert np.array_equal(out["flags"].astype(bool), flags)


def _worker_io(rank, world, port, outdir):
    """gather_and_save of a slab-sharded forward, and the all-excluded loss."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2407_11272_b200.distributed import SlabDriver
    from paper_2407_11272_b200.fieldio import gather_and_save
    from paper_2407_11272_b200.types import GridSpec
    g = golden("loss_grad")
    grid = grid_of(g)
    ev = OracleEvaluator(g["vertices"], g["faces"], grid)
    n_total = int(np.prod(grid[2]))
    drv = SlabDriver(ev, n_total, rank, world)
    gather_and_save(drv, GridSpec(grid[0], grid[1], grid[2]), os.path.join(outdir, "g.wvox"))
    n0, cnt = drv.slab
    raised = 0
    try:  # every node zero-weighted: the reference's ValueError on every rank
        drv.loss_grad(g["target"][n0:n0 + cnt], np.zeros(cnt))
    except ValueError as e:
        raised = int("no usable grid nodes" in str(e))
    flag = torch.tensor([raised], dtype=torch.int64)
    dist.all_reduce(flag)
    if rank == 0:
        np.savez(os.path.join(outdir, "io.npz"), raised=int(flag))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_and_save_and_empty_weights_world2(tmp_path):
    """fieldio.gather_and_save over two ranks writes the same WVOX1 bytes as
    save_field of the single-process grid (reference winding.py:396-443), and
    a loss with every node zero-weighted raises the reference's ValueError
    (grad.py:108-109) on both ranks instead of returning NaN."""
    port = _free_port()
    mp.spawn(_worker_io, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    from oracle import oracle as orc
    from paper_2407_11272_b200.fieldio import load_field, save_field
    from paper_2407_11272_b200.types import GridSpec, ScalarField
    g = golden("loss_grad")
    grid = grid_of(g)
    vals, _ = orc.voxelize(g["vertices"], g["faces"], orc.node_coordinates(*grid), mode="soft")
    save_field(ScalarField(GridSpec(grid[0], grid[1], grid[2]), vals), tmp_path / "ref.wvox")
    assert (tmp_path / "g.wvox").read_bytes() == (tmp_path / "ref.wvox").read_bytes()
    assert np.array_equal(load_field(tmp_path / "g.wvox").values, vals)
    assert int(np.load(tmp_path / "io.npz")["raised"]) == 2
