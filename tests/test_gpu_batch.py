"""Batched occupancy loss (C4 path) vs per-mesh calls and the oracle."""

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def test_batch_loss_matches_oracle_per_mesh(cuda_device):
    import torch
    from paper_2407_11272_b200 import configs
    from paper_2407_11272_b200.batch import DeformationNet, batch_occupancy_loss
    meshes = configs.c4_batch(3)
    faces = torch.from_numpy(meshes[0][1]).cuda()
    R = 12
    grid = ((-1.0,) * 3, (1.0,) * 3, (R, R, R))
    rng = np.random.default_rng(0)
    targets = torch.from_numpy(rng.uniform(0, 1, size=(3, R ** 3))).float().cuda()
    verts = torch.stack([torch.from_numpy(m[0]) for m in meshes]).float().cuda()
    verts.requires_grad_(True)
    losses = batch_occupancy_loss(verts, faces, grid, targets)
    losses.sum().backward()
    pts = orc.node_coordinates(*grid)
    import paper_2407_11272_b200 as wv
    spec = wv.GridSpec(*grid)
    for b in range(3):
        # identical to the single-mesh device path (same kernels, same order)
        one = wv.occupancy_loss_grad(wv.TriangleMesh(verts[b].detach().double().cpu().numpy(),
                                                     meshes[b][1]),
                                     wv.ScalarField(spec, targets[b].double().cpu().numpy()),
                                     precision="f32")
        assert abs(float(losses[b]) - one.loss) <= 1e-6 * one.loss
        g = verts.grad[b].double().cpu().numpy()
        assert np.abs(g - one.grads.vectors).max() <= 1e-5 * np.abs(one.grads.vectors).max()
        # and close to the f64 oracle; the soft (dipole) loss of this coarse
        # grid has nodes within ~1e-2 of face centroids (loss ~1e2), where
        # the fp32 rounding of the centroids alone is ~1e-4 relative
        v32 = meshes[b][0].astype(np.float32).astype(np.float64)
        loss, grads, _ = orc.occupancy_loss_grad(v32, meshes[b][1], pts.astype(np.float32)
                                                 .astype(np.float64),
                                                 targets[b].double().cpu().numpy())
        assert abs(float(losses[b]) - loss) <= 2e-3 * loss
        assert np.abs(g - grads).max() <= 2e-3 * np.abs(grads).max()
    # the deformation net trains through it
    torch.manual_seed(0)
    net = DeformationNet(3).cuda()
    opt = torch.optim.Adam(net.parameters(), lr=3e-3)
    ids = torch.arange(3, device="cuda")
    tmpl = verts.detach()
    first = None
    for _ in range(15):
        opt.zero_grad()
        l = batch_occupancy_loss(net(tmpl, ids), faces, grid, targets).mean()
        l.backward()
        opt.step()
        first = float(l) if first is None else first
    assert float(l) < first
