"""Warp-row forward kernels (RowSrcW, wv_fwd.cuh): when every warp's 256
nodes lie in one k-row, each face's row terms are computed once per warp
into a shared table instead of in every lane.  Same formula, same inputs:
the per-face terms must be bitwise those of the per-lane row kernel
(RowSrc) on the same nodes (the sums to an f32 ulp: the launches' split
plans differ), for the strip forward and
the face-ordered pair forward, and within 1e-5 of the oracle."""

import numpy as np
import pytest

from oracle import oracle as orc
from test_gpu_fuzz import r32

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("strip", [True, False])
def test_warp_rows_match_lane_rows_bitwise(cuda_device, strip):
    from paper_2407_11272_b200 import _lib as L, configs, device
    if strip:
        v, f = configs.soup(*configs.torus(0.7, 0.3, 40, 30), seed=2)
    else:
        w = configs.make("c3r")
        v, f = w.vertices[: 3 * 3000], np.arange(9000).reshape(-1, 3)
    grid = ((-1.0,) * 3, (1.0,) * 3, (3, 4, 256))
    dm = device.DeviceMesh.from_numpy(v, f)
    kw = dict(grid=grid, policy=L.POLICY_RAW, strip=strip)
    # warp rows: start and count multiples of 256
    a, fa = device.forward(dm, "exact", "f32", n0=256, count=2048, **kw)
    # lane rows over a superset shifted by 8 nodes (start not a multiple of 256)
    b, fb = device.forward(dm, "exact", "f32", n0=248, count=2064, **kw)
    a, b = a.cpu().numpy(), b.cpu().numpy()[8:8 + 2048]
    assert np.array_equal(fa.cpu().numpy(), fb.cpu().numpy()[8:8 + 2048])
    # (the two launches' face-split plans differ, so fp64 tile partials may
    # group differently: allow an f32 ulp, require nearly all bitwise equal)
    assert np.abs(a - b).max() <= 2.4e-7
    assert np.mean(a.view(np.uint32) == b.view(np.uint32)) > 0.99
    p32 = r32(orc.node_coordinates(*grid))[256:256 + 2048]
    ref, rf = orc.winding_number_batch(r32(v), f, p32, mode="exact", threads=1)
    assert np.array_equal(rf, fa.cpu().numpy().astype(bool))
    assert np.abs(a - ref)[~rf].max() <= 1e-5


def test_f64_strip_grid_equals_points_bitwise(cuda_device):
    """The f64 strip forward on a lattice range equals the same kernel on
    the same nodes given as a point list BIT FOR BIT, flags included (the
    node expression is the reference's, winding.py:118-140) -- on a welded
    soup and a random mesh with on-surface nodes."""
    import torch
    from paper_2407_11272_b200 import _lib as L, configs, device
    from test_gpu_fuzz import random_case
    cases = [configs.soup(*configs.torus(0.7, 0.3, 30, 20), seed=3), random_case(5)[:2]]
    for v, f in cases:
        s = float(np.abs(v).max())
        grid = ((-1.1 * s,) * 3, (1.1 * s,) * 3, (6, 5, 24))
        dm = device.DeviceMesh.from_numpy(v, f)
        a, fa = device.forward(dm, "exact", "f64", grid=grid, policy=L.POLICY_RAW, strip=True)
        pts = torch.from_numpy(orc.node_coordinates(*grid)).cuda()
        b, fb = device.forward(dm, "exact", "f64", points=pts, policy=L.POLICY_RAW, strip=True)
        assert np.array_equal(fa.cpu().numpy(), fb.cpu().numpy())
        a, b = a.cpu().numpy(), b.cpu().numpy()
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
