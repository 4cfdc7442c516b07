"""Parity at the full BASELINE configs on seeded node subsets:
C3 (100k-face shuffled soup, 256^3) and its stress variant C3r (100k random
triangles: nothing welds, the face-ordered kernels run) forward + exact
backward, C5 (1M-face torus, 512^3) forward.  The oracle is the bit-exact C
port of the reference kernels (multi-threaded), evaluated on the same
f32-rounded nodes and vertices the FP32 kernels see."""

import numpy as np
import pytest

from oracle import oracle as orc
from test_gpu_fuzz import r32

pytestmark = pytest.mark.gpu


def _subset(w, n, seed):
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(w.n_nodes, size=n, replace=False))
    i, rem = np.divmod(idx, w.res[1] * w.res[2])
    j, k = np.divmod(rem, w.res[2])
    ax = [orc.axis_nodes(w.lo[a], w.hi[a], w.res[a]) for a in range(3)]
    return idx, np.stack([ax[0][i], ax[1][j], ax[2][k]], axis=1)


def _check_forward(w, n, seed):
    import torch
    from paper_2407_11272_b200 import device
    idx, pts = _subset(w, n, seed)
    dm = device.DeviceMesh.from_numpy(w.vertices, w.faces)
    got, gf = device.forward(dm, "exact", "f32", points=torch.as_tensor(pts, dtype=torch.float32))
    got = got.double().cpu().numpy()
    gf = gf.cpu().numpy().astype(bool)
    ref, rf = orc.winding_number_batch(r32(w.vertices), w.faces, r32(pts))
    assert np.array_equal(gf, rf)
    err = np.abs(got - ref)[~rf]
    assert err.max() <= 1e-5, err.max()
    amb = np.abs(ref - 0.5) < 1e-3
    assert np.array_equal((got > 0.5)[~amb], (ref > 0.5)[~amb])
    return dm, pts, ref


@pytest.mark.parametrize("name", ["c3", "c3r"])
def test_c3_soup_forward_and_exact_backward_subset(cuda_device, name):
    import torch
    from paper_2407_11272_b200 import configs, device
    w = configs.make(name)
    dm, pts, ref = _check_forward(w, 1024, 3)
    coefs = np.random.default_rng(4).normal(size=len(pts))
    pts32 = r32(pts)
    coefs[orc.winding_number_batch(r32(w.vertices), w.faces, pts32)[1]] = 0.0
    fg = device.face_grad(dm, "exact", "f32", torch.as_tensor(coefs, dtype=torch.float32),
                          points=torch.as_tensor(pts, dtype=torch.float32))
    got = device.vertex_grad(dm, fg).cpu().numpy()
    gref = orc.exact_grad(r32(w.vertices), w.faces, pts32, r32(coefs), chunk=64)
    assert np.abs(got - gref).max() <= 1e-4 * np.abs(gref).max()


def test_c3_grid_slab_matches_point_path(cuda_device):
    """The lattice kernel (node ranges, as the bench and driver use it) equals
    the point-list kernel on the same nodes."""
    import torch
    from paper_2407_11272_b200 import configs, device
    w = configs.make("c3")
    dm = device.DeviceMesh.from_numpy(w.vertices, w.faces)
    n0 = 128 * 256 * 256 + 77 * 256  # an i-slab interior range through the torus
    cnt = 2048
    gv, gfl = device.forward(dm, "exact", "f32", grid=(w.lo, w.hi, w.res), n0=n0, count=cnt)
    idx = np.arange(n0, n0 + cnt)
    i, rem = np.divmod(idx, w.res[1] * w.res[2])
    j, k = np.divmod(rem, w.res[2])
    ax = [orc.axis_nodes(w.lo[a], w.hi[a], w.res[a]) for a in range(3)]
    pts = np.stack([ax[0][i], ax[1][j], ax[2][k]], axis=1)
    pv, pfl = device.forward(dm, "exact", "f32", points=torch.as_tensor(pts, dtype=torch.float32))
    assert torch.equal(gfl, pfl)
    assert (gv - pv).abs().max().item() <= 1e-6
    ref, rf = orc.winding_number_batch(r32(w.vertices), w.faces, r32(pts))
    assert np.abs(gv.double().cpu().numpy() - ref)[~rf].max() <= 1e-5


def test_c5_million_faces_forward_subset(cuda_device):
    from paper_2407_11272_b200 import configs
    w = configs.make("c5")
    assert w.n_faces == 1_000_000
    _check_forward(w, 192, 5)


def test_c3r_lattice_rows_auto_path(cuda_device):
    """C3r through the bench's automatic path choice on a full-lattice slab
    (the face-ordered row kernels: no strips form on a random soup), checked
    on whole k-rows inside it: forward values at every unflagged node within
    1e-5 of the oracle, flags identical; the exact backward of one of those
    row ranges within 1e-4 of the oracle's gradient."""
    import torch
    from paper_2407_11272_b200 import configs, device
    w = configs.make("c3r")
    rz = w.res[2]
    grid = (w.lo, w.hi, w.res)
    dm = device.DeviceMesh.from_numpy(w.vertices, w.faces)
    n0, cnt = 128 * 256 * 256, 32 * 256 * 256       # 2M nodes: the strip threshold
    assert device.lattice_paths(dm, "exact", "f32", grid, n0, cnt) == (False, False)
    assert device.backward_path(dm, "exact", "f32", grid, n0, cnt) == "faces"
    vals, flags = device.forward(dm, "exact", "f32", grid=grid, n0=n0, count=cnt)
    rows = np.sort(np.random.default_rng(9).choice(cnt // rz, size=8, replace=False))
    idx = (n0 + rows[:, None] * rz + np.arange(rz)[None, :]).reshape(-1)
    i, rem = np.divmod(idx, w.res[1] * w.res[2])
    j, k = np.divmod(rem, w.res[2])
    ax = [orc.axis_nodes(w.lo[a], w.hi[a], w.res[a]) for a in range(3)]
    p32 = r32(np.stack([ax[0][i], ax[1][j], ax[2][k]], axis=1))
    ref, rf = orc.winding_number_batch(r32(w.vertices), w.faces, p32)
    got = vals.double().cpu().numpy()[idx - n0]
    assert np.array_equal(flags.cpu().numpy()[idx - n0].astype(bool), rf)
    assert np.abs(got - ref)[~rf].max() <= 1e-5
    # backward over one 4-row range (coefficients at every unflagged node)
    m0 = n0 + int(rows[0]) * rz
    c = np.random.default_rng(10).normal(size=4 * rz)
    i, rem = np.divmod(np.arange(m0, m0 + 4 * rz), w.res[1] * w.res[2])
    j, k = np.divmod(rem, w.res[2])
    q32 = r32(np.stack([ax[0][i], ax[1][j], ax[2][k]], axis=1))
    _, fl = orc.winding_number_batch(r32(w.vertices), w.faces, q32)
    c32 = np.where(fl, 0.0, r32(c))
    fg = device.face_grad(dm, "exact", "f32", torch.from_numpy(c32).float().cuda(), grid=grid,
                          n0=m0, count=4 * rz)
    g = device.vertex_grad(dm, fg).cpu().numpy()
    gr = orc.exact_grad(r32(w.vertices), w.faces, q32, c32)
    assert np.abs(g - gr).max() <= 1e-4 * np.abs(gr).max()
