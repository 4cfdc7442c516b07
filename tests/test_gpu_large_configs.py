"""Parity at the full BASELINE configs on seeded node subsets:
C3 (100k-face shuffled soup, 256^3) forward + exact backward, C5 (1M-face
torus, 512^3) forward, C2 full 128^3 grid invariants.  The oracle is the
bit-exact C port of the reference kernels (multi-threaded)."""

import numpy as np
import pytest

from oracle import oracle as orc

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
    ref, rf = orc.winding_number_batch(w.vertices, w.faces, pts.astype(np.float32).astype(np.float64))
    assert np.array_equal(gf, rf)
    err = np.abs(got - ref)[~rf]
    assert err.max() <= 1e-5, err.max()
    amb = np.abs(ref - 0.5) < 1e-3
    assert np.array_equal((got > 0.5)[~amb], (ref > 0.5)[~amb])
    return dm, pts, ref


def test_c3_soup_forward_and_exact_backward_subset(cuda_device):
    import torch
    from paper_2407_11272_b200 import configs, device
    w = configs.make("c3")
    dm, pts, ref = _check_forward(w, 1024, 3)
    coefs = np.random.default_rng(4).normal(size=len(pts))
    pts32 = pts.astype(np.float32).astype(np.float64)
    fg = device.face_grad(dm, "exact", "f32", torch.as_tensor(coefs, dtype=torch.float32),
                          points=torch.as_tensor(pts, dtype=torch.float32))
    got = device.vertex_grad(dm, fg).cpu().numpy()
    gref = orc.exact_grad(w.vertices, w.faces, pts32, coefs.astype(np.float32).astype(np.float64),
                          chunk=64)
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
    ref, rf = orc.winding_number_batch(w.vertices, w.faces, pts.astype(np.float32).astype(np.float64))
    assert np.abs(gv.double().cpu().numpy() - ref)[~rf].max() <= 1e-5


def test_c5_million_faces_forward_subset(cuda_device):
    from paper_2407_11272_b200 import configs
    w = configs.make("c5")
    assert w.n_faces == 1_000_000
    _check_forward(w, 192, 5)
