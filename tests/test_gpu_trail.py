"""Exact backward over edge trails (wv_trail.cu + ExactEdgeBwdTrail): the
same vertex gradients as the single-face kernel up to fp32 summation order,
and within north_star's 1e-4 (of the largest component) of the f64 oracle
on the same f32-rounded inputs, with coefficients at every unflagged node:
soups, index-welded meshes with holes, random non-manifold meshes with
degenerate / duplicated faces, broken welds (the trails are rebuilt), a
closed mesh (no window at all), a single triangle, and C3's full 256^3
lattice with the bench's split plan."""

import numpy as np
import pytest

from oracle import oracle as orc
from test_gpu_fuzz import r32, random_case

pytestmark = pytest.mark.gpu


def _grad(dm, coefs, grid, **kw):
    import torch
    from paper_2407_11272_b200 import device
    c = torch.from_numpy(np.asarray(coefs)).float().cuda()
    fg = device.face_grad(dm, "exact", "f32", c, grid=grid, **kw)
    return device.vertex_grad(dm, fg).cpu().numpy()


def _coefs(dm, grid, seed):
    from paper_2407_11272_b200 import device
    _, flags = device.forward(dm, "exact", "f32", grid=grid)
    n = int(flags.numel())
    c = np.random.default_rng(seed).normal(size=n)
    c[flags.cpu().numpy().astype(bool)] = 0.0
    return r32(c)


@pytest.mark.parametrize("kind", ["soup", "holes", "broken"])
def test_trail_backward_matches_single_and_oracle(cuda_device, kind):
    import torch
    from paper_2407_11272_b200 import configs, device
    if kind == "holes":
        v, f = configs.torus_with_holes(40, 30, holes=3, patch=4, seed=1)
    else:
        v, f = configs.soup(*configs.torus(0.7, 0.3, 60, 40), seed=1)
    grid = ((-1.0,) * 3, (1.0,) * 3, (24, 20, 64))
    dm = device.DeviceMesh.from_numpy(v, f)
    if kind == "broken":
        dm.exact_trail_setup()
        v2 = v.copy()
        rng = np.random.default_rng(2)
        moved = rng.random(len(v)) < 0.3
        v2[moved] += rng.normal(scale=1e-3, size=(int(moved.sum()), 3))
        dm.set_vertices(torch.from_numpy(v2).to(dm.vertices.device))
        assert getattr(dm, "_exact_trail", None) is None  # welds split: rebuilt on use
        v = v2
    c = _coefs(dm, grid, 3)
    a = _grad(dm, c, grid, trails=False, pairs=False)
    b = _grad(dm, c, grid, trails=True)
    scale = np.abs(a).max()
    assert scale > 0 and np.isfinite(b).all()
    assert np.abs(a - b).max() <= 2e-4 * scale, (kind, np.abs(a - b).max() / scale)
    p32 = r32(orc.node_coordinates(*grid))
    sel = np.random.default_rng(5).choice(len(v), min(len(v), 300), replace=False)
    r = orc.exact_grad(r32(v), f, p32, c)[sel]
    err = np.abs(b[sel] - r).max() / np.abs(r).max()
    print(kind, "trail vs oracle", err)
    assert err <= 1e-4


@pytest.mark.parametrize("seed", range(12))
def test_trail_backward_random_meshes(cuda_device, seed):
    """Random meshes (degenerate / duplicated faces, scales 1e-2..1e2): the
    trail backward within 1e-4 of the f64 oracle at every vertex, near-surface
    nodes included (their ill-conditioned pairs take the fp64 path)."""
    from paper_2407_11272_b200 import device
    v, f, _ = random_case(seed)
    scale = float(np.abs(v).max())
    grid = ((-1.1 * scale,) * 3, (1.1 * scale,) * 3, (10, 12, 32))
    p32 = r32(orc.node_coordinates(*grid))
    _, fl = orc.winding_number_batch(r32(v), f, p32, mode="exact", threads=1)
    c = np.random.default_rng(200 + seed).normal(size=len(p32))
    c32 = np.where(fl, 0.0, r32(c))
    dm = device.DeviceMesh.from_numpy(v, f)
    g = _grad(dm, c32, grid, trails=True)
    r = orc.exact_grad(r32(v), f, p32, c32, threads=1)
    assert np.isfinite(g).all()
    assert np.abs(g - r).max() <= 1e-4 * max(np.abs(r).max(), 1e-300), seed


def test_trail_backward_closed_and_tiny_meshes(cuda_device):
    from paper_2407_11272_b200 import configs, device
    grid = ((-1.0,) * 3, (1.0,) * 3, (6, 6, 16))
    n = 6 * 6 * 16
    v, f = configs.icosphere(2)
    dm = device.DeviceMesh.from_numpy(v, f)
    g = _grad(dm, np.ones(n), grid, trails=True)
    assert dm.exact_trail_setup()[2] == 0 and np.abs(g).max() == 0.0
    v1 = np.array([[0.1, 0.2, 0.05], [0.8, -0.1, 0.1], [0.2, 0.7, -0.2]])
    f1 = np.array([[0, 1, 2]])
    dm = device.DeviceMesh.from_numpy(v1, f1)
    c = _coefs(dm, grid, 0)
    p32 = r32(orc.node_coordinates(*grid))
    g = _grad(dm, c, grid, trails=True)
    r = orc.exact_grad(r32(v1), f1, p32, c, threads=1)
    assert dm.exact_trail_setup()[2] == 1
    assert np.abs(g - r).max() <= 1e-4 * np.abs(r).max()
    # sub-range of the lattice (n0 even, whole rows and a partial one)
    g2 = _grad(dm, c[32:32 + 200], grid, n0=32, count=200, trails=True)
    r2 = orc.exact_grad(r32(v1), f1, p32[32:232], c[32:232], threads=1)
    assert np.abs(g2 - r2).max() <= 1e-4 * np.abs(r2).max()


def test_trail_backward_rejects_unaligned(cuda_device):
    from paper_2407_11272_b200 import configs, device
    v, f = configs.soup(*configs.torus(0.7, 0.3, 12, 8), seed=1)
    dm = device.DeviceMesh.from_numpy(v, f)
    with pytest.raises(ValueError):
        _grad(dm, np.ones(6 * 6 * 15), ((-1.0,) * 3, (1.0,) * 3, (6, 6, 15)), trails=True)


def test_trail_backward_c3_full_lattice(cuda_device):
    """C3 at full size through the automatic choice (which takes the trails):
    against the single-face backward with the occupancy loss's coefficients
    at every node (both fp32; each is checked against the oracle on row
    subsets in test_gpu_error_report.py)."""
    from paper_2407_11272_b200 import configs, device
    w = configs.make("c3")
    grid = (w.lo, w.hi, w.res)
    dm = device.DeviceMesh.from_numpy(w.vertices, w.faces)
    assert device.backward_path(dm, "exact", "f32", grid, 0, w.n_nodes) == "trails"
    vals, flags = device.forward(dm, "exact", "f32", grid=grid)
    tm = device.DeviceMesh.from_numpy(w.vertices * 1.03, w.faces)
    tv, _ = device.forward(tm, "exact", "f32", grid=grid)
    coefs, _ = device.loss_terms(vals, flags, (tv > 0.5).float())
    out = []
    for kw in ({"pairs": False}, {}):
        fg = device.face_grad(dm, "exact", "f32", coefs, grid=grid, **kw)
        out.append(device.vertex_grad(dm, fg).cpu().numpy())
    a, b = out
    scale = np.abs(a).max()
    err = np.abs(a - b).max() / scale
    print("C3 full lattice: trail vs single-face backward, max |dg| / max |g| =", err)
    assert scale > 0 and np.isfinite(b).all() and err <= 1e-4, err


@pytest.mark.parametrize("kind", ["soup", "holes", "random"])
def test_trail_backward_f64(cuda_device, kind):
    """The f64 parity path over the same trails (ExactTrail64): equal to the
    f64 single-face backward and to the oracle to f64 rounding (1e-10 of the
    largest component), on a lattice range and on a point list."""
    import torch
    from paper_2407_11272_b200 import configs, device
    if kind == "holes":
        v, f = configs.torus_with_holes(30, 20, holes=3, patch=3, seed=1)
    elif kind == "soup":
        v, f = configs.soup(*configs.torus(0.7, 0.3, 30, 20), seed=1)
    else:
        v, f, _ = random_case(3)
    s = float(np.abs(v).max())
    grid = ((-1.1 * s,) * 3, (1.1 * s,) * 3, (12, 10, 17))  # odd rows: no row kernel needed
    dm = device.DeviceMesh.from_numpy(v, f)
    p = orc.node_coordinates(*grid)
    _, fl = orc.winding_number_batch(v, f, p, mode="exact", threads=1)
    c = np.random.default_rng(4).normal(size=len(p))
    c[fl] = 0.0
    ct = torch.from_numpy(c).cuda()
    out = []
    for kw in ({"trails": False, "pairs": False}, {"trails": True}):
        fg = device.face_grad(dm, "exact", "f64", ct, grid=grid, **kw)
        out.append(device.vertex_grad(dm, fg).cpu().numpy())
    a, b = out
    r = orc.exact_grad(v, f, p, c, threads=1)
    scale = max(np.abs(r).max(), 1e-300)
    assert np.abs(a - b).max() <= 1e-10 * scale
    assert np.abs(b - r).max() <= 1e-9 * scale, np.abs(b - r).max() / scale
    sel = np.random.default_rng(6).choice(len(p), 500, replace=False)
    fg = device.face_grad(dm, "exact", "f64", ct[sel], points=torch.from_numpy(p[sel]).cuda(),
                          trails=True)
    g = device.vertex_grad(dm, fg).cpu().numpy()
    r2 = orc.exact_grad(v, f, p[sel], c[sel], threads=1)
    assert np.abs(g - r2).max() <= 1e-9 * max(np.abs(r2).max(), 1e-300)
