"""Strip-ordered exact forward (wv_strip.cu + ExactStripPol): the same
winding numbers as the face-ordered kernel up to fp32 summation order, and
within the north_star 1e-5 of the f64 oracle, on welded meshes, shuffled
soups (welded by position), random meshes with degenerate / duplicated faces
(lattice-aligned vertices for the on-vertex flags) and soups whose welds were
broken after the strip order was built (the packer restarts the strip)."""

import numpy as np
import pytest

from oracle import oracle as orc
from test_gpu_fuzz import r32, random_case

pytestmark = pytest.mark.gpu


def _dist_to_faces(p, tri):
    """Distance from one point to a set of triangles (vectorised over faces)."""
    a, b, c = tri[:, 0], tri[:, 1], tri[:, 2]
    best = np.minimum(np.minimum(np.linalg.norm(p - a, axis=1), np.linalg.norm(p - b, axis=1)),
                      np.linalg.norm(p - c, axis=1))
    for p0, p1 in ((a, b), (b, c), (c, a)):
        e = p1 - p0
        ee = np.maximum((e * e).sum(1), 1e-300)
        t = np.clip(((p - p0) * e).sum(1) / ee, 0.0, 1.0)
        best = np.minimum(best, np.linalg.norm(p - (p0 + t[:, None] * e), axis=1))
    n = np.cross(b - a, c - a)
    nn = np.sqrt((n * n).sum(1))
    ok = nn > 0
    nh = n[ok] / nn[ok, None]
    dist = ((p - a[ok]) * nh).sum(1)
    proj = p - dist[:, None] * nh
    ab, ac, v2 = b[ok] - a[ok], c[ok] - a[ok], proj - a[ok]
    d00, d01, d11 = (ab * ab).sum(1), (ab * ac).sum(1), (ac * ac).sum(1)
    d20, d21 = (v2 * ab).sum(1), (v2 * ac).sum(1)
    den = d00 * d11 - d01 * d01
    bv = (d11 * d20 - d01 * d21) / den
    bw = (d00 * d21 - d01 * d20) / den
    inside = (bv >= 0) & (bw >= 0) & (bv + bw <= 1)
    if inside.any():
        best = min(best.min(), np.abs(dist[inside]).min())
    return float(np.min(best))


def _both(dm, grid, **kw):
    from paper_2407_11272_b200 import _lib as L, device
    a, fa = device.forward(dm, "exact", "f32", grid=grid, policy=L.POLICY_RAW, strip=False, **kw)
    b, fb = device.forward(dm, "exact", "f32", grid=grid, policy=L.POLICY_RAW, strip=True, **kw)
    return (a.double().cpu().numpy(), fa.cpu().numpy().astype(bool),
            b.double().cpu().numpy(), fb.cpu().numpy().astype(bool))


@pytest.mark.parametrize("kind", ["welded", "soup"])
def test_strip_matches_face_order(cuda_device, kind):
    from paper_2407_11272_b200 import configs, device
    v, f = configs.torus(0.7, 0.3, 60, 40)
    if kind == "soup":
        v, f = configs.soup(v, f, seed=1)
    grid = ((-1.0,) * 3, (1.0,) * 3, (24, 20, 64))
    dm = device.DeviceMesh.from_numpy(v, f)
    a, fa, b, fb = _both(dm, grid)
    assert np.array_equal(fa, fb)
    assert np.abs(a - b)[~fa].max() <= 2e-6
    # sub-ranges (splits start at tile boundaries, strips restart there)
    a2, _, b2, _ = _both(dm, grid, n0=64 * 40, count=64 * 24)
    assert np.abs(a2 - b2).max() <= 2e-6 and np.abs(b2 - b[64 * 40:64 * 64]).max() <= 2e-6
    nodes = orc.node_coordinates(*grid)
    p32 = nodes.astype(np.float32).astype(np.float64)
    sel = np.random.default_rng(0).choice(len(nodes), 3000, replace=False)
    ref, rf = orc.winding_number_batch(r32(v), f, p32[sel], mode="exact")
    assert np.array_equal(rf, fb[sel])
    assert np.abs(ref - b[sel])[~rf].max() <= 1e-5


@pytest.mark.parametrize("seed", range(12))
def test_strip_random_meshes_lattice(cuda_device, seed):
    from paper_2407_11272_b200 import device
    v, f, pts = random_case(seed)
    scale = float(np.abs(v).max())
    res = (10, 12, 32)
    lo, hi = (-1.1 * scale,) * 3, (1.1 * scale,) * 3
    if seed % 3 == 0:  # lattice-aligned vertices: on-vertex nodes
        ax = [orc.axis_nodes(lo[a], hi[a], res[a]) for a in range(3)]
        v = np.stack([ax[a][np.abs(ax[a][None, :] - v[:, a:a + 1]).argmin(axis=1)]
                      for a in range(3)], axis=1)
    grid = (lo, hi, res)
    p32 = orc.node_coordinates(*grid).astype(np.float32).astype(np.float64)
    dm = device.DeviceMesh.from_numpy(v, f)
    a, fa, b, fb = _both(dm, grid)
    assert np.array_equal(fa, fb), seed
    ref, rf = orc.winding_number_batch(r32(v), f, p32, mode="exact", threads=1)
    assert np.array_equal(fb, rf), seed
    assert np.abs(b[~rf] - ref[~rf]).max() <= 1e-5, seed
    # the point-list launch of the strip records (generic face path)
    got, gf = device.forward(dm, "exact", "f32", points=pts, strip=True)
    ref, rf = orc.winding_number_batch(r32(v), f, r32(pts), mode="exact", threads=1)
    assert np.array_equal(gf.cpu().numpy().astype(bool), rf), seed
    assert np.abs(got.double().cpu().numpy()[~rf] - ref[~rf]).max() <= 1e-5, seed


def test_strip_broken_welds(cuda_device):
    """Strips built on the welded soup, then half of the vertex copies moved
    (as after a morph step of a soup): the packer must restart wherever the
    carried positions differ, and the values must still match."""
    import torch
    from paper_2407_11272_b200 import configs, device
    v, f = configs.soup(*configs.torus(0.7, 0.3, 40, 30), seed=2)
    grid = ((-1.0,) * 3, (1.0,) * 3, (16, 16, 32))
    dm = device.DeviceMesh.from_numpy(v, f)
    dm.strip_setup()
    v2 = v.copy()
    rng = np.random.default_rng(1)
    moved = rng.random(len(v)) < 0.5
    v2[moved] += rng.normal(scale=1e-3, size=(int(moved.sum()), 3))
    dm.set_vertices(torch.from_numpy(v2).to(dm.vertices.device))
    a, fa, b, fb = _both(dm, grid)
    assert np.array_equal(fa, fb)
    assert np.abs(a - b)[~fa].max() <= 2e-6


def test_strip_c3_disagreements_are_within_tolerance(cuda_device):
    """C3 (the headline soup, full 256^3 lattice): wherever the strip and
    face-ordered kernels differ by more than 1e-6, both must be within the
    north_star 1e-5 of the f64 oracle at that node, evaluated on the same
    f32-rounded nodes and vertices (differences come from fp32 rounding near
    the surface: the two orders evaluate alpha from different corners)."""
    from paper_2407_11272_b200 import _lib as L, configs, device
    w = configs.make("c3")
    grid = (w.lo, w.hi, w.res)
    dm = device.DeviceMesh.from_numpy(w.vertices, w.faces)
    a, fa, b, fb = _both(dm, grid)
    assert np.array_equal(fa, fb)
    d = np.abs(a - b)
    d[fa] = 0.0
    idx = np.argsort(d)[::-1][:64]
    idx = idx[d[idx] > 1e-6]
    print("strip vs face order: max", d.max(), "nodes > 1e-6:", int((d > 1e-6).sum()))
    if len(idx) == 0:
        return
    p32 = orc.node_coordinates(*grid)[idx].astype(np.float32).astype(np.float64)
    ref, rf = orc.winding_number_batch(r32(w.vertices), w.faces, p32, mode="exact")
    assert np.array_equal(rf, fa[idx])
    ea, eb = np.abs(a[idx] - ref)[~rf], np.abs(b[idx] - ref)[~rf]
    print("vs oracle: face order", ea.max(initial=0), "strip", eb.max(initial=0))
    assert eb.max(initial=0) <= 1e-5 and ea.max(initial=0) <= 1e-5


def _grads(dm, coefs, **kw):
    import torch
    from paper_2407_11272_b200 import device
    c = torch.from_numpy(coefs).float().cuda()
    out = []
    for pairs in (False, True):
        fg = device.face_grad(dm, "exact", "f32", c, pairs=pairs, **kw)
        out.append(device.vertex_grad(dm, fg).cpu().numpy())
    return out


@pytest.mark.parametrize("kind", ["soup", "holes", "broken"])
def test_pair_backward_matches_single(cuda_device, kind):
    """The strip-pair exact backward (ExactEdgeBwdPair) against the
    single-face kernel: same vertex gradients up to fp32 summation order."""
    import torch
    from paper_2407_11272_b200 import configs, device
    if kind == "holes":
        v, f = configs.torus_with_holes(40, 30, holes=3, patch=4, seed=1)
    else:
        v, f = configs.soup(*configs.torus(0.7, 0.3, 60, 40), seed=1)
    grid = ((-1.0,) * 3, (1.0,) * 3, (24, 20, 64))
    dm = device.DeviceMesh.from_numpy(v, f)
    if kind == "broken":
        dm.exact_pair_setup()
        v2 = v.copy()
        rng = np.random.default_rng(2)
        moved = rng.random(len(v)) < 0.3
        v2[moved] += rng.normal(scale=1e-3, size=(int(moved.sum()), 3))
        dm.set_vertices(torch.from_numpy(v2).to(dm.vertices.device))
        v = v2
    vals, flags = device.forward(dm, "exact", "f32", grid=grid)
    p32 = orc.node_coordinates(*grid).astype(np.float32).astype(np.float64)
    c = np.random.default_rng(3).normal(size=len(p32))
    c[flags.cpu().numpy().astype(bool)] = 0.0
    a, b = _grads(dm, c, grid=grid)
    scale = np.abs(a).max()
    assert scale > 0 and np.isfinite(b).all()
    # both are fp32 evaluations ~1e-5 from the f64 gradient near the surface
    assert np.abs(a - b).max() <= 2e-4 * scale, (kind, np.abs(a - b).max() / scale)
    if kind != "holes":
        sel = np.random.default_rng(5).choice(len(v), 200, replace=False)
        r = orc.exact_grad(r32(v), f, p32, r32(c))[sel]
        assert np.abs(b[sel] - r).max() <= 1e-4 * np.abs(r).max()
    # generic (point-list) launch of the pair records
    sel = np.random.default_rng(4).choice(len(p32), 2000, replace=False)
    a2, b2 = _grads(dm, c[sel], points=torch.from_numpy(p32[sel]).float().cuda())
    assert np.abs(a2 - b2).max() <= 2e-4 * np.abs(a2).max()


def test_pair_backward_c3_full_lattice(cuda_device):
    """C3 (100k-face soup, the full 256^3 lattice, the bench's split plan):
    the strip-pair backward against the single-face backward with the
    occupancy loss's own coefficients (2 (W - target), 0 on flagged nodes) at
    every node.  Both are fp32 evaluations of the same sum in different
    orders (each is checked against the f64 oracle on row subsets in
    test_gpu_error_report.py; a full-lattice oracle gradient is 1.7e12
    pairs)."""
    import torch
    from paper_2407_11272_b200 import configs, device
    w = configs.make("c3")
    grid = (w.lo, w.hi, w.res)
    dm = device.DeviceMesh.from_numpy(w.vertices, w.faces)
    vals, flags = device.forward(dm, "exact", "f32", grid=grid)
    tm = device.DeviceMesh.from_numpy(w.vertices * 1.03, w.faces)
    tv, _ = device.forward(tm, "exact", "f32", grid=grid)
    coefs, _ = device.loss_terms(vals, flags, (tv > 0.5).float())
    out = []
    for pairs in (False, True):
        fg = device.face_grad(dm, "exact", "f32", coefs, grid=grid, pairs=pairs)
        out.append(device.vertex_grad(dm, fg).cpu().numpy())
    a, b = out
    scale = np.abs(a).max()
    err = np.abs(a - b).max() / scale
    print("C3 full lattice: pair vs single-face backward, max |dg| / max |g| =", err)
    assert scale > 0 and np.isfinite(b).all() and err <= 1e-4, err


@pytest.mark.parametrize("seed", range(12))
def test_pair_backward_random_meshes(cuda_device, seed):
    """Random meshes (degenerate / duplicated faces, several scales) on a
    lattice: pair backward within 1e-4 of the f64 oracle on the same
    f32-rounded inputs, coefficients at every unflagged node (near-surface
    nodes included)."""
    import torch
    from paper_2407_11272_b200 import device
    v, f, _ = random_case(seed)
    scale = float(np.abs(v).max())
    grid = ((-1.1 * scale,) * 3, (1.1 * scale,) * 3, (10, 12, 32))
    p32 = r32(orc.node_coordinates(*grid))
    _, fl = orc.winding_number_batch(r32(v), f, p32, mode="exact", threads=1)
    c = np.random.default_rng(200 + seed).normal(size=len(p32))
    c32 = np.where(fl, 0.0, r32(c))
    dm = device.DeviceMesh.from_numpy(v, f)
    fg = device.face_grad(dm, "exact", "f32", torch.from_numpy(c32).float().cuda(), grid=grid,
                          pairs=True)
    g = device.vertex_grad(dm, fg).cpu().numpy()
    r = orc.exact_grad(r32(v), f, p32, c32, threads=1)
    assert np.isfinite(g).all()
    assert np.abs(g - r).max() <= 1e-4 * max(np.abs(r).max(), 1e-300), seed


def test_pair_backward_closed_mesh_and_tiny_meshes(cuda_device):
    """Edge cases of the strip paths: a closed mesh (no active face: every
    edge cancels), a single triangle (one pair with a zero-weight partner),
    and a strip forward of a one-face mesh."""
    import torch
    from paper_2407_11272_b200 import configs, device
    grid = ((-1.0,) * 3, (1.0,) * 3, (6, 6, 16))
    n = 6 * 6 * 16
    c = torch.ones(n, device="cuda")
    v, f = configs.icosphere(2)
    dm = device.DeviceMesh.from_numpy(v, f)
    fg = device.face_grad(dm, "exact", "f32", c, grid=grid, pairs=True)
    assert fg[0].shape == (0, 3, 3)
    assert float(device.vertex_grad(dm, fg).abs().max()) == 0.0
    v1 = np.array([[0.1, 0.2, 0.05], [0.8, -0.1, 0.1], [0.2, 0.7, -0.2]])
    f1 = np.array([[0, 1, 2]])
    dm = device.DeviceMesh.from_numpy(v1, f1)
    vals, flags = device.forward(dm, "exact", "f32", grid=grid, strip=True)
    p32 = orc.node_coordinates(*grid).astype(np.float32).astype(np.float64)
    ref, rf = orc.winding_number_batch(r32(v1), f1, p32, mode="exact", threads=1)
    assert np.array_equal(flags.cpu().numpy().astype(bool), rf)
    assert np.abs(vals.double().cpu().numpy() - ref)[~rf].max() <= 1e-6
    cc = np.random.default_rng(0).normal(size=n)
    cc[rf] = 0.0
    c32 = cc.astype(np.float32).astype(np.float64)
    g = device.vertex_grad(dm, device.face_grad(dm, "exact", "f32",
                                                torch.from_numpy(c32).float().cuda(),
                                                grid=grid, pairs=True)).cpu().numpy()
    r = orc.exact_grad(r32(v1), f1, p32, c32, threads=1)
    assert np.abs(g - r).max() <= 1e-4 * np.abs(r).max()


@pytest.mark.parametrize("seed", range(8))
def test_f64_strip_forward_matches_reference_order(cuda_device, seed):
    """The f64 parity forward over strip records: every face term is the
    reference's (true-order alpha / beta / on-surface tests), only the order
    of the face sum differs -- agreement with the index-order f64 kernel and
    the oracle to 1e-12, identical flags (random meshes with degenerate and
    duplicated faces; lattice-aligned vertices for on-vertex nodes; both
    atan branches)."""
    from paper_2407_11272_b200 import _lib as L, device
    v, f, pts = random_case(seed)
    scale = float(np.abs(v).max())
    res = (10, 12, 32)
    lo, hi = (-1.1 * scale,) * 3, (1.1 * scale,) * 3
    if seed % 2 == 0:
        ax = [orc.axis_nodes(lo[a], hi[a], res[a]) for a in range(3)]
        v = np.stack([ax[a][np.abs(ax[a][None, :] - v[:, a:a + 1]).argmin(axis=1)]
                      for a in range(3)], axis=1)
    grid = (lo, hi, res)
    dm = device.DeviceMesh.from_numpy(v, f)
    nodes = orc.node_coordinates(*grid)
    for use_atan2 in (True, False):
        a, fa = device.forward(dm, "exact", "f64", grid=grid, policy=L.POLICY_RAW,
                               use_atan2=use_atan2, strip=False)
        b, fb = device.forward(dm, "exact", "f64", grid=grid, policy=L.POLICY_RAW,
                               use_atan2=use_atan2, strip=True)
        a, b = a.cpu().numpy(), b.cpu().numpy()
        assert np.array_equal(fa.cpu().numpy(), fb.cpu().numpy()), seed
        assert np.abs(a - b).max() <= 1e-12 * max(1.0, np.abs(a).max()), seed
        if use_atan2:
            ref, rf = orc.winding_number_batch(v, f, nodes, mode="exact", threads=1)
            assert np.array_equal(fb.cpu().numpy().astype(bool), rf), seed
            assert np.abs(b - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()), seed
    got, gf = device.forward(dm, "exact", "f64", points=pts, strip=True)
    ref, rf = orc.winding_number_batch(v, f, pts, mode="exact", threads=1)
    assert np.array_equal(gf.cpu().numpy().astype(bool), rf)
    assert np.abs(got.cpu().numpy() - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


def test_f64_strip_forward_soup_and_broken_welds(cuda_device):
    import torch
    from paper_2407_11272_b200 import _lib as L, configs, device
    v, f = configs.soup(*configs.torus(0.7, 0.3, 40, 30), seed=2)
    grid = ((-1.0,) * 3, (1.0,) * 3, (16, 16, 32))
    dm = device.DeviceMesh.from_numpy(v, f)
    for step in range(2):
        a, fa = device.forward(dm, "exact", "f64", grid=grid, policy=L.POLICY_HALF, strip=False)
        b, fb = device.forward(dm, "exact", "f64", grid=grid, policy=L.POLICY_HALF, strip=True)
        assert np.array_equal(fa.cpu().numpy(), fb.cpu().numpy())
        assert float((a - b).abs().max()) <= 1e-12
        v2 = v.copy()  # break half of the welds after the strips were built
        rng = np.random.default_rng(1)
        moved = rng.random(len(v)) < 0.5
        v2[moved] += rng.normal(scale=1e-3, size=(int(moved.sum()), 3))
        dm.set_vertices(torch.from_numpy(v2).to(dm.vertices.device))
