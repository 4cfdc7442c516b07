"""Seeded random parity sweep: random meshes (generic, with degenerate and
duplicated faces, at several coordinate scales) against query points that
include random points, mesh vertices, edge points and face centroids -- the
on-surface cases of _kernels.py:65-88.

* f64 exact / soft vs the oracle (the reference's own arithmetic): values to
  1e-12 (exact) / bitwise (soft), flags identical;
* f32 exact: within 1e-5 of the f64 oracle at EVERY unflagged point, with
  flags identical -- the oracle evaluates the same f32-rounded points and
  vertices the kernel sees (the reference's f32 path rounds both,
  winding.py:362-387), so no exclusion band around the surface is needed --
  and every mesh vertex used as a query point is flagged (an exact hit in
  f32 coordinates).
* f32 gradients (exact and soft): within 1e-4 of the largest component of
  the f64 oracle's, with random coefficients at every unflagged point
  (near-surface points included).
"""

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def r32(a):
    """f32 rounding, back in f64: the inputs the FP32 kernels actually see."""
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def surface_distance(pts, tri):
    """Unsigned distance from each point to the union of triangles (numpy,
    closest point by region tests)."""
    d = np.full(len(pts), np.inf)
    for a, b, c in tri:
        ab, ac = b - a, c - a
        n = np.cross(ab, ac)
        nn = float(n @ n)
        for q0 in range(0, len(pts), 256):
            q = pts[q0:q0 + 256]
            best = np.minimum(np.minimum(np.linalg.norm(q - a, axis=1),
                                         np.linalg.norm(q - b, axis=1)),
                              np.linalg.norm(q - c, axis=1))
            for p0, p1 in ((a, b), (b, c), (c, a)):
                e = p1 - p0
                ee = float(e @ e)
                if ee > 0:
                    t = np.clip(((q - p0) @ e) / ee, 0.0, 1.0)
                    best = np.minimum(best, np.linalg.norm(q - (p0 + t[:, None] * e), axis=1))
            if nn > 0:
                w = q - a
                dist = (w @ n) / np.sqrt(nn)
                proj = q - dist[:, None] * n / np.sqrt(nn)
                # barycentric inside test of the projection
                v2 = proj - a
                d00, d01, d11 = ab @ ab, ab @ ac, ac @ ac
                d20, d21 = v2 @ ab, v2 @ ac
                den = d00 * d11 - d01 * d01
                bv = (d11 * d20 - d01 * d21) / den
                bw = (d00 * d21 - d01 * d20) / den
                inside = (bv >= 0) & (bw >= 0) & (bv + bw <= 1)
                best = np.where(inside, np.minimum(best, np.abs(dist)), best)
            d[q0:q0 + 256] = np.minimum(d[q0:q0 + 256], best)
    return d


def random_case(seed):
    rng = np.random.default_rng(seed)
    scale = 10.0 ** rng.integers(-2, 3)
    nv = int(rng.integers(4, 40))
    v = rng.uniform(-1, 1, size=(nv, 3)) * scale
    nf = int(rng.integers(1, 60))
    f = rng.integers(0, nv, size=(nf, 3))
    f[0] = [0, 1, 1] if nf > 2 else f[0]          # a degenerate face
    if nf > 3:
        f[1] = f[2]                                # a duplicated face
    pts = [rng.uniform(-1.2, 1.2, size=(60, 3)) * scale, v[:5]]
    t = v[f]
    pts.append(t.mean(axis=1)[:10])                # centroids (soft on-centroid, exact on-face)
    pts.append((0.3 * t[:, 0] + 0.7 * t[:, 1])[:10])  # edge points
    return v, f, np.concatenate(pts)


@pytest.mark.parametrize("seed", range(24))
def test_random_meshes_parity(cuda_device, seed):
    import paper_2407_11272_b200 as wv
    v, f, pts = random_case(seed)
    mesh = wv.TriangleMesh(v, f)
    for mode in ("exact", "soft"):
        got, gf = wv.winding_number_batch(mesh, pts, mode=mode, precision="f64")
        ref, rf = orc.winding_number_batch(v, f, pts, mode=mode, threads=1)
        assert np.array_equal(gf, rf), (mode, seed)
        if mode == "soft":
            assert got.tobytes() == ref.tobytes(), seed
        else:
            assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()), seed
    p32 = r32(pts)
    got, gf = wv.winding_number_batch(mesh, pts, mode="exact", precision="f32")
    ref, rf = orc.winding_number_batch(r32(v), f, p32, mode="exact", threads=1)
    assert np.array_equal(gf, rf), seed
    assert (~rf).sum() >= 40
    assert np.abs(got[~rf] - ref[~rf]).max() <= 1e-5, seed
    # query points 60..64 are vertices 0..4: flagged when on a live face
    # (degenerate faces are dropped, winding.py:262-264)
    t = v[f]
    live = np.linalg.norm(np.cross(t[:, 1] - t[:, 0], t[:, 2] - t[:, 0]), axis=1) > 0
    used = np.isin(np.arange(5), f[live])
    assert gf[60:60 + int(min(5, len(v)))][used[:min(5, len(v))]].all(), seed


@pytest.mark.parametrize("seed", range(12))
def test_random_meshes_gradient_parity(cuda_device, seed):
    """Exact and soft f32 backward (generic point path) on the random cases
    vs the f64 oracle on the same f32-rounded inputs, random coefficients at
    every point the mode's forward does not flag (the loss zeroes flagged
    nodes, grad.py:106) -- vertices, edge points and near-surface points
    included -- 1e-4 relative to the largest component (the reference's
    gradient convention)."""
    import torch
    from paper_2407_11272_b200 import device
    v, f, pts = random_case(seed)
    p32, v32 = r32(pts), r32(v)
    c = np.random.default_rng(100 + seed).normal(size=len(pts))
    dm = device.DeviceMesh.from_numpy(v, f)
    for mode, ofn in (("exact", orc.exact_grad), ("soft", orc.soft_grad)):
        _, fl = orc.winding_number_batch(v32, f, p32, mode=mode, threads=1)
        c32 = np.where(fl, 0.0, r32(c))
        fg = device.face_grad(dm, mode, "f32", torch.from_numpy(c32).float().cuda(),
                              points=torch.from_numpy(p32).float().cuda())
        got = device.vertex_grad(dm, fg).cpu().numpy()
        ref = ofn(v32, f, p32, c32, threads=1)
        assert np.isfinite(got).all(), (mode, seed)
        assert np.abs(got - ref).max() <= 1e-4 * max(np.abs(ref).max(), 1e-300), (mode, seed)


@pytest.mark.parametrize("seed", range(12))
def test_random_meshes_lattice_parity(cuda_device, seed):
    """The same random meshes on a lattice (rz = 32: the row kernels, both
    directions) whose nodes include the mesh's own vertices for some seeds
    (a lattice-aligned mesh): forward values at every unflagged node within
    1e-5 of the f64 oracle on the same f32-rounded inputs, flags identical
    (vertex nodes flagged), exact and soft gradients with coefficients at
    every unflagged node within 1e-4 of the oracle."""
    import torch
    from paper_2407_11272_b200 import _lib as L, device
    v, f, _ = random_case(seed)
    scale = float(np.abs(v).max())
    res = (10, 12, 32)
    lo, hi = (-1.1 * scale,) * 3, (1.1 * scale,) * 3
    if seed % 3 == 0:  # snap the vertices onto lattice nodes
        ax = [orc.axis_nodes(lo[a], hi[a], res[a]) for a in range(3)]
        v = np.stack([ax[a][np.abs(ax[a][None, :] - v[:, a:a + 1]).argmin(axis=1)]
                      for a in range(3)], axis=1)
    grid = (lo, hi, res)
    nodes = orc.node_coordinates(*grid)
    p32, v32 = r32(nodes), r32(v)
    dm = device.DeviceMesh.from_numpy(v, f)
    got, gf = device.forward(dm, "exact", "f32", grid=grid, policy=L.POLICY_RAW)
    got, gf = got.cpu().numpy(), gf.cpu().numpy().astype(bool)
    ref, rf = orc.winding_number_batch(v32, f, p32, mode="exact", threads=1)
    assert np.array_equal(gf, rf), seed
    assert np.abs(got[~rf] - ref[~rf]).max() <= 1e-5, seed
    t = v[f]
    live = np.linalg.norm(np.cross(t[:, 1] - t[:, 0], t[:, 2] - t[:, 0]), axis=1) > 0
    on_vertex = np.isin(np.arange(len(v)), f[live])
    idx = {tuple(p): i for i, p in enumerate(p32)}
    for k in np.flatnonzero(on_vertex):
        i = idx.get(tuple(v[k].astype(np.float32).astype(np.float64)))
        if i is not None:
            assert gf[i], (seed, k)
    c = np.random.default_rng(200 + seed).normal(size=len(nodes))
    for mode, ofn in (("exact", orc.exact_grad), ("soft", orc.soft_grad)):
        _, fl = orc.winding_number_batch(v32, f, p32, mode=mode, threads=1)
        c32 = np.where(fl, 0.0, r32(c))
        fg = device.face_grad(dm, mode, "f32", torch.from_numpy(c32).float().cuda(), grid=grid)
        g = device.vertex_grad(dm, fg).cpu().numpy()
        r = ofn(v32, f, p32, c32, threads=1)
        assert np.isfinite(g).all(), (mode, seed)
        assert np.abs(g - r).max() <= 1e-4 * max(np.abs(r).max(), 1e-300), (mode, seed)


@pytest.mark.parametrize("seed", range(8))
def test_random_meshes_f64_gradient_parity(cuda_device, seed):
    """The f64 parity backward (exact edge form and soft, the reference's
    formula) on the random cases: 1e-9 of the largest component (fp64
    rounding and a different summation order than the oracle)."""
    import torch
    from paper_2407_11272_b200 import device
    v, f, pts = random_case(seed)
    scale = np.abs(v).max()
    c = np.random.default_rng(300 + seed).normal(size=len(pts))
    c[surface_distance(pts, v[f]) <= 1e-6 * scale] = 0.0
    cen = v[f].mean(axis=1)
    dm = device.DeviceMesh.from_numpy(v, f)
    for mode, ofn in (("exact", orc.exact_grad), ("soft", orc.soft_grad)):
        cc = c.copy()
        if mode == "soft":
            d = np.linalg.norm(pts[:, None, :] - cen[None], axis=2).min(axis=1)
            cc[d <= 1e-6 * scale] = 0.0
        fg = device.face_grad(dm, mode, "f64", torch.from_numpy(cc).cuda(),
                              points=torch.from_numpy(pts).cuda())
        g = device.vertex_grad(dm, fg).cpu().numpy()
        r = ofn(v, f, pts, cc, threads=1)
        assert np.abs(g - r).max() <= 1e-9 * max(np.abs(r).max(), 1e-300), (mode, seed)
