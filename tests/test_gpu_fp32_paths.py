"""FP32 hot-path parity against the FP64 oracle: soft forward, soft and exact
backward, fused loss, autograd.  Tolerances (north_star / SURVEY 8c):
winding numbers 1e-5 absolute; vertex gradients 1e-4 relative to the
largest component (the reference's own convention, test_grad.py:61,72,164).
"""

import numpy as np
import pytest

from conftest import golden, grid_of
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

G_TOL = 1e-4


@pytest.fixture(scope="module")
def torch_(cuda_device):
    import torch
    return torch


def rel_err(got, ref):
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-300))


@pytest.fixture(scope="module")
def c2():
    from paper_2407_11272_b200 import configs
    return configs.make("c2")


def test_soft_forward_f32_vs_oracle(torch_):
    import paper_2407_11272_b200 as wv
    g = golden("voxelize_icosphere2_r13")
    mesh = wv.TriangleMesh(g["vertices"], g["faces"])
    spec = wv.GridSpec(*grid_of(g))
    got = wv.voxelize(mesh, spec, mode="soft", precision="f32").values.astype(np.float64)
    ref = g["soft_f64"]
    # soft terms grow like 1/r^2 near faces: scale-aware bound
    assert np.abs(got - ref).max() <= 1e-5 * max(1.0, np.abs(ref).max())
    c1 = golden("c1_icosphere3_r32")
    m1 = wv.TriangleMesh(c1["vertices"], c1["faces"])
    s1 = wv.voxelize(m1, wv.GridSpec(*grid_of(c1)), mode="soft", precision="f32").values
    assert np.abs(s1 - c1["soft_f64"]).max() <= 1e-5 * max(1.0, np.abs(c1["soft_f64"]).max())


def test_soft_forward_flags_on_centroid(torch_):
    import paper_2407_11272_b200 as wv
    g = golden("census_cube_r9")
    mesh = wv.TriangleMesh(g["vertices"], g["faces"])
    cen = mesh.vertices[mesh.faces].mean(axis=1)
    pts = np.concatenate([cen[:3], [[3.0, 0.0, 0.0]]])
    # f64 (the reference's default): exact centroids are on-centroid hits
    w, f = wv.winding_number_batch(mesh, pts, mode="soft", precision="f64")
    ref, rf = orc.winding_number_batch(g["vertices"], g["faces"], pts, mode="soft")
    assert np.array_equal(f, rf) and f[:3].all() and not f[3]
    # f32: the kernels see f32-rounded points and corners (winding.py:362-373);
    # with the centroid carried as hi + lo a rounded centroid is ~1e-8 off
    # the true one, i.e. farther than eps = 1e-9 * diag: flags and values as
    # the oracle's on the same rounded inputs
    from test_gpu_fuzz import r32
    w, f = wv.winding_number_batch(mesh, pts, mode="soft", precision="f32")
    ref, rf = orc.winding_number_batch(r32(g["vertices"]), g["faces"], r32(pts), mode="soft")
    assert np.array_equal(f, rf)
    assert np.abs(w[~rf] - ref[~rf]).max() <= 1e-5 * np.abs(ref[~rf]).max()
    # a point that IS the centroid in f32 arithmetic (a dyadic triangle) is hit
    v = np.array([[0.0, 0.0, 0.0], [0.75, 0.0, 0.0], [0.0, 0.75, 0.0]])
    w, f = wv.winding_number_batch(wv.TriangleMesh(v, [[0, 1, 2]]), [[0.25, 0.25, 0.0]],
                                   mode="soft", precision="f32")
    assert f[0]


def _subset(w, n, seed):
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(w.n_nodes, size=n, replace=False))
    return orc.node_coordinates(w.lo, w.hi, w.res)[idx]


@pytest.mark.parametrize("mode", ["soft", "exact"])
def test_backward_f32_vs_oracle_open_torus(torch_, c2, mode):
    """C2 (open torus with holes, 19.8k faces): random coefficients on 2048
    seeded lattice nodes, vertex gradients vs the f64 oracle."""
    torch = torch_
    from paper_2407_11272_b200 import device
    pts = _subset(c2, 2048, 5)
    coefs = np.random.default_rng(6).normal(size=len(pts))
    dm = device.DeviceMesh.from_numpy(c2.vertices, c2.faces)
    fg = device.face_grad(dm, mode, "f32", torch.as_tensor(coefs, dtype=torch.float32),
                          points=torch.as_tensor(pts, dtype=torch.float32))
    got = device.vertex_grad(dm, fg).cpu().numpy()
    coefs32 = coefs.astype(np.float32).astype(np.float64)
    pts32 = pts.astype(np.float32).astype(np.float64)
    if mode == "soft":
        ref = orc.soft_grad(c2.vertices, c2.faces, pts32, coefs32, chunk=256)
    else:
        ref = orc.exact_grad(c2.vertices, c2.faces, pts32, coefs32, chunk=256)
    assert rel_err(got, ref) <= G_TOL


def test_exact_backward_f32_vs_reference_fd(torch_):
    torch = torch_
    from paper_2407_11272_b200 import device
    g = golden("exact_grad_fd")
    for i in range(int(g["n"])):
        v, f, p, c, fd = (g[f"m{i}_{k}"] for k in ("vertices", "faces", "points", "coefs", "fd"))
        dm = device.DeviceMesh.from_numpy(v, f)
        fg = device.face_grad(dm, "exact", "f32", torch.as_tensor(c, dtype=torch.float32),
                              points=torch.as_tensor(p, dtype=torch.float32))
        got = device.vertex_grad(dm, fg).cpu().numpy()
        assert rel_err(got, fd) <= G_TOL, i


def test_exact_backward_closed_mesh_cancels(torch_):
    """Interior of a closed mesh: W is pinned at 1, the exact gradient sums
    to ~0 per vertex (test_grad.py:231-246)."""
    torch = torch_
    from paper_2407_11272_b200 import configs, device
    v, f = configs.icosphere(2, 1.0)
    pts = np.random.default_rng(1).normal(size=(512, 3)) * 0.2
    dm = device.DeviceMesh.from_numpy(v, f)
    fg = device.face_grad(dm, "exact", "f32", torch.ones(512), points=torch.as_tensor(pts))
    assert fg[0].shape[0] == 0  # every edge cancels: no active face
    got = device.vertex_grad(dm, fg).abs().max().item()
    assert got == 0.0
    ref = orc.exact_grad(v, f, pts, np.ones(512))  # face-wise closed form: rounding only
    assert np.abs(ref).max() < 1e-12


def test_soft_jacobians_f32(torch_):
    import paper_2407_11272_b200 as wv
    g = golden("soft_jacobians")
    for i in range(int(g["n"])):
        mesh = wv.TriangleMesh(g[f"m{i}_vertices"], g[f"m{i}_faces"])
        got = wv.soft_winding_vertex_jacobian(mesh, g[f"m{i}_q"], precision="f32").vectors
        assert rel_err(got, g[f"m{i}_jac"]) <= G_TOL, i


def test_loss_grad_f32_vs_reference(torch_):
    import paper_2407_11272_b200 as wv
    g = golden("loss_grad")
    mesh = wv.TriangleMesh(g["vertices"], g["faces"])
    spec = wv.GridSpec(*grid_of(g))
    r = wv.occupancy_loss_grad(mesh, wv.ScalarField(spec, g["target"]), precision="f32")
    assert abs(r.loss - float(g["loss"])) <= 1e-5 * abs(float(g["loss"]))
    assert rel_err(r.grads.vectors, g["grads"]) <= G_TOL
    assert r.excluded_nodes == int(g["excluded"])


def test_loss_grad_c2_exact_and_soft_vs_oracle(torch_, c2):
    """C2 config at a reduced 24^3 grid: loss against the closed torus's
    binarized occupancy, soft and exact, f32 device path vs f64 oracle."""
    import paper_2407_11272_b200 as wv
    from paper_2407_11272_b200 import configs
    cv, cf = configs.torus(0.7, 0.3, 100, 100)
    spec = wv.GridSpec(c2.lo, c2.hi, 24)
    pts = spec.node_coordinates()
    occ, _ = orc.winding_number_batch(cv, cf, pts)
    target = (occ > 0.5).astype(np.float64)
    mesh = wv.TriangleMesh(c2.vertices, c2.faces)
    for mode, fn, ofn in (("soft", wv.occupancy_loss_grad, orc.occupancy_loss_grad),
                          ("exact", wv.exact_loss_grad, orc.exact_loss_grad)):
        r = fn(mesh, wv.ScalarField(spec, target), precision="f32")
        loss, grads, excl = ofn(c2.vertices, c2.faces, pts.astype(np.float32).astype(np.float64),
                                target)
        assert abs(r.loss - loss) <= 1e-4 * abs(loss), mode
        assert r.excluded_nodes == excl, mode
        assert rel_err(r.grads.vectors, grads) <= G_TOL, mode


def test_autograd_matches_device_kernels(torch_):
    torch = torch_
    import paper_2407_11272_b200 as wv
    from paper_2407_11272_b200 import configs
    v, f = configs.icosphere(2, 0.6)
    f = f[v[f].mean(axis=1)[:, 2] < 0.3]  # open cap: the exact gradient lives on the rim
    verts = torch.tensor(v, dtype=torch.float32, device="cuda", requires_grad=True)
    faces = torch.tensor(f, dtype=torch.int32, device="cuda")
    grid = ((-1.0,) * 3, (1.0,) * 3, (12, 12, 12))
    for mode in ("soft", "exact"):
        W, flags = wv.winding_number(verts, faces, grid=grid, mode=mode)
        tgt = torch.rand(W.shape, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
        loss = ((W - tgt) ** 2).sum()
        (g,) = torch.autograd.grad(loss, verts)
        coefs = (2 * (W - tgt)).detach().double().cpu().numpy()
        pts = wv.GridSpec(*grid).node_coordinates().astype(np.float32).astype(np.float64)
        vv = v.astype(np.float32).astype(np.float64)
        ref = (orc.soft_grad if mode == "soft" else orc.exact_grad)(vv, f, pts, coefs)
        assert rel_err(g.double().cpu().numpy(), ref) <= G_TOL, mode


@pytest.mark.parametrize("mode", ["exact", "soft"])
def test_row_kernels_match_generic_bitwise(torch_, c2, mode):
    """Row-aligned grid ranges run the lattice-row kernels (x/y parts hoisted
    per face); they must reproduce the generic point kernels on the same f32
    coordinates, flags included; values to fp32 rounding.  Exact: both pair
    faces for one angle evaluation, but the row kernel's vertex-hit screen is
    the per-face row bound and the generic one's the per-lane distances, so a
    pair can go face by face in one and not the other.  Soft: the row kernel
    drops the centroid's lo part for pairs beyond the face's near threshold
    (< 2e-8 per term), the generic kernel always adds it.  rz=40 (row mode),
    rz=36 (generic grid), and an unaligned slab start."""
    from paper_2407_11272_b200 import device as D
    dm = D.DeviceMesh.from_numpy(c2.vertices, c2.faces)
    for res, n0, count in [((24, 20, 40), 0, None), ((24, 20, 40), 40 * 20 * 5, 40 * 20 * 7),
                           ((22, 18, 36), 0, None), ((24, 20, 40), 12, 4000)]:
        grid = ((-1.0, -1.0, -1.0), (1.0, 1.0, 1.0), res)
        n = int(np.prod(res))
        count = n - n0 if count is None else count
        wg, fg = D.forward(dm, mode, "f32", grid=grid, n0=n0, count=count)
        pts = orc.node_coordinates(*grid)[n0:n0 + count].astype(np.float32)
        wp, fp = D.forward(dm, mode, "f32", points=torch_.from_numpy(pts).cuda())
        assert np.array_equal(fg.cpu().numpy(), fp.cpu().numpy())
        scale = max(1.0, wp.abs().max().item())
        assert (wg - wp).abs().max().item() <= (2e-7 if mode == "exact" else 1e-6) * scale


@pytest.mark.parametrize("mode", ["exact", "soft"])
def test_row_backward_matches_generic_and_oracle(torch_, c2, mode):
    """Grid backward in row mode (k-row runs, per-face row constants) vs the
    generic point-list kernel on the same f32 nodes and coefficients, and vs
    the f64 oracle.  Includes zero coefficients (skipped / parked pairs), an
    odd count, a slab start inside a row, and rz=18 (short runs)."""
    torch = torch_
    from paper_2407_11272_b200 import device as D
    dm = D.DeviceMesh.from_numpy(c2.vertices, c2.faces)
    rng = np.random.default_rng(9)
    for res, n0, count in [((12, 10, 40), 0, 4800), ((12, 10, 40), 402, 3001),
                           ((14, 12, 18), 36, 2000)]:
        grid = ((-1.0, -1.0, -1.0), (1.0, 1.0, 1.0), res)
        coefs = rng.normal(size=count)
        coefs[rng.random(count) < 0.3] = 0.0
        ct = torch.as_tensor(coefs, dtype=torch.float32)
        got = D.vertex_grad(dm, D.face_grad(dm, mode, "f32", ct, grid=grid, n0=n0,
                                            count=count)).cpu().numpy()
        pts32 = orc.node_coordinates(*grid)[n0:n0 + count].astype(np.float32)
        gen = D.vertex_grad(dm, D.face_grad(dm, mode, "f32", ct,
                                            points=torch.from_numpy(pts32).cuda())).cpu().numpy()
        assert rel_err(got, gen) <= 2e-6
        ofn = orc.soft_grad if mode == "soft" else orc.exact_grad
        ref = ofn(c2.vertices, c2.faces, pts32.astype(np.float64),
                  coefs.astype(np.float32).astype(np.float64), chunk=256)
        assert rel_err(got, ref) <= G_TOL


@pytest.mark.parametrize("scale", [1.0e6, 3.0e-4])
def test_row_backward_scale_invariance(torch_, c2, scale):
    """The row backward forms d01 d12 d20 (~|x|^6) for its shared reciprocal;
    a power-of-two rescaling keeps that product in range at any input scale.
    Scaling mesh and lattice by L scales dW/dv by 1/L (f32 tolerance)."""
    torch = torch_
    from paper_2407_11272_b200 import device as D
    res = (12, 10, 40)
    coefs = torch.from_numpy(np.random.default_rng(3).normal(size=int(np.prod(res)))).float()

    def grads(L):
        dm = D.DeviceMesh.from_numpy(c2.vertices * L, c2.faces)
        grid = ((-L,) * 3, (L,) * 3, res)
        return D.vertex_grad(dm, D.face_grad(dm, "exact", "f32", coefs, grid=grid)).cpu().numpy()

    g1, gs = grads(1.0), grads(scale)
    assert np.isfinite(gs).all()
    assert rel_err(gs * scale, g1) <= G_TOL  # inputs re-rounded at the new scale
