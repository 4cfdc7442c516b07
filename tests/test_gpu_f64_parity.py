"""GPU f64 parity path against the reference's own outputs (golden fixtures).

The f64 kernels mirror the reference kernels' operation order: the soft
forward is bit-exact, the exact forward differs only through CUDA's vs
libm's atan2 (<= a few ulp per term), so the reference's own tolerances
(1e-9 and tighter, pkg/tests/test_winding.py) hold with room to spare.
"""

import numpy as np
import pytest

from conftest import golden, grid_of

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wv(cuda_device):
    import paper_2407_11272_b200 as wv
    return wv


def test_census_and_c1_f64(wv):
    g = golden("census_cube_r9")
    f = wv.voxelize(wv.TriangleMesh(g["vertices"], g["faces"]), wv.GridSpec(*grid_of(g)))
    assert f.values.dtype == np.float64
    assert np.array_equal(f.values == 0.5, g["values"] == 0.5)
    assert np.abs(f.values - g["values"]).max() < 1e-12
    c1 = golden("c1_icosphere3_r32")
    mesh = wv.TriangleMesh(c1["vertices"], c1["faces"])
    spec = wv.GridSpec(*grid_of(c1))
    got = wv.voxelize(mesh, spec).values
    assert np.abs(got - c1["exact_f64"]).max() < 1e-12
    soft = wv.voxelize(mesh, spec, mode="soft").values
    assert soft.tobytes() == c1["soft_f64"].tobytes()  # bit-exact


@pytest.mark.parametrize("tag", ["ico", "torus"])
def test_point_batches_f64(wv, tag):
    g = golden("point_batches")
    mesh = wv.TriangleMesh(g[f"{tag}_vertices"], g[f"{tag}_faces"])
    p = g[f"{tag}_points"]
    ex, fe = wv.winding_number_batch(mesh, p)
    assert np.array_equal(fe, g[f"{tag}_exact_flags"])
    assert np.abs(ex - g[f"{tag}_exact"]).max() < 1e-12
    so, fs = wv.winding_number_batch(mesh, p, mode="soft")
    assert np.array_equal(fs, g[f"{tag}_soft_flags"])
    assert so.tobytes() == g[f"{tag}_soft"].tobytes()
    ar, fa = wv.winding_number_batch(mesh, p, use_atan2=False)
    assert np.abs(ar - g[f"{tag}_arctan"]).max() < 1e-12


def test_flip_antisymmetry_f64(wv):
    g = golden("point_batches")
    mesh = wv.TriangleMesh(g["ico_vertices"], g["ico_faces"])
    flipped = wv.TriangleMesh(mesh.vertices, mesh.faces[:, [0, 2, 1]])
    pts = np.random.default_rng(7).normal(size=(200, 3)) * 1.5
    for mode in ("exact", "soft"):
        a, fa = wv.winding_number_batch(mesh, pts, mode=mode)
        b, fb = wv.winding_number_batch(flipped, pts, mode=mode)
        assert np.array_equal(fa, fb)
        assert np.array_equal(a[~fa], -b[~fb])


def test_soft_jacobians_f64(wv):
    g = golden("soft_jacobians")
    for i in range(int(g["n"])):
        mesh = wv.TriangleMesh(g[f"m{i}_vertices"], g[f"m{i}_faces"])
        got = wv.soft_winding_vertex_jacobian(mesh, g[f"m{i}_q"]).vectors
        ref = g[f"m{i}_jac"]
        assert np.abs(got - ref).max() <= 1e-13 * max(np.abs(ref).max(), 1e-300), i


def test_soft_jacobian_raises_on_centroid(wv):
    mesh = wv.TriangleMesh(golden("census_cube_r9")["vertices"], golden("census_cube_r9")["faces"])
    centroid = mesh.vertices[mesh.faces[4]].mean(axis=0)
    with pytest.raises(wv.OnSurfaceError):
        wv.soft_winding_vertex_jacobian(mesh, centroid)


def test_occupancy_loss_grad_f64(wv):
    g = golden("loss_grad")
    mesh = wv.TriangleMesh(g["vertices"], g["faces"])
    spec = wv.GridSpec(*grid_of(g))
    r = wv.occupancy_loss_grad(mesh, wv.ScalarField(spec, g["target"]))
    assert abs(r.loss - float(g["loss"])) <= 1e-13 * abs(float(g["loss"]))
    assert np.abs(r.grads.vectors - g["grads"]).max() <= 1e-12 * np.abs(g["grads"]).max()
    assert r.excluded_nodes == int(g["excluded"])
    rw = wv.occupancy_loss_grad(mesh, wv.ScalarField(spec, g["target"]), weights=g["weights"])
    assert abs(rw.loss - float(g["wloss"])) <= 1e-13 * abs(float(g["wloss"]))
    assert np.abs(rw.grads.vectors - g["wgrads"]).max() <= 1e-12 * np.abs(g["wgrads"]).max()
    em = wv.TriangleMesh(g["ex_vertices"], g["ex_faces"])
    espec = wv.GridSpec(*grid_of(g, "ex_grid"))
    er = wv.occupancy_loss_grad(em, wv.ScalarField(espec, g["ex_target"]))
    assert er.excluded_nodes == 1
    assert abs(er.loss - float(g["ex_loss"])) <= 1e-13 * abs(float(g["ex_loss"]))
    assert np.abs(er.grads.vectors - g["ex_grads"]).max() <= 1e-12 * np.abs(g["ex_grads"]).max()
    # tampering with the excluded node's target changes nothing (test_grad.py:183-202)
    t2 = g["ex_target"].copy()
    origin = int(np.flatnonzero((np.abs(espec.node_coordinates()) < 1e-12).all(axis=1))[0])
    t2[origin] = 123.0
    er2 = wv.occupancy_loss_grad(em, wv.ScalarField(espec, t2))
    assert er2.loss == er.loss
    assert np.array_equal(er2.grads.vectors, er.grads.vectors)


def test_loss_validation(wv):
    g = golden("loss_grad")
    mesh = wv.TriangleMesh(g["vertices"], g["faces"])
    spec = wv.GridSpec(*grid_of(g))
    tgt = wv.ScalarField(spec, g["target"])
    with pytest.raises(ValueError):
        wv.occupancy_loss_grad(mesh, tgt, weights=-np.ones(spec.num_nodes))
    with pytest.raises(ValueError):
        wv.occupancy_loss_grad(mesh, tgt, weights=np.zeros(spec.num_nodes))
    empty = wv.TriangleMesh(np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int64))
    with pytest.raises(ValueError):
        wv.occupancy_loss_grad(empty, tgt)


def test_exact_grad_f64_vs_reference_fd(wv):
    """Exact d(W)/dv (no reference kernel) against central finite differences
    of the reference's exact_batch itself."""
    import torch
    from paper_2407_11272_b200 import device
    g = golden("exact_grad_fd")
    for i in range(int(g["n"])):
        v, f, p, c, fd = (g[f"m{i}_{k}"] for k in ("vertices", "faces", "points", "coefs", "fd"))
        dm = device.DeviceMesh.from_numpy(v, f)
        pts = torch.as_tensor(p, dtype=torch.float64)
        cf = torch.as_tensor(c, dtype=torch.float64)
        fg = device.face_grad(dm, "exact", "f64", cf, points=pts)
        got = device.vertex_grad(dm, fg).cpu().numpy()
        assert np.abs(got - fd).max() / np.abs(fd).max() < 1e-6, i


def test_flipped_duplication_bit_exact(wv):
    g = golden("openmesh_and_io")
    hemi = wv.TriangleMesh(g["hemi_vertices"], g["hemi_faces"])
    dup = wv.flipped_duplication(hemi, epsilon=0.02)
    assert dup.vertices.tobytes() == g["dup_vertices"].tobytes()
    assert np.array_equal(dup.faces, g["dup_faces"])
    with pytest.raises(ValueError):
        wv.flipped_duplication(hemi, epsilon=0.0)
    with pytest.raises(wv.DegenerateError):
        wv.flipped_duplication(wv.TriangleMesh(np.array([[0.0, 0, 0], [1, 0, 0], [2, 0, 0]]),
                                               [[0, 1, 2]]))
