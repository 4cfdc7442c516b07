"""GPU parity of the FP32 exact forward against the reference (golden
fixtures) and the CPU oracle.

Tolerances are north_star's: |W_gpu - W_ref| <= 1e-5 absolute against an
FP64 reference evaluation on unflagged nodes; thresholded occupancy
bit-exact except nodes with |w - 0.5| < 1e-3; identical on-surface flags.
"""

import numpy as np
import pytest

from conftest import golden, grid_of
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

W_TOL = 1e-5


@pytest.fixture(scope="module")
def wv(cuda_device):
    import paper_2407_11272_b200 as wv
    return wv


def assert_parity(w_gpu, f_gpu, w_ref, f_ref, tol=W_TOL):
    w_gpu = np.asarray(w_gpu, dtype=np.float64)
    assert np.array_equal(np.asarray(f_gpu, bool), np.asarray(f_ref, bool)), \
        f"flag mismatches: {(np.asarray(f_gpu, bool) != np.asarray(f_ref, bool)).sum()}"
    ok = ~np.asarray(f_ref, bool)
    err = np.abs(w_gpu[ok] - w_ref[ok])
    assert err.max(initial=0.0) <= tol, f"max |dW| = {err.max():.3e}"
    amb = (np.abs(w_ref - 0.5) < 1e-3) | (np.abs(w_gpu - 0.5) < 1e-3)
    assert np.array_equal((w_gpu > 0.5)[~amb], (w_ref > 0.5)[~amb])


def test_c1_full_grid_vs_reference(wv):
    g = golden("c1_icosphere3_r32")
    lo, hi, res = grid_of(g)
    mesh = wv.TriangleMesh(g["vertices"], g["faces"])
    spec = wv.GridSpec(lo, hi, res)
    field = wv.voxelize(mesh, spec, precision="f32")
    assert field.values.dtype == np.float32
    assert_parity(field.values, g["flags"], g["exact_f64"], g["flags"])
    raw, flags = wv.winding_number_batch(mesh, spec.node_coordinates(), precision="f32")
    assert_parity(raw, flags, g["raw"], g["flags"])


def test_census_cube_r9(wv):
    g = golden("census_cube_r9")
    mesh = wv.TriangleMesh(g["vertices"], g["faces"])
    field = wv.voxelize(mesh, wv.GridSpec(*grid_of(g)), precision="f32")
    v = field.values.astype(np.float64)
    counts = (np.sum(np.abs(v - 1.0) < 1e-6), np.sum(v == 0.5), np.sum(np.abs(v) < 1e-6))
    assert counts == (27, 98, 604)  # test_winding.py:276-288
    assert np.array_equal(v == 0.5, g["values"] == 0.5)


@pytest.mark.parametrize("tag", ["ico", "torus"])
def test_point_batches(wv, tag):
    g = golden("point_batches")
    mesh = wv.TriangleMesh(g[f"{tag}_vertices"], g[f"{tag}_faces"])
    w, f = wv.winding_number_batch(mesh, g[f"{tag}_points"], precision="f32")
    assert_parity(w, f, g[f"{tag}_exact"], g[f"{tag}_exact_flags"])


def test_flip_negates_exactly(wv):
    g = golden("point_batches")
    mesh = wv.TriangleMesh(g["ico_vertices"], g["ico_faces"])
    flipped = wv.TriangleMesh(mesh.vertices, mesh.faces[:, [0, 2, 1]])
    pts = np.random.default_rng(7).normal(size=(4096, 3)) * 1.5
    a, fa = wv.winding_number_batch(mesh, pts, precision="f32")
    b, fb = wv.winding_number_batch(flipped, pts, precision="f32")
    assert np.array_equal(fa, fb)
    # test_winding.py:131-140 asserts a bit-exact negation for the f64 kernel
    # (the f64 path keeps it, test_gpu_f64_parity.py); the FP32 path fuses
    # beta's products into FMAs, so the negation holds to rounding
    assert np.abs(a[~fa] + b[~fb]).max() <= 1e-6


def test_icosphere2_r13_vs_reference(wv):
    g = golden("voxelize_icosphere2_r13")
    mesh = wv.TriangleMesh(g["vertices"], g["faces"])
    spec = wv.GridSpec(*grid_of(g))
    field = wv.voxelize(mesh, spec, precision="f32")
    ref = g["exact_f64"]
    assert np.abs(field.values.astype(np.float64) - ref).max() <= W_TOL


def test_open_shell_and_vertex_hit(wv):
    g = golden("open_hemisphere_shell")
    mesh = wv.TriangleMesh(g["vertices"], g["faces"])
    w, f = wv.winding_number_batch(mesh, g["points"], precision="f32")
    assert_parity(w, f, g["values"], g["flags"])
    s = golden("kernel_abi_soup")
    soupm = wv.TriangleMesh(s["vertices"], s["faces"])  # one degenerate face
    w, f = wv.winding_number_batch(soupm, s["points"], precision="f32")
    assert f[0]  # query exactly on a vertex is flagged (_kernels.py:65-67)
    assert_parity(w, f, s["exact"], s["exact_flags"])


def test_empty_mesh_and_empty_points(wv):
    empty = wv.TriangleMesh(np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int64))
    spec = wv.GridSpec((-1.0,) * 3, (1.0,) * 3, 4)
    assert np.array_equal(wv.voxelize(empty, spec, precision="f32").values, np.zeros(64))
    w, f = wv.winding_number_batch(empty, np.zeros((0, 3)), precision="f32")
    assert w.shape == (0,) and f.shape == (0,)


def test_torus20k_random_nodes_vs_oracle(wv):
    from paper_2407_11272_b200 import configs
    w = configs.make("c2")
    rng = np.random.default_rng(11)
    spec = wv.GridSpec(w.lo, w.hi, w.res)
    idx = np.sort(rng.choice(spec.num_nodes, size=3000, replace=False))
    pts = orc.node_coordinates(w.lo, w.hi, w.res)[idx]
    ref, rf = orc.winding_number_batch(w.vertices, w.faces, pts)
    got, gf = wv.winding_number_batch(wv.TriangleMesh(w.vertices, w.faces), pts, precision="f32")
    assert_parity(got, gf, ref, rf)


def test_grid_slabs_equal_full_grid(cuda_device):
    """Node-range slabs (the multi-GPU shard unit) reproduce the full grid
    bit-for-bit, with and without face splits."""
    import torch
    from paper_2407_11272_b200 import configs, device
    w = configs.make("c2")
    dm = device.DeviceMesh.from_numpy(w.vertices, w.faces)
    grid = (w.lo, w.hi, (64, 64, 64))
    full, ff = device.exact_forward_f32(dm, grid=grid)
    n = 64 ** 3
    parts = [device.exact_forward_f32(dm, grid=grid, n0=s, count=n // 4)
             for s in range(0, n, n // 4)]
    got = torch.cat([p[0] for p in parts])
    gotf = torch.cat([p[1] for p in parts])
    torch.cuda.synchronize()
    assert torch.equal(gotf, ff)
    assert (got - full).abs().max().item() <= 1e-6
