"""Properties the reference's own test suite asserts, run through
the device path: invariances, known answers, the two-argument arctangent
regression, determinism, batch == scalar, the loss optimum, the gradient sum
rule, translation equivariance and orientation antisymmetry of the Jacobian.

Reference sites: test_winding.py:45-83, 114-179, 299-333;
test_acceptance.py:89-111; test_grad.py:75-132.
"""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wv(cuda_device):
    import paper_2407_11272_b200 as m
    return m


def cube(wv):
    g = golden("census_cube_r9")
    return wv.TriangleMesh(g["vertices"], g["faces"])


def rotation(seed):
    q, _ = np.linalg.qr(np.random.default_rng(seed).normal(size=(3, 3)))
    return q * np.sign(np.linalg.det(q))


@pytest.mark.parametrize("precision,tol", [("f64", 1e-9), ("f32", 1e-5)])
def test_rigid_motion_and_scale_invariance(wv, precision, tol):
    """test_winding.py:143-163: W is invariant under a rigid motion and a
    uniform scale of mesh and points together."""
    from paper_2407_11272_b200 import configs
    v, f = configs.torus(0.6, 0.25, 24, 16)
    rng = np.random.default_rng(3)
    pts = rng.uniform(-1.0, 1.0, size=(400, 3))
    w0, f0 = wv.winding_number_batch(wv.TriangleMesh(v, f), pts, precision=precision)
    R, t = rotation(5), np.array([0.3, -1.2, 2.0])
    w1, f1 = wv.winding_number_batch(wv.TriangleMesh(v @ R.T + t, f), pts @ R.T + t,
                                     precision=precision)
    w2, f2 = wv.winding_number_batch(wv.TriangleMesh(v * 3.5, f), pts * 3.5, precision=precision)
    assert not f0.any() and np.array_equal(f0, f1) and np.array_equal(f0, f2)
    assert np.abs(w0 - w1).max() < tol and np.abs(w0 - w2).max() < tol


@pytest.mark.parametrize("precision,tol", [("f64", 1e-9), ("f32", 1e-6)])
def test_octahedron_and_single_triangle(wv, precision, tol):
    """test_winding.py:50-56, 174-179: the octahedron's eight solid angles
    sum to 4 pi (W = 1 at its centre); a single triangle gives Omega / 4 pi."""
    ov = np.array([[1.0, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]])
    of = np.array([[0, 2, 4], [2, 1, 4], [1, 3, 4], [3, 0, 4],
                   [2, 0, 5], [1, 2, 5], [3, 1, 5], [0, 3, 5]])
    w, _ = wv.winding_number_batch(wv.TriangleMesh(ov, of), np.zeros((1, 3)), precision=precision)
    assert abs(w[0] - 1.0) < tol
    tri = np.array([[0.3, -0.2, 0.9], [1.1, 0.4, 0.2], [-0.5, 0.8, 0.4]])
    q = np.array([[0.05, 0.1, -0.3]])
    w, _ = wv.winding_number_batch(wv.TriangleMesh(tri, np.array([[0, 1, 2]])), q,
                                   precision=precision)
    omega = wv.solid_angle_triangle(tri[0], tri[1], tri[2], q[0])
    assert abs(w[0] - omega / (4 * np.pi)) < (1e-15 if precision == "f64" else tol)


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_two_argument_arctangent_keeps_nodes_saturated(wv, precision):
    """test_acceptance.py:89-111: on the cube at 64^3, nodes farther than one
    spacing from the surface are < 1e-3 fractional (0.1 < W < 0.9)."""
    spec = wv.GridSpec((-1.0,) * 3, (1.0,) * 3, 64)
    vals = wv.voxelize(cube(wv), spec, precision=precision).values
    from oracle import oracle as orc
    nodes = orc.node_coordinates((-1.0,) * 3, (1.0,) * 3, (64,) * 3)
    clear = np.abs(np.abs(nodes).max(axis=1) - 0.5) > 2.0 / 63
    v = vals[clear]
    assert float(np.mean((v > 0.1) & (v < 0.9))) < 1e-3


def test_determinism_and_batch_equals_scalar(wv):
    """test_winding.py:299-333: repeated evaluations are byte-identical;
    batched values equal per-point calls bitwise (f64)."""
    import torch
    from paper_2407_11272_b200 import configs, device
    v, f = configs.torus_with_holes()
    spec = wv.GridSpec((-1.0,) * 3, (1.0,) * 3, 40)
    mesh = wv.TriangleMesh(v, f)
    a = wv.voxelize(mesh, spec, precision="f32").values
    b = wv.voxelize(mesh, spec, precision="f32").values
    assert a.tobytes() == b.tobytes()
    dm = device.DeviceMesh.from_numpy(v, f)
    grid = ((-1.0,) * 3, (1.0,) * 3, (40, 40, 40))
    coefs = torch.from_numpy(np.random.default_rng(2).normal(size=40 ** 3)).float().cuda()
    g1 = device.vertex_grad(dm, device.face_grad(dm, "exact", "f32", coefs, grid=grid))
    g2 = device.vertex_grad(dm, device.face_grad(dm, "exact", "f32", coefs, grid=grid))
    assert g1.cpu().numpy().tobytes() == g2.cpu().numpy().tobytes()
    pts = np.random.default_rng(4).uniform(-0.9, 0.9, size=(24, 3))
    wb, _ = wv.winding_number_batch(mesh, pts)
    ws = np.array([wv.winding_number_exact(mesh, p) for p in pts])
    assert wb.tobytes() == ws.tobytes()


def test_loss_at_global_minimum_is_zero(wv):
    """test_grad.py:124-132 (f64 path)."""
    from paper_2407_11272_b200 import configs
    v, f = configs.icosphere(0, 0.5)
    mesh = wv.TriangleMesh(v, f)
    spec = wv.GridSpec((-1.0,) * 3, (1.0,) * 3, 6)
    from oracle import oracle as orc
    nodes = orc.node_coordinates((-1.0,) * 3, (1.0,) * 3, (6, 6, 6))
    values, flags = wv.winding_number_batch(mesh, nodes, mode="soft")
    assert not flags.any()
    r = wv.occupancy_loss_grad(mesh, wv.ScalarField(spec, values))
    assert r.loss < 1e-20 and np.abs(r.grads.vectors).max() < 1e-10 and r.excluded_nodes == 0


@pytest.mark.parametrize("precision,tol", [("f64", 1e-9), ("f32", 2e-4)])
def test_soft_jacobian_sum_rule_equivariance_antisymmetry(wv, precision, tol):
    """test_grad.py:75-107: sum over vertices of dW/dv = -dW/dq (central FD
    of the reference-exact f64 forward in q); translation equivariance;
    orientation antisymmetry (bit-exact in f64)."""
    from paper_2407_11272_b200 import configs
    v, f = configs.icosphere(1, 0.8)
    mesh = wv.TriangleMesh(v, f)
    q = np.array([0.3, 1.4, -0.2])
    jac = wv.soft_winding_vertex_jacobian(mesh, q, precision=precision).vectors
    h = 1e-6
    gq = np.array([(wv.winding_number_soft(mesh, q + h * e) - wv.winding_number_soft(mesh, q - h * e))
                   / (2 * h) for e in np.eye(3)])
    assert np.abs(jac.sum(axis=0) + gq).max() < tol * max(1.0, np.abs(gq).max())
    t = np.array([5.0, -3.0, 2.0])
    moved = wv.soft_winding_vertex_jacobian(wv.TriangleMesh(v + t, f), q + t,
                                            precision=precision).vectors
    assert np.abs(jac - moved).max() < (1e-12 if precision == "f64" else tol) * np.abs(jac).max()
    flipped = wv.soft_winding_vertex_jacobian(wv.TriangleMesh(v, f[:, [0, 2, 1]]), q,
                                              precision=precision).vectors
    if precision == "f64":
        assert np.array_equal(jac, -flipped)
    else:
        assert np.abs(jac + flipped).max() < tol * np.abs(jac).max()


def test_exact_gradient_sum_rule(wv):
    """Exact backward: translating every vertex by t moves W like moving q
    by -t, so the vertex gradients of sum_p c_p W_p sum to -sum_p c_p dW_p/dq
    (central FD of the f64 forward), on an open mesh (a closed one has zero
    vertex gradient, test_grad.py:231-246)."""
    import torch
    from paper_2407_11272_b200 import device
    g = golden("open_hemisphere_shell")
    v, f = g["hemi_vertices"], g["hemi_faces"]
    mesh = wv.TriangleMesh(v, f)
    rng = np.random.default_rng(8)
    pts = rng.uniform(-0.6, 0.6, size=(16, 3))
    c = rng.normal(size=16)
    dm = device.DeviceMesh.from_numpy(v, f)
    grads = device.vertex_grad(dm, device.face_grad(dm, "exact", "f64", torch.from_numpy(c).cuda(),
                                                    points=torch.from_numpy(pts).cuda()))
    total = grads.sum(dim=0).cpu().numpy()
    h = 1e-6
    gq = np.zeros(3)
    for k, e in enumerate(np.eye(3)):
        wp, _ = wv.winding_number_batch(mesh, pts + h * e)
        wm, _ = wv.winding_number_batch(mesh, pts - h * e)
        gq[k] = float(((wp - wm) * c).sum()) / (2 * h)
    assert np.abs(total + gq).max() < 1e-7 * max(1.0, np.abs(gq).max())
