"""Pin the CPU oracle to the reference (CPU-only).

Every fixture was produced by importing the reference package itself
(tests/golden/make_golden.py).  The oracle restates the reference numba
kernels with identical operation order, so forward values, flags and soft
gradients must match BIT-FOR-BIT; the new exact d(Omega)/dv closed form is
pinned against central finite differences of the reference exact kernel.
"""

import numpy as np
import pytest

from conftest import golden, grid_of
from oracle import oracle as orc


def test_census_cube_r9_bit_exact():
    g = golden("census_cube_r9")
    pts = orc.node_coordinates(*grid_of(g))
    vals, flags = orc.voxelize(g["vertices"], g["faces"], pts)
    assert vals.tobytes() == g["values"].tobytes()
    assert np.array_equal(flags, g["flags"])
    ones = np.sum(np.abs(vals - 1.0) < 1e-9)
    halves = np.sum(vals == 0.5)
    zeros = np.sum(np.abs(vals) < 1e-9)
    assert (ones, halves, zeros) == (27, 98, 604)  # test_winding.py:276-288


@pytest.mark.parametrize("tag", ["ico", "torus"])
def test_point_batches_bit_exact(tag):
    g = golden("point_batches")
    v, f, p = g[f"{tag}_vertices"], g[f"{tag}_faces"], g[f"{tag}_points"]
    for mode, key, atan2 in (("exact", "exact", True), ("soft", "soft", True),
                             ("exact", "arctan", False)):
        vals, flags = orc.winding_number_batch(v, f, p, mode=mode, use_atan2=atan2)
        assert vals.tobytes() == g[f"{tag}_{key}"].tobytes(), (mode, key)
        assert np.array_equal(flags, g[f"{tag}_{key}_flags"])


@pytest.mark.parametrize("threads,chunk", [(1, 2000), (3, 7), (8, 64)])
def test_oracle_independent_of_threads_and_chunks(threads, chunk):
    g = golden("voxelize_icosphere2_r13")
    pts = orc.node_coordinates(*grid_of(g))
    vals, _ = orc.winding_number_batch(g["vertices"], g["faces"], pts, chunk=chunk,
                                       threads=threads)
    vals[_] = 0.5
    assert vals.tobytes() == g["exact_f64"].tobytes()


def test_voxelize_f64_and_f32_bit_exact():
    g = golden("voxelize_icosphere2_r13")
    pts = orc.node_coordinates(*grid_of(g))
    for mode in ("exact", "soft"):
        v64, _ = orc.voxelize(g["vertices"], g["faces"], pts, mode=mode)
        assert v64.tobytes() == g[f"{mode}_f64"].tobytes(), mode
        v32, _ = orc.voxelize(g["vertices"], g["faces"], pts, mode=mode, precision="f32")
        assert v32.dtype == np.float32
        assert v32.tobytes() == g[f"{mode}_f32"].tobytes(), mode


def test_c1_config_bit_exact():
    g = golden("c1_icosphere3_r32")
    pts = orc.node_coordinates(*grid_of(g))
    raw, flags = orc.winding_number_batch(g["vertices"], g["faces"], pts)
    assert raw.tobytes() == g["raw"].tobytes()
    assert np.array_equal(flags, g["flags"])
    soft, _ = orc.voxelize(g["vertices"], g["faces"], pts, mode="soft")
    assert soft.tobytes() == g["soft_f64"].tobytes()


def test_open_mesh_shell():
    g = golden("open_hemisphere_shell")
    vals, flags = orc.winding_number_batch(g["vertices"], g["faces"], g["points"])
    assert vals.tobytes() == g["values"].tobytes()
    assert np.array_equal(flags, g["flags"])
    between = vals[:-2]
    assert between.min() > 0.9 and between.max() < 1.1  # test_openmesh.py:44-55
    assert abs(vals[-2]) < 0.1


def test_soft_jacobians_bit_exact():
    g = golden("soft_jacobians")
    for i in range(int(g["n"])):
        v, f, q = g[f"m{i}_vertices"], g[f"m{i}_faces"], g[f"m{i}_q"]
        jac = orc.soft_grad(v, f, q.reshape(1, 3), np.ones(1))
        assert jac.tobytes() == g[f"m{i}_jac"].tobytes(), i


def test_occupancy_loss_grad_bit_exact():
    g = golden("loss_grad")
    pts = orc.node_coordinates(*grid_of(g))
    loss, grads, excl = orc.occupancy_loss_grad(g["vertices"], g["faces"], pts, g["target"])
    assert loss == float(g["loss"])
    assert grads.tobytes() == g["grads"].tobytes()
    assert excl == int(g["excluded"])
    wl, wg, _ = orc.occupancy_loss_grad(g["vertices"], g["faces"], pts, g["target"],
                                        weights=g["weights"])
    assert wl == float(g["wloss"])
    assert wg.tobytes() == g["wgrads"].tobytes()
    epts = orc.node_coordinates(*grid_of(g, "ex_grid"))
    el, eg, ee = orc.occupancy_loss_grad(g["ex_vertices"], g["ex_faces"], epts, g["ex_target"])
    assert ee == int(g["ex_excluded"]) == 1
    assert el == float(g["ex_loss"])
    assert eg.tobytes() == g["ex_grads"].tobytes()


def test_kernel_abi_soup_bit_exact():
    g = golden("kernel_abi_soup")
    v, f, p = g["vertices"], g["faces"], g["points"]
    ex, fl = orc.winding_number_batch(v, f, p)
    assert ex.tobytes() == g["exact"].tobytes()
    assert np.array_equal(fl, g["exact_flags"]) and fl[0]
    so, sf = orc.winding_number_batch(v, f, p, mode="soft")
    assert so.tobytes() == g["soft"].tobytes()
    assert np.array_equal(sf, g["soft_flags"])
    e32, f32 = orc.voxelize_f32(v, f, p, "exact")
    raw32 = e32.copy()
    ref32 = g["exact32"].copy()
    ref32[g["exact32_flags"]] = 0.5
    assert raw32.tobytes() == ref32.tobytes()
    s32, _ = orc.voxelize_f32(v, f, p, "soft")
    sref = g["soft32"].copy()
    sref[g["soft32_flags"]] = 0.5
    assert s32.tobytes() == sref.tobytes()
    grad = orc.soft_grad(v, f, p, g["coefs"], chunk=10 ** 9, threads=1)
    assert grad.tobytes() == g["soft_grad"].tobytes()


def test_exact_grad_closed_form_matches_reference_fd():
    g = golden("exact_grad_fd")
    for i in range(int(g["n"])):
        v, f, p, c, fd = (g[f"m{i}_{k}"] for k in ("vertices", "faces", "points",
                                                     "coefs", "fd"))
        an = orc.exact_grad(v, f, p, c)
        assert np.abs(an - fd).max() / np.abs(fd).max() < 1e-6, i


def test_exact_grad_sum_rule_and_closed_mesh_cancellation():
    # closed mesh: moving any vertex leaves interior/exterior W unchanged
    # (test_grad.py:231-246), so the per-vertex exact gradient cancels.
    g = golden("point_batches")
    v, f = g["ico_vertices"], g["ico_faces"]
    pts = np.array([[0.1, -0.05, 0.2], [2.0, 0.3, -0.4]])
    grad = orc.exact_grad(v, f, pts, np.ones(2))
    assert np.abs(grad).max() < 1e-12


def test_solid_angle_known_answers():
    g = golden("solid_angle_known")
    assert abs(float(g["octant"]) - np.pi / 2) < 1e-12
    w, _ = orc.winding_number_batch(np.array([[0, 0, 0], [1.0, 0, 0], [0, 1.0, 0]]),
                                    [[0, 1, 2]], np.array([[0.2, 0.3, 0.7]]))
    assert abs(float(g["cube_face_center"]) - 0.5) < 1e-9


def big_vector():
    """Same seeds as tests/golden/make_golden.py:big_vector."""
    return (np.random.default_rng(62).random(100003)
            * 10.0 ** np.random.default_rng(63).integers(-3, 3, size=100003))


def test_metrics_oracle_bit_exact():
    """Reconstruction metrics (metrics.py:43-150) restated in numpy vs the
    reference's own outputs: SplitMix64 streams, area-weighted samples (with
    zero-area faces present), nearest distances, Chamfer / Hausdorff, and the
    evaluate_reconstruction statistics."""
    g = golden("metrics")
    assert np.array_equal(orc.splitmix64_uniform(7, 10000), g["u_seed7"])
    assert np.array_equal(orc.splitmix64_uniform((1 << 64) - 3, 999), g["u_seed_big"])
    assert orc.sample_surface(g["ico_vertices"], g["ico_faces"], 4001, 3).tobytes() \
        == g["s_ico"].tobytes()
    assert orc.sample_surface(g["degen_vertices"], g["degen_faces"], 2000, 11).tobytes() \
        == g["s_degen"].tobytes()
    assert orc.nearest_distances(g["pa"], g["pb"]).tobytes() == g["nn_ab"].tobytes()
    assert orc.chamfer_distance(g["pa"], g["pb"]) == float(g["chamfer_ab"])
    assert orc.hausdorff_distance(g["pa"], g["pb"]) == float(g["hausdorff_ab"])
    ch, hd = [], []
    for r in range(3):
        a = orc.sample_surface(g["ico_vertices"], g["ico_faces"], 3000, 5 + r)
        b = orc.sample_surface(g["cube_vertices"], g["cube_faces"], 3000, 5 + r)
        ch.append(orc.chamfer_distance(a, b))
        hd.append(orc.hausdorff_distance(a, b))
    got = np.array([np.mean(ch), np.std(ch), np.mean(hd), np.std(hd)])
    assert got.tobytes() == g["recon"].tobytes()
    big = big_vector()
    assert float(np.sum(big)) == float(g["big_sum"]) and float(big.mean()) == float(g["big_mean"])
