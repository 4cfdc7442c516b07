"""Device-resident morph loop vs the reference's own traces (golden
morph_traces.npz, produced by windvox.morph.morph)."""

import numpy as np
import pytest

from conftest import golden, grid_of

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wv(cuda_device):
    import paper_2407_11272_b200 as wv
    return wv


def test_morph_trace_matches_reference_f64(wv):
    from paper_2407_11272_b200.morph import MorphConfig, morph
    g = golden("morph_traces")
    tmpl = wv.TriangleMesh(g["tmpl_vertices"], g["tmpl_faces"])
    target = wv.ScalarField(wv.GridSpec(*grid_of(g)), g["target"])
    res, rep = morph(tmpl, target, MorphConfig(iterations=10))
    losses = np.array([e["loss"] for e in rep.entries])
    assert len(losses) == len(g["losses"])
    assert np.abs(losses - g["losses"]).max() <= 1e-10 * g["losses"].max()
    gn = np.array([e["grad_inf_norm"] for e in rep.entries])
    assert np.abs(gn - g["gnorms"]).max() <= 1e-8 * g["gnorms"].max()
    assert np.abs(res.vertices - g["final"]).max() <= 1e-9
    assert all(b <= a for a, b in zip(losses, losses[1:]))  # monotone (morph.py:98-104)
    res2, rep2 = morph(tmpl, target, MorphConfig(iterations=6, momentum=0.0, smooth_weight=0.0,
                                                 step_size=0.2))
    l2 = np.array([e["loss"] for e in rep2.entries])
    assert np.abs(l2 - g["losses2"]).max() <= 1e-10 * g["losses2"].max()
    assert np.abs(res2.vertices - g["final2"]).max() <= 1e-9


def test_morph_f32_decreases_and_is_deterministic(wv):
    from paper_2407_11272_b200.morph import MorphConfig, morph
    g = golden("morph_traces")
    tmpl = wv.TriangleMesh(g["tmpl_vertices"], g["tmpl_faces"])
    target = wv.ScalarField(wv.GridSpec(*grid_of(g)), g["target"])
    a, ra = morph(tmpl, target, MorphConfig(iterations=10), precision="f32")
    b, rb = morph(tmpl, target, MorphConfig(iterations=10), precision="f32")
    la = [e["loss"] for e in ra.entries]
    assert all(y <= x for x, y in zip(la, la[1:]))
    assert la[-1] < la[0]
    assert a.vertices.tobytes() == b.vertices.tobytes()  # run-to-run bit-identical
    assert abs(la[-1] - g["losses"][-1]) <= 1e-3 * g["losses"][-1]


def test_morph_validation(wv):
    from paper_2407_11272_b200.morph import MorphConfig, morph
    g = golden("morph_traces")
    tmpl = wv.TriangleMesh(g["tmpl_vertices"], g["tmpl_faces"])
    target = wv.ScalarField(wv.GridSpec(*grid_of(g)), g["target"])
    with pytest.raises(ValueError):
        MorphConfig(momentum=1.0)
    with pytest.raises(ValueError):
        morph(wv.TriangleMesh(tmpl.vertices * 10, tmpl.faces), target)
    res, rep = morph(tmpl, target, MorphConfig(iterations=0))
    assert len(rep.entries) == 1 and np.array_equal(res.vertices, tmpl.vertices)


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_criterion_8_morph_demo(cuda_device, precision):
    """The reference's acceptance criterion 8 (test_acceptance.py:305-327):
    morphing icosphere(2, 0.5) onto a cube(0.6) occupancy at 32^3 for 300
    iterations halves the sampled surface Chamfer distance with a
    monotone loss.  The reference needs up to 300 s (286 s recorded,
    test_output.txt:191); the elapsed time here is printed."""
    import time
    import paper_2407_11272_b200 as wv
    from paper_2407_11272_b200 import configs
    h = 0.6
    cv = np.array([[x, y, z] for x in (-h, h) for y in (-h, h) for z in (-h, h)])
    cf = np.array([[0, 2, 3], [0, 3, 1], [4, 5, 7], [4, 7, 6], [0, 1, 5], [0, 5, 4],
                   [2, 6, 7], [2, 7, 3], [0, 4, 6], [0, 6, 2], [1, 3, 7], [1, 7, 5]])
    cube = wv.TriangleMesh(cv, cf[:, [0, 2, 1]])  # outward
    template = wv.TriangleMesh(*configs.icosphere(2, 0.5))
    target = wv.voxelize(cube, wv.GridSpec((-0.75,) * 3, (0.75,) * 3, 32), mode="exact")
    assert abs(wv.winding_number_exact(cube, [0.0, 0.0, 0.0]) - 1.0) < 1e-12

    def chamfer(m):
        return wv.chamfer_distance(wv.sample_surface(m, 20000, seed=0),
                                   wv.sample_surface(cube, 20000, seed=1))

    initial = chamfer(template)
    t0 = time.perf_counter()
    result, report = wv.morph(template, target, wv.MorphConfig(iterations=300),
                              precision=precision)
    elapsed = time.perf_counter() - t0
    final = chamfer(result)
    losses = [e["loss"] for e in report.entries]
    print(f"criterion 8 ({precision}): chamfer {initial:.4f} -> {final:.4f}, {elapsed:.2f} s")
    assert all(b <= a for a, b in zip(losses, losses[1:]))
    assert final <= 0.5 * initial and elapsed < 300.0


def test_morph_graphs_equal_eager_and_faster(wv):
    """The CUDA-graph replay of the evaluations (default) runs the same
    kernels as eager launches: identical traces and vertices, bit for bit.
    The two loops' times at the reference's acceptance size (icosphere(2) ->
    cube, 32^3) are printed (each morph() call captures its graphs anew, so
    short runs include the capture)."""
    import time
    from paper_2407_11272_b200 import configs
    from paper_2407_11272_b200.morph import MorphConfig, morph
    g = golden("morph_traces")
    tmpl = wv.TriangleMesh(g["tmpl_vertices"], g["tmpl_faces"])
    target = wv.ScalarField(wv.GridSpec(*grid_of(g)), g["target"])
    for prec in ("f64", "f32"):
        a, ra = morph(tmpl, target, MorphConfig(iterations=8), precision=prec, graphs=True)
        b, rb = morph(tmpl, target, MorphConfig(iterations=8), precision=prec, graphs=False)
        assert a.vertices.tobytes() == b.vertices.tobytes(), prec
        assert [e["loss"] for e in ra.entries] == [e["loss"] for e in rb.entries], prec
    v, f = configs.icosphere(2, 0.5)
    spec = wv.GridSpec((-1.0,) * 3, (1.0,) * 3, 32)
    nodes = spec.node_coordinates()
    cube = wv.ScalarField(spec, (np.abs(nodes).max(axis=1) < 0.45).astype(np.float64))
    times = {}
    for graphs in (True, False):
        morph(wv.TriangleMesh(v, f), cube, MorphConfig(iterations=3), precision="f32",
              graphs=graphs)
        t0 = time.perf_counter()
        morph(wv.TriangleMesh(v, f), cube, MorphConfig(iterations=60), precision="f32",
              graphs=graphs)
        times[graphs] = time.perf_counter() - t0
    print("morph 60 iterations: graphs %.3f s, eager %.3f s" % (times[True], times[False]))
