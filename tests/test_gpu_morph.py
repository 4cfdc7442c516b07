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
