"""Reconstruction metrics on the device vs the reference
(metrics.py), bit for bit: SplitMix64 streams, area-weighted surface samples,
nearest distances, numpy-order pairwise sums, Chamfer / Hausdorff,
evaluate_reconstruction; and the reference's error behaviour
(test_metrics.py)."""

import numpy as np
import pytest

from conftest import golden
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M(cuda_device):
    from paper_2407_11272_b200 import metrics
    return metrics


@pytest.fixture(scope="module")
def g():
    return golden("metrics")


def mesh(g, name):
    import paper_2407_11272_b200 as wv
    return wv.TriangleMesh(g[f"{name}_vertices"], g[f"{name}_faces"])


def test_splitmix_bit_exact(M, g):
    assert np.array_equal(M.splitmix64_uniform(7, 10000), g["u_seed7"])
    assert np.array_equal(M.splitmix64_uniform((1 << 64) - 3, 999), g["u_seed_big"])
    assert np.array_equal(M.splitmix64_uniform(-5, 300), orc.splitmix64_uniform(-5, 300))
    assert M.splitmix64_uniform(3, 0).shape == (0,)


def test_samples_bit_exact(M, g):
    assert M.sample_surface(mesh(g, "ico"), 4001, seed=3).tobytes() == g["s_ico"].tobytes()
    # zero-area faces are never chosen (test_metrics.py:102-106)
    s = M.sample_surface(mesh(g, "degen"), 2000, seed=11)
    assert s.tobytes() == g["s_degen"].tobytes() and np.abs(s).max() <= 1.0
    # samples lie on the surface of the cube (test_metrics.py:96-99)
    c = M.sample_surface(mesh(g, "cube"), 5000, seed=2)
    assert np.isclose(np.abs(c).max(axis=1), 0.5).all()


def test_distances_bit_exact(M, g):
    import torch
    from paper_2407_11272_b200.metrics import nearest_distances, _pairwise_sum
    d = nearest_distances(torch.as_tensor(g["pa"]).cuda(), torch.as_tensor(g["pb"]).cuda())
    assert d.cpu().numpy().tobytes() == g["nn_ab"].tobytes()
    assert M.chamfer_distance(g["pa"], g["pb"]) == float(g["chamfer_ab"])
    assert M.hausdorff_distance(g["pa"], g["pb"]) == float(g["hausdorff_ab"])
    assert M.chamfer_distance(g["pa"], g["pb"]) == M.chamfer_distance(g["pb"], g["pa"])
    # numpy's pairwise summation order, every leaf/tail shape
    from test_oracle_golden import big_vector
    big = big_vector()
    assert float(_pairwise_sum(torch.as_tensor(big).cuda()).item()) == float(g["big_sum"])
    rng = np.random.default_rng(4)
    for n in list(range(1, 140)) + [255, 256, 257, 1000, 4097]:
        x = rng.normal(size=n) * 10.0 ** rng.integers(-4, 4, size=n)
        assert float(_pairwise_sum(torch.as_tensor(x).cuda()).item()) == float(np.sum(x)), n
    # trivial values (test_metrics.py:112-118)
    a = np.zeros((1, 3))
    b = np.array([[1.0, 0.0, 0.0]])
    assert M.chamfer_distance(a, a) == 0.0 and M.chamfer_distance(a, b) == 1.0
    assert M.hausdorff_distance(a, a) == 0.0 and M.hausdorff_distance(a, b) == 1.0


def test_evaluate_reconstruction_bit_exact(M, g):
    r = M.evaluate_reconstruction(mesh(g, "ico"), mesh(g, "cube"), n=3000, repeats=3, seed=5)
    got = np.array([r["chamfer_mean"], r["chamfer_std"], r["hausdorff_mean"],
                    r["hausdorff_std"]])
    assert got.tobytes() == g["recon"].tobytes()
    same = M.evaluate_reconstruction(mesh(g, "ico"), mesh(g, "ico"), n=2000, repeats=2)
    assert same == {"chamfer_mean": 0.0, "chamfer_std": 0.0, "hausdorff_mean": 0.0,
                    "hausdorff_std": 0.0}


def test_metric_errors(M, g):
    import paper_2407_11272_b200 as wv
    from paper_2407_11272_b200.errors import DegenerateError
    ico = mesh(g, "ico")
    with pytest.raises(ValueError):
        M.sample_surface(ico, -1, seed=0)
    assert M.sample_surface(ico, 0, seed=0).shape == (0, 3)
    with pytest.raises(DegenerateError):
        M.sample_surface(wv.TriangleMesh(np.zeros((0, 3)), np.zeros((0, 3), np.int64)), 5, 0)
    flat = wv.TriangleMesh(np.array([[0.0, 0, 0], [1, 0, 0], [2, 0, 0]]), np.array([[0, 1, 2]]))
    with pytest.raises(DegenerateError):
        M.sample_surface(flat, 5, seed=0)
    with pytest.raises(ValueError):
        M.chamfer_distance(np.zeros((0, 3)), np.zeros((4, 3)))
    with pytest.raises(ValueError):
        M.hausdorff_distance(np.zeros((4, 3)), np.zeros((0, 3)))
    with pytest.raises(ValueError):
        M.evaluate_reconstruction(ico, ico, repeats=0)
