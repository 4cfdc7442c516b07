"""CPU-only tests: the C-ABI library loads and exports every symbol the
public header declares (no compute calls -- there is no GPU here), plus the
host-side logic of the package (types, CSR, exact-gradient edge weights)."""

import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def header_symbols():
    text = (ROOT / "include" / "windvox_b200.h").read_text()
    return sorted(set(re.findall(r"\b(wv_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2407_11272_b200 import _lib
    lib = _lib.load_library()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_lib.EXPORTED) == syms
    assert lib.wv_version().startswith(b"windvox_b200")
    assert lib.wv_status_string(2) == b"workspace missing or too small"


def test_packed_sizes():
    from paper_2407_11272_b200 import _lib
    lib = _lib.load_library()
    assert lib.wv_packed_bytes(1, 10) == 64 + 10 * 64
    assert lib.wv_packed_bytes(2, 10) == 64 + 10 * 32
    assert lib.wv_packed_bytes(3, 10) == 64 + 10 * 128
    assert lib.wv_packed_bytes(7, 10) == 64 + 10 * 64
    assert lib.wv_packed_bytes(9, 10) == 64 + 10 * 64  # strip-ordered exact records
    assert lib.wv_packed_bytes(99, 10) == 0


def test_strip_and_pair_entry_points_validate_before_touching_the_gpu():
    """Argument checks of the strip / pair entry points return WV_ERR_ARG
    (1) without any CUDA call: odd face counts for pairs, bad ranges, null
    buffers."""
    import ctypes
    from paper_2407_11272_b200 import _lib
    lib = _lib.load_library()
    g = _lib.make_grid((-1.0,) * 3, (1.0,) * 3, (4, 4, 4))
    dummy = ctypes.c_void_p(16)
    assert lib.wv_exact_pair_bwd_grid_f32(dummy, 3, g, 0, 8, dummy, 1.0, dummy, None, 0,
                                          None) == 1
    assert lib.wv_exact_pair_bwd_points_f32(dummy, 5, dummy, 8, dummy, 1.0, dummy, None, 0,
                                            None) == 1
    assert lib.wv_exact_pair_bwd_grid_f32(dummy, 2, g, 60, 8, dummy, 1.0, dummy, None, 0,
                                          None) == 1  # range past the 64 nodes
    assert lib.wv_exact_strip_fwd_grid_f32(None, 2, g, 0, 8, 0, dummy, None, None, 0,
                                           None) == 1
    assert lib.wv_pack_exact_strip(dummy, 1, 3, dummy, 1, 1, None, None, None, dummy,
                                   None) == 1
    assert lib.wv_exact_pair_bwd_workspace_bytes(0, 10) == 0


def test_no_cpu_fallback():
    """The product path refuses to run without a CUDA device."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2407_11272_b200 as wv
    from paper_2407_11272_b200._lib import WindvoxCudaUnavailable
    mesh = wv.TriangleMesh(np.eye(3), [[0, 1, 2]])
    with pytest.raises(WindvoxCudaUnavailable):
        wv.voxelize(mesh, wv.GridSpec((-1.0,) * 3, (1.0,) * 3, 4))


def test_types_mirror_reference_validation():
    import paper_2407_11272_b200 as wv
    with pytest.raises(ValueError):
        wv.GridSpec((0.0,) * 3, (0.0, 1.0, 1.0), 4)
    with pytest.raises(ValueError):
        wv.GridSpec((0.0,) * 3, (1.0,) * 3, (4, 0, 4))
    with pytest.raises(ValueError):
        wv.ScalarField(wv.GridSpec((0.0,) * 3, (1.0,) * 3, 2), np.zeros(9))
    with pytest.raises(IndexError):
        wv.TriangleMesh(np.zeros((3, 3)), [[0, 1, 3]])
    with pytest.raises(ValueError):
        wv.QueryBatchConfig(chunk_size=0)
    spec = wv.GridSpec((-1.0, 0.0, 2.0), (1.0, 3.0, 2.5), (3, 4, 2))
    from oracle import oracle as orc
    assert np.array_equal(spec.node_coordinates(),
                          orc.node_coordinates((-1.0, 0.0, 2.0), (1.0, 3.0, 2.5), (3, 4, 2)))
    one = wv.GridSpec((0.0,) * 3, (2.0,) * 3, (1, 1, 3))
    assert np.allclose(one.node_coordinates()[:, :2], 1.0)
    f = wv.binarize(wv.ScalarField(wv.GridSpec((0.0,) * 3, (1.0,) * 3, (1, 1, 3)),
                                   np.array([0.9, 0.1, 0.5])))
    assert f.values.tolist() == [1.0, 0.0, 0.0]


def test_solid_angle_triangle_known_answers():
    import paper_2407_11272_b200 as wv
    assert abs(wv.solid_angle_triangle([1, 0, 0], [0, 1, 0], [0, 0, 1], [0, 0, 0]) - np.pi / 2) < 1e-12
    assert wv.solid_angle_triangle([1, 0, 0], [1, 0, 0], [0, 1, 0], [0.3, 0.1, -2.0]) == 0.0
    assert wv.solid_angle_triangle([0, 0, 0], [1, 0, 0], [0, 1, 0], [3.0, 3.0, 0.0]) == 0.0
    with pytest.raises(wv.OnSurfaceError):
        wv.solid_angle_triangle([0, 0, 0], [1, 0, 0], [0, 1, 0], [0.2, 0.2, 0.0])


def test_vertex_csr_order():
    from paper_2407_11272_b200.device import vertex_csr
    faces = np.array([[0, 1, 2], [2, 1, 3], [3, 0, 2]])
    off, slots = vertex_csr(faces, 5)
    assert off.tolist() == [0, 2, 4, 7, 9, 9]
    for v in range(4):
        s = slots[off[v]:off[v + 1]]
        assert (faces.reshape(-1)[s] == v).all() and (np.diff(s) > 0).all()


def _edge_form_grad(v, faces, pts, coefs, active, w):
    """numpy restatement of the kernels' edge form (test-side)."""
    g = np.zeros_like(v)
    for fi, ww in zip(active, w):
        tri = faces[fi]
        for k in range(3):
            i, j = tri[k], tri[(k + 1) % 3]
            if ww[k] == 0:
                continue
            for q, c in zip(pts, coefs):
                a, b = v[i] - q, v[j] - q
                la, lb = np.linalg.norm(a), np.linalg.norm(b)
                t = -c * ww[k] / (4 * np.pi * (la * lb + a @ b))
                m = np.cross(a, b)
                g[i] += m * t / la
                g[j] += m * t / lb
    return g


@pytest.mark.parametrize("case", ["holes", "soup", "random"])
def test_exact_edge_weights_reproduce_face_closed_form(case):
    from oracle import oracle as orc
    from paper_2407_11272_b200 import configs
    from paper_2407_11272_b200.device import dead_faces, exact_edge_weights
    rng = np.random.default_rng(3)
    if case == "holes":
        v, f = configs.torus_with_holes(nu=16, nv=12, holes=2, patch=2, seed=1)
    elif case == "soup":
        v, f = configs.soup(*configs.torus(0.7, 0.3, 8, 6))
    else:
        v = rng.normal(size=(12, 3))
        f = rng.integers(0, 12, size=(20, 3))
        f[0] = [4, 4, 5]  # degenerate (dropped by the reference forward)
    pts = rng.normal(size=(6, 3)) * 1.3
    coefs = rng.normal(size=6)
    active, w = exact_edge_weights(f, dead_faces(v, f))
    got = _edge_form_grad(v, f, pts, coefs, active, w)
    ref = orc.exact_grad(v, f, pts, coefs)
    assert np.abs(got - ref).max() <= 1e-10 * max(np.abs(ref).max(), 1e-12)
    if case == "holes":
        assert len(active) < len(f) // 2


def test_wvox1_bytes_match_reference(tmp_path):
    """WVOX1 writer reproduces the reference's bytes (golden) and round-trips."""
    import paper_2407_11272_b200 as wv
    from conftest import golden
    g = golden("openmesh_and_io")
    spec = wv.GridSpec((-1.0, 0.0, 0.5), (1.0, 2.0, 0.75), (4, 3, 5))
    f64 = wv.ScalarField(spec, g["field_values"])
    wv.save_field(f64, tmp_path / "a.wvox")
    assert (tmp_path / "a.wvox").read_bytes() == g["wvox_f64"].tobytes()
    wv.save_field(wv.ScalarField(spec, g["field_values"].astype(np.float32)), tmp_path / "b.wvox")
    assert (tmp_path / "b.wvox").read_bytes() == g["wvox_f32"].tobytes()
    back = wv.load_field(tmp_path / "a.wvox")
    assert back.spec == spec and back.values.tobytes() == f64.values.tobytes()
    bad = tmp_path / "bad.wvox"
    bad.write_bytes(g["wvox_f64"].tobytes().replace(b"WVOX1", b"WVOX9", 1))
    with pytest.raises(wv.ParseError):
        wv.load_field(bad)
    short = tmp_path / "short.wvox"
    short.write_bytes(g["wvox_f64"].tobytes()[:-8])
    with pytest.raises(wv.ParseError):
        wv.load_field(short)


def test_uniform_laplacian_matches_definition():
    from paper_2407_11272_b200 import configs
    from paper_2407_11272_b200.morph import uniform_laplacian
    v, f = configs.icosphere(1, 0.5)
    ip, ix, d = uniform_laplacian(f, len(v))
    dense = np.zeros((len(v), len(v)))
    for r in range(len(v)):
        dense[r, ix[ip[r]:ip[r + 1]]] += d[ip[r]:ip[r + 1]]
    assert np.allclose(dense.sum(axis=1), 0.0)  # rows of I - D^-1 A sum to 0
    assert np.allclose(np.diag(dense), 1.0)


def test_bench_metric_is_baseline_metric():
    """Both bench arms print BASELINE.json's metric and one unit, so the
    driver can pair the lines (round-1 verdict: they differed)."""
    import json
    import bench
    base = json.loads((ROOT / "BASELINE.json").read_text())
    assert bench.METRIC == base["metric"]
    assert bench.UNIT == "pairs/s"


def test_random_soup_config_and_path_choice():
    """C3's stress variant: 100k independent equilateral-ish triangles
    (edge 0.04-0.06, centres in [-0.8,0.8]^3) share no corner position, so the
    automatic choice takes the face-ordered kernels; the welded C3 soup takes
    the strip forward and the edge-trail backward (host-side decision, no GPU
    needed)."""
    import torch
    from paper_2407_11272_b200 import configs, device
    w = configs.make("c3r")
    assert w.n_faces == 100_000 and w.res == (256, 256, 256)
    t = w.vertices.reshape(-1, 3, 3)
    e = np.linalg.norm(t[:, 1] - t[:, 0], axis=1)
    assert 0.0399 < e.min() and e.max() < 0.0601
    c = t.mean(axis=1)
    assert np.abs(c).max() <= 0.8
    for name, pay in (("c3r", False), ("c3", True)):
        w = configs.make(name)
        m = device.DeviceMesh(torch.from_numpy(w.vertices), torch.from_numpy(w.faces))
        m._verts_np, m._faces_np = w.vertices, w.faces
        assert m.strips_pay() is pay, name
        grid = (w.lo, w.hi, w.res)
        assert device.lattice_paths(m, "exact", "f32", grid, 0, w.n_nodes) == (pay, pay)
        assert device.lattice_paths(m, "exact", "f64", grid, 0, w.n_nodes) == (pay, False)
        # the exact f32 backward: edge trails where corner positions are shared
        assert device.backward_path(m, "exact", "f32", grid, 0, w.n_nodes) == \
            ("trails" if pay else "faces")
        assert device.backward_path(m, "exact", "f64", grid, 0, w.n_nodes) == \
            ("trails" if pay else "faces")
        assert device.backward_path(m, "soft", "f32", grid, 0, w.n_nodes) == "soft"
    # a mesh reaching far beyond the lattice keeps the face kernels (the trail
    # kernel's four-fold denominator product must stay inside f32 range)
    w = configs.make("c3")
    m = device.DeviceMesh(torch.from_numpy(w.vertices), torch.from_numpy(w.faces))
    m._verts_np, m._faces_np = w.vertices, w.faces
    small = ((-1e-4,) * 3, (1e-4,) * 3, w.res)
    assert device.backward_path(m, "exact", "f32", small, 0, w.n_nodes) == "pairs"
