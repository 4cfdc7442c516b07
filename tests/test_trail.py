"""Edge trails (wv_edge_trails, host code in the C-ABI library, no GPU) for
the exact backward: evaluating each window edge's two end terms in f64 and
gathering them through the signed CSR must give the face-wise closed-form
exact gradient (the oracle) -- on soups (positions shared,
vertex ids private), index-welded open and closed meshes (interior edges
cancel), and random non-manifold meshes with degenerate and duplicated
faces.  Also: consecutive window positions are edges, every live edge is in
exactly one window, and the build does not depend on the thread count."""

import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2407_11272_b200 import configs


def _trails(v, f, dead=None):
    from paper_2407_11272_b200 import _lib as L
    try:
        L.load_library()
    except L.WindvoxCudaUnavailable:
        pytest.skip("library not built")
    from paper_2407_11272_b200.device import edge_trails
    return edge_trails(v, f, dead)


def _window_terms(v, win, pts, coefs):
    """f64 end terms of every window edge: (W, 2K, 3), slot 2e + end."""
    K = win.shape[1] - 1
    out = np.zeros((len(win), 2 * K, 3))
    for e in range(K):
        P, Q = v[win[:, e]], v[win[:, e + 1]]
        for q, c in zip(pts, coefs):
            a, b = P - q, Q - q
            la, lb = np.linalg.norm(a, axis=1), np.linalg.norm(b, axis=1)
            m = np.cross(a, b)
            den = la * lb + np.einsum("ij,ij->i", a, b)
            s = -c / (4 * np.pi * den)
            out[:, 2 * e] += m * (s / la)[:, None]
            out[:, 2 * e + 1] += m * (s / lb)[:, None]
    return out


def _gather(terms, off, slots, V):
    flat = terms.reshape(-1, 3)
    g = np.zeros((V, 3))
    for vid in range(V):
        for s in slots[off[vid]:off[vid + 1]]:
            g[vid] += flat[s] if s >= 0 else -flat[-s - 1]
    return g


def _case(name):
    if name == "soup":
        return configs.soup(*configs.torus(0.7, 0.3, 14, 10), seed=4)
    if name == "holes":
        return configs.torus_with_holes(16, 12, holes=2, patch=3, seed=1)
    if name == "closed":
        return configs.torus(0.7, 0.3, 12, 8)
    rng = np.random.default_rng(7)
    v = rng.normal(size=(25, 3))
    f = rng.integers(0, 25, size=(70, 3))
    f = np.concatenate([f, f[:5], f[5:8, ::-1], [[0, 0, 3], [4, 5, 4]]])  # dup / flipped / degenerate
    v[24] = v[23]  # two vertex ids at one position
    return v, f


@pytest.mark.parametrize("name", ["soup", "holes", "closed", "random"])
def test_trails_gather_to_the_exact_gradient(name):
    v, f = _case(name)
    dead = np.linalg.norm(np.cross(v[f[:, 1]] - v[f[:, 0]], v[f[:, 2]] - v[f[:, 0]]), axis=1) == 0
    win, off, slots, vrep = _trails(v, f, dead)
    # windows walk edges of the welded graph: consecutive positions differ
    for e in range(win.shape[1] - 1):
        assert not np.any(np.all(v[win[:, e]] == v[win[:, e + 1]], axis=1))
    # representatives share their vertex's position
    assert np.array_equal(v[vrep], v)
    rng = np.random.default_rng(11)
    pts = rng.uniform(-1.3, 1.3, size=(40, 3))
    coefs = rng.normal(size=len(pts))
    g = _gather(_window_terms(v, win, pts, coefs), off, slots, len(v))
    ref = orc.exact_grad(v, f, pts, coefs, threads=1)
    scale = max(np.abs(ref).max(), 1e-300)
    if name == "closed":
        # every interior edge cancels: no window at all, zero gradient
        assert len(win) == 0 and np.abs(g).max() == 0.0
        assert np.abs(ref).max() <= 1e-12
        return
    assert np.abs(g - ref).max() <= 1e-10 * scale, np.abs(g - ref).max() / scale


def test_trails_cover_each_live_edge_once():
    """A closed soup: 1.5 edges per face, each in one window, windows of K
    edges (the trails of a 6-regular position graph are Euler circuits: few
    padded windows)."""
    v, f = configs.soup(*configs.torus(0.7, 0.3, 20, 12), seed=2)
    win, off, slots, _ = _trails(v, f)
    K = win.shape[1] - 1
    E = 3 * len(f) // 2
    assert len(win) * K >= E and len(win) <= E // K + 4
    keys = set()
    pos = {tuple(p): i for i, p in enumerate(np.unique(v, axis=0))}
    for w in win:
        for e in range(K):
            a, b = pos[tuple(v[w[e]])], pos[tuple(v[w[e + 1]])]
            keys.add((min(a, b), max(a, b)))
    assert len(keys) == E
    # every soup vertex gets its two incident face edges' terms
    assert np.array_equal(np.diff(off), np.full(len(v), 2))


def test_trails_independent_of_thread_count():
    code = ("import sys, numpy as np; sys.path.insert(0, %r); "
            "from paper_2407_11272_b200 import configs, device; "
            "v, f = configs.soup(*configs.torus(0.7, 0.3, 30, 20), seed=5); "
            "w, o, s, r = device.edge_trails(v, f); "
            "print(hash((w.tobytes(), o.tobytes(), s.tobytes())))")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    _trails(np.zeros((3, 3)), np.zeros((0, 3), np.int64))
    outs = []
    for t in ("1", "4"):
        env = dict(os.environ, OMP_NUM_THREADS=t, PYTHONHASHSEED="0")
        outs.append(subprocess.run([sys.executable, "-c", code % root], env=env, check=True,
                                   capture_output=True, text=True).stdout.strip())
    assert outs[0] == outs[1]


def test_trails_reject_bad_indices():
    from paper_2407_11272_b200 import _lib as L
    _trails(np.zeros((3, 3)), np.zeros((0, 3), np.int64))
    import ctypes
    lib = L.load_library()
    v = np.zeros((3, 3))
    f = np.array([[0, 1, 3]], dtype=np.int64)
    win = np.empty((3, lib.wv_trail_edges() + 1), np.int64)
    off = np.empty(4, np.int64)
    sl = np.empty(6, np.int64)
    nw, ns = ctypes.c_int64(), ctypes.c_int64()
    rc = lib.wv_edge_trails(v.ctypes.data, 3, f.ctypes.data, 1, None, win.ctypes.data,
                            ctypes.addressof(nw), off.ctypes.data, sl.ctypes.data,
                            ctypes.addressof(ns), None)
    assert rc == 1


def test_host_plan_cache_keys_on_content():
    """The host-plan cache (strip order, trails) is keyed by the mesh bytes:
    a DeviceMesh rebuilt from equal arrays reuses the plan, a moved vertex
    gets its own."""
    import torch
    from paper_2407_11272_b200 import device
    _trails(np.zeros((3, 3)), np.zeros((0, 3), np.int64))
    v, f = configs.soup(*configs.torus(0.7, 0.3, 16, 10), seed=3)

    def mesh(vv):
        m = device.DeviceMesh(torch.from_numpy(vv), torch.from_numpy(f))
        m._verts_np, m._faces_np = vv, f
        return m
    a, b = mesh(v.copy()), mesh(v.copy())
    ta, tb = a.exact_trail_setup(), b.exact_trail_setup()
    assert a._plan_key(a._verts_np) == b._plan_key(b._verts_np)
    assert torch.equal(ta[0], tb[0]) and torch.equal(ta[1][1], tb[1][1])
    v2 = v.copy()
    v2[0, 0] += 1e-3  # splits one weld
    c = mesh(v2)
    assert c._plan_key(v2) != a._plan_key(a._verts_np)
    tc = c.exact_trail_setup()
    assert tc[2] != ta[2] or not torch.equal(tc[1][1], ta[1][1])
