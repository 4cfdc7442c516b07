"""Face strips (wv_strip_order, host code in the C-ABI library, no GPU): the
order is a permutation of the faces, every window is its face's vertex set,
consecutive windows of a strip share two corner POSITIONS (the forward
carries their distances), and the reflection flag is the parity of the
window against the face's own vertex order (the fp64 rare path restores the
orientation from it)."""

import numpy as np
import pytest

from paper_2407_11272_b200 import configs


def _strips(v, f):
    from paper_2407_11272_b200 import _lib as L
    try:
        L.load_library()
    except L.WindvoxCudaUnavailable:
        pytest.skip("library not built")
    from paper_2407_11272_b200.device import strip_order
    return strip_order(v, f)


def _check(v, f, max_restart_frac):
    perm, win, fl = _strips(v, f)
    F = len(f)
    assert np.array_equal(np.sort(perm), np.arange(F))
    assert np.array_equal(np.sort(win, axis=1), np.sort(f[perm], axis=1))
    restart = (fl & 1).astype(bool)
    assert restart[0]
    k = np.flatnonzero(~restart)
    assert np.array_equal(v[win[k, 0]], v[win[k - 1, 1]])
    assert np.array_equal(v[win[k, 1]], v[win[k - 1, 2]])
    # parity: window (A,B,C) is a rotation of the face's order iff bit1 clear
    fo = f[perm]
    pos = np.stack([np.argmax(fo == win[:, c:c + 1], axis=1) for c in range(3)], axis=1)
    even = ((pos[:, 1] - pos[:, 0]) % 3 == 1) & ((pos[:, 2] - pos[:, 1]) % 3 == 1)
    assert np.array_equal(even, (fl & 2) == 0)
    assert restart.mean() <= max_restart_frac, restart.mean()
    return restart.mean()


def test_strips_welded_torus():
    v, f = configs.torus(0.7, 0.3, 48, 24)
    _check(v, f, 0.05)


def test_strips_shuffled_soup_welds_by_position():
    v, f = configs.soup(*configs.torus(0.7, 0.3, 40, 30), seed=3)
    assert len(v) == 3 * len(f)  # private vertices: only positions are shared
    _check(v, f, 0.08)


def test_strips_degenerate_and_open_meshes():
    v, f = configs.icosphere(2)
    f = np.concatenate([f[:50], [[0, 0, 1], [2, 3, 3]], f[60:]])  # open + degenerate faces
    _check(v, f, 0.5)
    rng = np.random.default_rng(0)
    v = rng.normal(size=(30, 3))
    f = rng.integers(0, 30, size=(80, 3))
    _check(v, f, 1.0)


def test_strip_order_rejects_bad_indices():
    from paper_2407_11272_b200 import _lib as L
    try:
        lib = L.load_library()
    except L.WindvoxCudaUnavailable:
        pytest.skip("library not built")
    v = np.zeros((3, 3))
    f = np.array([[0, 1, 3]], dtype=np.int64)
    out = [np.empty(1, np.int64), np.empty(3, np.int64), np.empty(1, np.uint8)]
    rc = lib.wv_strip_order(v.ctypes.data, 3, f.ctypes.data, 1, *(a.ctypes.data for a in out))
    assert rc == L.WV_ERR_ARG if hasattr(L, "WV_ERR_ARG") else rc == 1


def _edge_weight_sums(rows, weights):
    acc = {}
    for (a, b, c), w in zip(rows, weights):
        for (p, q), x in zip(((a, b), (b, c), (c, a)), w):
            if x == 0:
                continue
            k = (min(p, q), max(p, q))
            acc[k] = acc.get(k, 0.0) + (x if p < q else -x)
    return {k: v for k, v in acc.items() if v != 0}


@pytest.mark.parametrize("case", ["soup", "open_welded", "random"])
def test_strip_pairs_preserve_edge_weights(case):
    """strip_pairs (the exact backward's pair rows): every active face
    appears once among the valid rows, pairs share two corner positions, and
    the directed-edge weights (window order, negated for reflected windows)
    sum to the same net per-edge weights as the original faces."""
    from paper_2407_11272_b200 import device
    _strips(np.zeros((3, 3)), np.zeros((0, 3), np.int64))  # skips if the library is absent
    if case == "soup":
        v, f = configs.soup(*configs.torus(0.7, 0.3, 24, 16), seed=4)
    elif case == "open_welded":
        v, f = configs.torus(0.7, 0.3, 30, 20)
        f = f[: len(f) - 37]
    else:
        rng = np.random.default_rng(3)
        v = rng.normal(size=(25, 3))
        f = rng.integers(0, 25, size=(70, 3))
    active, w = device.exact_edge_weights(f, device.dead_faces(v, f))
    rows, rw, valid = device.strip_pairs(v, f[active], w)
    assert len(rows) % 2 == 0 and valid[0::2].all()
    assert np.array_equal(v[rows[1::2, 0]], v[rows[0::2, 1]])
    assert np.array_equal(v[rows[1::2, 1]], v[rows[0::2, 2]])
    got = np.sort(np.sort(rows[valid], axis=1), axis=0)
    ref = np.sort(np.sort(f[active], axis=1), axis=0)
    assert np.array_equal(got, ref)
    assert not rw[~valid].any()
    assert _edge_weight_sums(rows[valid], rw[valid]) == _edge_weight_sums(f[active], w)
    if case == "soup":
        assert valid.mean() > 0.9  # nearly every row is a real pair member
    off, slots = device.vertex_csr_rows(rows, valid, len(v))
    assert off[-1] == 3 * valid.sum() and np.all(valid[slots // 3])


def test_strip_pairs_reuse_the_forward_order():
    """strip_pairs with a precomputed strip_order (the forward's, reused for
    soups whose faces are all active) gives the same rows."""
    from paper_2407_11272_b200 import device
    _strips(np.zeros((3, 3)), np.zeros((0, 3), np.int64))
    v, f = configs.soup(*configs.torus(0.7, 0.3, 20, 12), seed=5)
    active, w = device.exact_edge_weights(f, device.dead_faces(v, f))
    assert np.array_equal(active, np.arange(len(f)))
    a = device.strip_pairs(v, f, w)
    b = device.strip_pairs(v, f, w, device.strip_order(v, f))
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_strip_order_independent_of_thread_count():
    """The builder's sorts run on all host cores (__gnu_parallel::sort); both
    comparators are total orders, so the strips must not depend on the
    OpenMP thread count (wv_strip.cu)."""
    import ctypes
    v, f = configs.soup(*configs.torus(0.7, 0.3, 120, 80), seed=7)  # 19,200 faces
    gomp = ctypes.CDLL("libgomp.so.1")
    default = gomp.omp_get_max_threads()
    ref = None
    try:
        for n in (1, 2, 3, 8):
            gomp.omp_set_num_threads(n)
            got = _strips(v, f)
            if ref is None:
                ref = got
            for a, b in zip(ref, got):
                assert np.array_equal(a, b), n
    finally:
        gomp.omp_set_num_threads(default)
