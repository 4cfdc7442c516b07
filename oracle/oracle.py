"""CPU oracle for the winding-number hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module, and
only as the checker or the timed CPU baseline -- never as the thing measured
or shipped.  The product package (``paper_2407_11272_b200``) does not import
it and has no CPU fallback.

It wraps ``windvox_oracle.c`` (a bit-exact C restatement of the reference
numba kernels, /root/reference/pkg/src/windvox/_kernels.py) and restates in
numpy the reference host-side staging it needs:

* ``surface_epsilon``     <- winding.py:193-197 (+ mesh_io.py:86-88)
* ``prepare_exact``       <- winding.py:258-268
* ``node_coordinates``    <- winding.py:118-140 (GridSpec.axis_nodes / node_coordinates)
* ``winding_number_batch``<- winding.py:271-309
* ``voxelize``            <- winding.py:336-387 (incl. the f32 branch)
* ``occupancy_loss_grad`` <- grad.py:71-127
* ``exact_loss_grad``     <- NEW (exact d(Omega)/dv), same
                             loss definition with the exact forward.
* ``splitmix64_uniform``, ``sample_surface``, ``nearest_distances``,
  ``chamfer_distance``, ``hausdorff_distance`` <- metrics.py:43-130
                             (reconstruction metrics).

Parity is pinned: ``tests/test_oracle_golden.py`` checks every function here
bit-for-bit against fixtures produced by importing the reference itself
(``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "libwvoracle.so"
SURFACE_EPS_FACTOR = 1e-9
_lib = None


def build() -> Path:
    """Compile the C oracle (gcc, -ffp-contract=off) into oracle/_build/."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        build()
    lib = ctypes.CDLL(str(_LIB_PATH))
    P = ctypes.c_void_p
    I64 = ctypes.c_int64
    D = ctypes.c_double
    F = ctypes.c_float
    I = ctypes.c_int
    lib.wvo_exact_batch.argtypes = [P, I64, P, P, P, I64, D, I, P, P]
    lib.wvo_soft_batch.argtypes = [P, I64, P, I64, D, P, P]
    lib.wvo_soft_grad_accum.argtypes = [P, P, I64, P, P, I64, D, P]
    lib.wvo_exact_grad_accum.argtypes = [P, P, I64, P, P, P, P, I64, D, P]
    lib.wvo_exact_batch_f32.argtypes = [P, I64, P, P, P, I64, F, P, P]
    lib.wvo_soft_batch_f32.argtypes = [P, I64, P, I64, F, P, P]
    lib.wvo_exact_batch_mt.argtypes = [P, I64, P, P, P, I64, D, I, P, P, I64, I]
    lib.wvo_soft_batch_mt.argtypes = [P, I64, P, I64, D, P, P, I64, I]
    lib.wvo_soft_grad_mt.argtypes = [P, P, I64, P, P, I64, I64, D, P, I64, I]
    lib.wvo_exact_grad_mt.argtypes = [P, P, I64, P, P, P, P, I64, I64, D, P, I64, I]
    for name in ("wvo_exact_batch_mt", "wvo_soft_batch_mt", "wvo_soft_grad_mt",
                 "wvo_exact_grad_mt"):
        getattr(lib, name).restype = I
    _lib = lib
    return lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=dtype))


def default_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return max(1, os.cpu_count() or 1)


# ---------------------------------------------------------------------------
# host-side staging (numpy restatements of the reference)

def surface_epsilon(vertices: np.ndarray) -> float:
    """winding.py:193-197: 1e-9 * bbox diagonal (0 for an empty mesh)."""
    v = np.asarray(vertices, dtype=np.float64).reshape(-1, 3)
    if len(v) == 0:
        return 0.0
    return SURFACE_EPS_FACTOR * float(np.linalg.norm(v.max(axis=0) - v.min(axis=0)))


def triangle_corners(vertices, faces) -> np.ndarray:
    """mesh_io.py:90-92."""
    v = _c(vertices, np.float64).reshape(-1, 3)
    f = _c(faces, np.int64).reshape(-1, 3)
    return v[f]


def prepare_exact(vertices, faces):
    """winding.py:258-268: drop |N|==0 faces, unit normals, plane offsets.
    Also returns the kept face index rows (needed by the gradient)."""
    f = _c(faces, np.int64).reshape(-1, 3)
    tri = triangle_corners(vertices, f)
    cross = np.cross(tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0])
    norm = np.linalg.norm(cross, axis=1)
    keep = norm > 0.0
    tri = np.ascontiguousarray(tri[keep])
    nhat = cross[keep] / norm[keep, None]
    pld = (nhat * tri[:, 0]).sum(axis=1) if len(tri) else np.zeros(0)
    return tri, np.ascontiguousarray(nhat), np.ascontiguousarray(pld), \
        np.ascontiguousarray(f[keep])


def axis_nodes(lo: float, hi: float, r: int) -> np.ndarray:
    """winding.py:118-125."""
    if r == 1:
        return np.array([(lo + hi) / 2.0])
    return lo + (hi - lo) * (np.arange(r, dtype=np.float64) / (r - 1))


def node_coordinates(bounds_min, bounds_max, resolution) -> np.ndarray:
    """winding.py:135-140: (N,3) f64, flat order k fastest."""
    lo = np.asarray(bounds_min, dtype=np.float64).reshape(3)
    hi = np.asarray(bounds_max, dtype=np.float64).reshape(3)
    res = (int(resolution),) * 3 if np.ndim(resolution) == 0 else tuple(int(r) for r in resolution)
    gx, gy, gz = (axis_nodes(lo[a], hi[a], res[a]) for a in range(3))
    xx, yy, zz = np.meshgrid(gx, gy, gz, indexing="ij")
    return np.ascontiguousarray(np.stack([xx, yy, zz], axis=-1).reshape(-1, 3))


# ---------------------------------------------------------------------------
# kernels

def winding_number_batch(vertices, faces, points, mode="exact", use_atan2=True,
                         chunk=2000, threads=None):
    """winding.py:271-309 -> (values f64, flags bool)."""
    lib = _load()
    pts = _c(points, np.float64).reshape(-1, 3)
    n = len(pts)
    out = np.zeros(n, dtype=np.float64)
    flags = np.zeros(n, dtype=np.uint8)
    eps = surface_epsilon(vertices)
    threads = threads or default_threads()
    if mode == "exact":
        tri, nhat, pld, _ = prepare_exact(vertices, faces)
        lib.wvo_exact_batch_mt(_p(pts), n, _p(tri), _p(nhat), _p(pld), len(tri),
                               eps, int(bool(use_atan2)), _p(out), _p(flags),
                               int(chunk), int(threads))
    elif mode == "soft":
        if not use_atan2:
            raise ValueError("the arctan demonstration path only exists in exact mode")
        tri = _c(triangle_corners(vertices, faces), np.float64)
        lib.wvo_soft_batch_mt(_p(pts), n, _p(tri), len(tri), eps, _p(out),
                              _p(flags), int(chunk), int(threads))
    else:
        raise ValueError(f"mode must be 'exact' or 'soft', got {mode!r}")
    return out, flags.astype(bool)


def voxelize_f32(vertices, faces, points, mode="exact"):
    """winding.py:362-387 (single-threaded; results do not depend on threads)."""
    lib = _load()
    pts = _c(np.asarray(points, dtype=np.float64).astype(np.float32), np.float32).reshape(-1, 3)
    n = len(pts)
    out = np.zeros(n, dtype=np.float32)
    flags = np.zeros(n, dtype=np.uint8)
    eps = np.float32(surface_epsilon(vertices))
    if mode == "exact":
        tri, nhat, pld, _ = prepare_exact(vertices, faces)
        tri32, nhat32, pld32 = (_c(a.astype(np.float32), np.float32) for a in (tri, nhat, pld))
        lib.wvo_exact_batch_f32(_p(pts), n, _p(tri32), _p(nhat32), _p(pld32),
                                len(tri32), float(eps), _p(out), _p(flags))
    else:
        tri32 = _c(triangle_corners(vertices, faces).astype(np.float32), np.float32)
        lib.wvo_soft_batch_f32(_p(pts), n, _p(tri32), len(tri32), float(eps),
                               _p(out), _p(flags))
    out[flags.astype(bool)] = 0.5
    return out, flags.astype(bool)


def voxelize(vertices, faces, points, mode="exact", precision="f64", threads=None):
    """winding.py:336-359: flagged nodes -> exactly 0.5."""
    if precision == "f32":
        return voxelize_f32(vertices, faces, points, mode)
    values, flags = winding_number_batch(vertices, faces, points, mode=mode, threads=threads)
    values[flags] = 0.5
    return values, flags


def soft_grad(vertices, faces, points, coefs, chunk=2000, threads=None):
    """soft_grad_accum through run_chunked with per-chunk buffers merged in
    chunk order (grad.py:111-127).  Returns (V,3) f64."""
    lib = _load()
    v = _c(vertices, np.float64).reshape(-1, 3)
    f = _c(faces, np.int64).reshape(-1, 3)
    pts = _c(points, np.float64).reshape(-1, 3)
    cf = _c(coefs, np.float64).reshape(-1)
    tri = _c(v[f], np.float64)
    grad = np.zeros((len(v), 3), dtype=np.float64)
    rc = lib.wvo_soft_grad_mt(_p(pts), _p(cf), len(pts), _p(tri), _p(f), len(f),
                              len(v), surface_epsilon(v), _p(grad), int(chunk),
                              int(threads or default_threads()))
    if rc != 0:
        raise MemoryError("oracle soft_grad: chunk buffers")
    return grad


def exact_grad(vertices, faces, points, coefs, chunk=2000, threads=None):
    """Closed-form sum_p coefs[p] * dW_exact(p)/dV, (V,3) f64."""
    lib = _load()
    v = _c(vertices, np.float64).reshape(-1, 3)
    pts = _c(points, np.float64).reshape(-1, 3)
    cf = _c(coefs, np.float64).reshape(-1)
    tri, nhat, pld, fk = prepare_exact(v, faces)
    grad = np.zeros((len(v), 3), dtype=np.float64)
    rc = lib.wvo_exact_grad_mt(_p(pts), _p(cf), len(pts), _p(tri), _p(nhat), _p(pld),
                               _p(fk), len(fk), len(v), surface_epsilon(v), _p(grad),
                               int(chunk), int(threads or default_threads()))
    if rc != 0:
        raise MemoryError("oracle exact_grad: chunk buffers")
    return grad


def _loss_terms(values, flags, targets, weights):
    n = len(values)
    t = np.asarray(targets, dtype=np.float64).reshape(n)
    w = np.ones(n) if weights is None else np.asarray(weights, dtype=np.float64).reshape(n)
    if np.any(w < 0):
        raise ValueError("weights must be non-negative")
    included = ~flags
    wsum = float(w[included].sum())
    if wsum == 0.0:
        raise ValueError("no usable grid nodes: all excluded or zero-weighted")
    residual = np.where(included, values - t, 0.0)
    loss = float((w * residual * residual).sum() / wsum)
    coefs = np.ascontiguousarray(2.0 * w * residual / wsum)
    return loss, coefs


def occupancy_loss_grad(vertices, faces, points, targets, weights=None, chunk=2000,
                        threads=None):
    """grad.py:71-127 -> (loss, grads (V,3), excluded_nodes)."""
    if len(np.asarray(faces).reshape(-1, 3)) == 0:
        raise ValueError("cannot evaluate occupancy loss for an empty mesh")
    values, flags = winding_number_batch(vertices, faces, points, mode="soft",
                                         chunk=chunk, threads=threads)
    loss, coefs = _loss_terms(values, flags, targets, weights)
    grads = soft_grad(vertices, faces, points, coefs, chunk=chunk, threads=threads)
    return loss, grads, int(flags.sum())


def exact_loss_grad(vertices, faces, points, targets, weights=None, chunk=2000,
                    threads=None):
    """Same loss with the exact forward and the exact closed-form gradient."""
    values, flags = winding_number_batch(vertices, faces, points, mode="exact",
                                         chunk=chunk, threads=threads)
    loss, coefs = _loss_terms(values, flags, targets, weights)
    grads = exact_grad(vertices, faces, points, coefs, chunk=chunk, threads=threads)
    return loss, grads, int(flags.sum())


def solid_angle_fd_grad(vertices, faces, points, coefs, h=1e-6):
    """Central finite differences of sum_p coefs[p]*W_exact(p) w.r.t. every
    vertex coordinate (the package's own authority for gradients,
    test_grad.py:3-6).  Small meshes only."""
    v = _c(vertices, np.float64).reshape(-1, 3)
    cf = _c(coefs, np.float64).reshape(-1)
    out = np.zeros_like(v)
    for vi in range(len(v)):
        for c in range(3):
            vp = v.copy()
            vp[vi, c] += h
            vm = v.copy()
            vm[vi, c] -= h
            wp, _ = winding_number_batch(vp, faces, points, threads=1)
            wm, _ = winding_number_batch(vm, faces, points, threads=1)
            out[vi, c] = float(((wp - wm) * cf).sum()) / (2 * h)
    return out


# ---------------------------------------------------------------------------
# reconstruction metrics (metrics.py:43-130)

_SM_GOLD = np.uint64(0x9E3779B97F4A7C15)
_SM_M1 = np.uint64(0xBF58476D1CE4E5B9)
_SM_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64_uniform(seed: int, count: int) -> np.ndarray:
    """metrics.py:43-51: counter-based SplitMix64, top 53 bits -> [0, 1)."""
    i = np.arange(1, int(count) + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(int(seed) & ((1 << 64) - 1)) + i * _SM_GOLD
        z = (z ^ (z >> np.uint64(30))) * _SM_M1
        z = (z ^ (z >> np.uint64(27))) * _SM_M2
    z ^= z >> np.uint64(31)
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def sample_surface(vertices, faces, n: int, seed: int) -> np.ndarray:
    """metrics.py:58-93: faces by area (searchsorted on the cumulative
    areas, side="right"), folded uniform barycentrics."""
    tri = triangle_corners(vertices, faces)
    e1, e2 = tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0]
    areas = 0.5 * np.sqrt((np.cross(e1, e2) ** 2).sum(axis=1))
    total = float(areas.sum())
    r = splitmix64_uniform(seed, 3 * int(n))
    face = np.minimum(np.searchsorted(np.cumsum(areas), r[0::3] * total, side="right"),
                      len(areas) - 1)
    u, v = r[1::3].copy(), r[2::3].copy()
    flip = u + v > 1.0
    u[flip], v[flip] = 1.0 - u[flip], 1.0 - v[flip]
    c = tri[face]
    return (c[:, 0] + u[:, None] * (c[:, 1] - c[:, 0])) + v[:, None] * (c[:, 2] - c[:, 0])


def nearest_distances(q, t, block: int = 512) -> np.ndarray:
    """Brute-force nearest distances (the scan metrics.py:96-104 equals)."""
    q = _c(q, np.float64).reshape(-1, 3)
    t = _c(t, np.float64).reshape(-1, 3)
    out = np.empty(len(q))
    for s in range(0, len(q), block):
        d = q[s:s + block, None, :] - t[None, :, :]
        out[s:s + block] = np.sqrt((d * d).sum(axis=2).min(axis=1))
    return out


def chamfer_distance(a, b) -> float:
    return 0.5 * (float(nearest_distances(a, b).mean()) + float(nearest_distances(b, a).mean()))


def hausdorff_distance(a, b) -> float:
    return max(float(nearest_distances(a, b).max()), float(nearest_distances(b, a).max()))
