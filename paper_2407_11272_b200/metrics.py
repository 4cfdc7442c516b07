"""Reconstruction quality on the device: area-weighted
surface sampling with the counter-based SplitMix64 stream, and sampled
Chamfer / Hausdorff distances.

Mirrors /root/reference/pkg/src/windvox/metrics.py (same names, arguments,
conventions and errors):

* ``splitmix64_uniform`` (metrics.py:43-51), ``sample_surface`` (:58-93),
  ``chamfer_distance`` (:111-119: 0.5 * (mean_a min_b |a-b| + mean_b min_a
  |a-b|), Euclidean, not squared), ``hausdorff_distance`` (:122-130),
  ``evaluate_reconstruction`` (:133-150: ``repeats`` draws of ``n`` samples
  per mesh with seed ``seed + r``, population std).

Every value is computed by the kernels of ``csrc/wv_metrics.cu`` in the
reference's IEEE operation order (numpy's cross/norm/cumsum/pairwise-sum
orders, the brute-force distance the reference's k-d tree is tested to
equal), so results are bit-identical to the reference's.  Only the final
scalar combination (two means, two maxima, the statistics over repeats) is
host arithmetic, exactly as in the reference.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from .device import _ptr, _stream, device
from .errors import DegenerateError
from .types import TriangleMesh

__all__ = [
    "splitmix64_uniform", "sample_surface", "chamfer_distance", "hausdorff_distance",
    "evaluate_reconstruction", "sample_surface_device", "nearest_distances",
]

_MASK = (1 << 64) - 1


def splitmix64_uniform(seed: int, count: int) -> np.ndarray:
    """``count`` uniforms in [0, 1): value i mixes the counter seed + (i+1)."""
    count = int(count)
    if count < 0:
        raise ValueError("count must be >= 0")
    lib = L.lib()
    out = torch.empty(count, dtype=torch.float64, device=device())
    L.check(lib.wv_splitmix64_uniform(int(seed) & _MASK, count, _ptr(out), _stream()),
            "wv_splitmix64_uniform")
    return out.cpu().numpy()


def _pairwise_sum(x: torch.Tensor) -> torch.Tensor:
    """np.sum(x) (pairwise order) as a 1-element device tensor."""
    lib = L.lib()
    n = int(x.numel())
    out = torch.empty(1, dtype=torch.float64, device=x.device)
    wsb = int(lib.wv_pairwise_sum_workspace_bytes(n))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=x.device)
    L.check(lib.wv_pairwise_sum(_ptr(x), n, _ptr(out), _ptr(ws), wsb, _stream()),
            "wv_pairwise_sum")
    return out


def sample_surface_device(vertices: torch.Tensor, faces: torch.Tensor, n: int,
                          seed: int) -> torch.Tensor:
    """(n,3) f64 device samples of the surface (vertices (V,3) f64, faces
    (F,3) int64, both on the device).  Raises like ``sample_surface``."""
    n = int(n)
    if n < 0:
        raise ValueError("sample count must be >= 0")
    dev = vertices.device
    if n == 0:
        return torch.zeros((0, 3), dtype=torch.float64, device=dev)
    F = int(faces.shape[0])
    if F == 0:
        raise DegenerateError("mesh has no faces to sample")
    lib = L.lib()
    v = vertices.to(torch.float64).contiguous()
    f = faces.to(torch.int64).contiguous()
    areas = torch.empty(F, dtype=torch.float64, device=dev)
    cdf = torch.empty(F, dtype=torch.float64, device=dev)
    total = torch.empty(1, dtype=torch.float64, device=dev)
    wsb = int(lib.wv_pairwise_sum_workspace_bytes(F))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    st = _stream()
    L.check(lib.wv_surface_cdf(_ptr(v), _ptr(f), F, _ptr(areas), _ptr(cdf), _ptr(total),
                               _ptr(ws), wsb, st), "wv_surface_cdf")
    if float(total.item()) <= 0.0:  # metrics.py:77-78
        raise DegenerateError("mesh has zero total area")
    out = torch.empty((n, 3), dtype=torch.float64, device=dev)
    L.check(lib.wv_sample_surface(_ptr(v), _ptr(f), F, _ptr(cdf), _ptr(total), int(seed) & _MASK,
                                  n, _ptr(out), st), "wv_sample_surface")
    return out


def sample_surface(mesh: TriangleMesh, n: int, seed: int) -> np.ndarray:
    """n points drawn uniformly by area from the mesh surface, (n, 3)."""
    n = int(n)
    if n < 0:
        raise ValueError("sample count must be >= 0")
    if n == 0:
        return np.zeros((0, 3))
    if mesh.num_faces == 0:
        raise DegenerateError("mesh has no faces to sample")
    dev = device()
    v = torch.from_numpy(np.ascontiguousarray(mesh.vertices, dtype=np.float64)).to(dev)
    f = torch.from_numpy(np.ascontiguousarray(mesh.faces, dtype=np.int64)).to(dev)
    return sample_surface_device(v, f, n, seed).cpu().numpy()


def nearest_distances(queries: torch.Tensor, targets: torch.Tensor) -> torch.Tensor:
    """Distance from each query to its nearest target, (nq,) f64 device."""
    lib = L.lib()
    q = queries.to(torch.float64).contiguous()
    t = targets.to(torch.float64).contiguous()
    out = torch.empty(q.shape[0], dtype=torch.float64, device=q.device)
    L.check(lib.wv_nearest_distances(_ptr(q), int(q.shape[0]), _ptr(t), int(t.shape[0]),
                                     _ptr(out), _stream()), "wv_nearest_distances")
    return out


def _as_points(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=device(), dtype=torch.float64).reshape(-1, 3).contiguous()
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1, 3))
    return torch.from_numpy(arr).to(device())


def _mean(d: torch.Tensor) -> float:
    return float(_pairwise_sum(d).item()) / d.numel()  # np.mean: pairwise sum / n


def chamfer_distance(a, b) -> float:
    """Symmetric mean nearest-neighbor distance (metrics.py:111-119)."""
    pa, pb = _as_points(a), _as_points(b)
    if not len(pa) or not len(pb):
        raise ValueError("chamfer distance needs two non-empty point sets")
    return 0.5 * (_mean(nearest_distances(pa, pb)) + _mean(nearest_distances(pb, pa)))


def hausdorff_distance(a, b) -> float:
    """Symmetric worst-case nearest-neighbor distance (metrics.py:122-130)."""
    pa, pb = _as_points(a), _as_points(b)
    if not len(pa) or not len(pb):
        raise ValueError("hausdorff distance needs two non-empty point sets")
    return max(float(nearest_distances(pa, pb).max().item()),
               float(nearest_distances(pb, pa).max().item()))


def evaluate_reconstruction(original: TriangleMesh, reconstructed: TriangleMesh,
                            n: int = 20000, repeats: int = 3, seed: int = 0) -> dict:
    """Sampled Chamfer/Hausdorff statistics between two meshes
    (metrics.py:133-150); the samples never leave the device."""
    if repeats < 1:
        raise ValueError("repeats must be >= 1")
    dev = device()

    def dev_mesh(m):
        return (torch.from_numpy(np.ascontiguousarray(m.vertices, dtype=np.float64)).to(dev),
                torch.from_numpy(np.ascontiguousarray(m.faces, dtype=np.int64)).to(dev))

    ov, of = dev_mesh(original)
    rv, rf = dev_mesh(reconstructed)
    chamfer = np.empty(repeats)
    hausdorff = np.empty(repeats)
    for r in range(repeats):
        pa = sample_surface_device(ov, of, n, seed + r)
        pb = sample_surface_device(rv, rf, n, seed + r)
        if not len(pa) or not len(pb):
            raise ValueError("chamfer distance needs two non-empty point sets")
        dab, dba = nearest_distances(pa, pb), nearest_distances(pb, pa)
        chamfer[r] = 0.5 * (_mean(dab) + _mean(dba))
        hausdorff[r] = max(float(dab.max().item()), float(dba.max().item()))
    return {
        "chamfer_mean": float(chamfer.mean()),
        "chamfer_std": float(chamfer.std()),
        "hausdorff_mean": float(hausdorff.mean()),
        "hausdorff_std": float(hausdorff.std()),
    }
