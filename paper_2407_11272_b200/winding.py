"""Reference-compatible winding-number API (numpy in, numpy out), running
on the B200 kernels.

Mirrors /root/reference/pkg/src/windvox/winding.py:
  winding_number_batch (:271-309), winding_number_exact (:312-320),
  winding_number_soft (:323-333), voxelize (:336-387), binarize (:390-393),
  solid_angle_triangle (:200-255).
Same names, argument order, defaults, return types and exceptions.  One
keyword-only extension: ``precision`` on ``winding_number_batch`` ("f64",
the reference default, or "f32", the FP32 hot path); ``voxelize`` already
has it in the reference.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from .device import DeviceMesh, forward
from .errors import OnSurfaceError
from .types import (SURFACE_EPS_FACTOR, GridSpec, QueryBatchConfig, ScalarField, TriangleMesh,
                    surface_epsilon)

__all__ = ["GridSpec", "ScalarField", "QueryBatchConfig", "solid_angle_triangle",
           "winding_number_exact", "winding_number_soft", "winding_number_batch", "voxelize",
           "binarize", "surface_epsilon"]


def _check_mode(mode: str, use_atan2: bool = True) -> None:
    if mode not in ("exact", "soft"):
        raise ValueError(f"mode must be 'exact' or 'soft', got {mode!r}")
    if mode == "soft" and not use_atan2:
        raise ValueError("the arctan demonstration path only exists in exact mode")


def _check_precision(precision: str) -> None:
    if precision not in ("f64", "f32"):
        raise ValueError(f"precision must be 'f64' or 'f32', got {precision!r}")


def _dispatch(dmesh: DeviceMesh, mode: str, precision: str, use_atan2: bool, *, grid=None,
              points=None, policy=L.POLICY_RAW):
    if not use_atan2 and precision == "f32":
        # the regression-demonstration branch is an f64 reference path only
        precision = "f64"
    return forward(dmesh, mode, precision, grid=grid, points=points, policy=policy,
                   use_atan2=use_atan2)


def winding_number_batch(mesh: TriangleMesh, points, mode: str = "exact",
                         batch: QueryBatchConfig | None = None, use_atan2: bool = True, *,
                         precision: str = "f64") -> tuple[np.ndarray, np.ndarray]:
    """Winding numbers at many points -> (values, on_surface flags)."""
    _check_mode(mode, use_atan2)
    _check_precision(precision)
    pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, 3))
    dtype = np.float64 if precision == "f64" else np.float32
    if len(pts) == 0:
        return np.zeros(0, dtype=dtype), np.zeros(0, dtype=bool)
    dmesh = DeviceMesh.from_numpy(mesh.vertices, mesh.faces)
    dev = dmesh.vertices.device
    tp = torch.from_numpy(pts.astype(np.float32 if precision == "f32" else np.float64))
    tp = tp.pin_memory().to(dev, non_blocking=True)
    vals, flags = _dispatch(dmesh, mode, precision, use_atan2, points=tp)
    return vals.cpu().numpy().astype(dtype, copy=False), flags.cpu().numpy().astype(bool)


def winding_number_exact(mesh: TriangleMesh, q) -> float:
    values, _ = winding_number_batch(mesh, np.asarray(q, dtype=np.float64).reshape(1, 3))
    return float(values[0])


def winding_number_soft(mesh: TriangleMesh, q) -> float:
    values, flags = winding_number_batch(mesh, np.asarray(q, dtype=np.float64).reshape(1, 3),
                                         mode="soft")
    if flags[0]:
        raise OnSurfaceError("query point lies on a face centroid")
    return float(values[0])


def voxelize(mesh: TriangleMesh, spec: GridSpec, mode: str = "exact",
             batch: QueryBatchConfig | None = None, precision: str = "f64") -> ScalarField:
    """Winding number at every lattice node; flagged nodes -> exactly 0.5."""
    _check_mode(mode)
    _check_precision(precision)
    dtype = np.float64 if precision == "f64" else np.float32
    dmesh = DeviceMesh.from_numpy(mesh.vertices, mesh.faces)
    vals, _ = _dispatch(dmesh, mode, precision, True,
                        grid=(spec.bounds_min, spec.bounds_max, spec.resolution),
                        policy=L.POLICY_HALF)
    return ScalarField(spec=spec, values=vals.cpu().numpy().astype(dtype, copy=False))


def binarize(field: ScalarField, threshold: float = 0.5) -> ScalarField:
    """1 where value > threshold (strict), else 0 (winding.py:390-393)."""
    return ScalarField(spec=field.spec,
                       values=(field.values > threshold).astype(field.values.dtype))


def solid_angle_triangle(v0, v1, v2, q) -> float:
    """Signed solid angle of one triangle seen from q (winding.py:200-242).

    A scalar convenience evaluated on the host in f64 (it is not on the hot
    path; one triangle, one point).  Raises OnSurfaceError within the
    surface tolerance; degenerate triangles give exactly 0.0."""
    v0, v1, v2, q = (np.asarray(x, dtype=np.float64).reshape(3) for x in (v0, v1, v2, q))
    corners = np.stack([v0, v1, v2])
    cross = np.cross(v1 - v0, v2 - v0)
    area2 = float(np.linalg.norm(cross))
    if area2 == 0.0:
        return 0.0
    eps = SURFACE_EPS_FACTOR * float(np.linalg.norm(corners.max(axis=0) - corners.min(axis=0)))
    offsets = corners - q
    norms = np.linalg.norm(offsets, axis=1)
    if np.any(norms < eps):
        raise OnSurfaceError("query point coincides with a triangle vertex")
    nhat = cross / area2
    if abs(float(nhat @ (q - v0))) < eps and _inside(q, v0, v1, v2):
        raise OnSurfaceError("query point lies on the triangle")
    e = offsets / norms[:, None]
    det = float(e[0] @ np.cross(e[1], e[2]))
    beta = (1.0 + float(e[0] @ e[1] + e[2] @ e[0])) + float(e[1] @ e[2])
    if det == 0.0 and beta == 0.0:
        return 0.0
    return 2.0 * float(np.arctan2(det, beta))


def _inside(q, v0, v1, v2, tol: float = 1e-12) -> bool:
    u, w, r = v1 - v0, v2 - v0, q - v0
    d00, d01, d11 = u @ u, u @ w, w @ w
    denom = d00 * d11 - d01 * d01
    if denom == 0.0:
        return False
    b1 = (d11 * (r @ u) - d01 * (r @ w)) / denom
    b2 = (d00 * (r @ w) - d01 * (r @ u)) / denom
    return bool(b1 >= -tol and b2 >= -tol and b1 + b2 <= 1.0 + tol)
