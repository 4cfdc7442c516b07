"""Boundary types of the hot path, with the reference's semantics.

* ``TriangleMesh``     <- mesh_io.py:41-92   (immutable f64 (V,3) + int64 (F,3))
* ``GridSpec``         <- winding.py:69-140  (lattice nodes, bounds included,
                                              flat order k fastest)
* ``ScalarField``      <- winding.py:143-170
* ``QueryBatchConfig`` <- winding.py:173-190 (accepted for API compatibility;
                                              on the GPU the tiling is fixed
                                              and results never depend on it)
* ``VertexGradients`` / ``LossReport`` <- grad.py:30-51
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DegenerateError

SURFACE_EPS_FACTOR = 1e-9


@dataclass(frozen=True)
class TriangleMesh:
    """Indexed triangle soup; faces are 0-based vertex triples (CCW = outward).
    Degenerate, duplicated and non-manifold faces are admitted.  Raises
    ``IndexError`` for out-of-range face indices."""

    vertices: np.ndarray
    faces: np.ndarray

    def __post_init__(self):
        v = np.ascontiguousarray(np.asarray(self.vertices, dtype=np.float64).reshape(-1, 3))
        f = np.ascontiguousarray(np.asarray(self.faces, dtype=np.int64).reshape(-1, 3))
        if f.size:
            bad = (f < 0) | (f >= len(v))
            if bad.any():
                raise IndexError(
                    f"face references vertex {f[bad][0]}, but mesh has {len(v)} vertices")
        object.__setattr__(self, "vertices", v)
        object.__setattr__(self, "faces", f)

    @property
    def num_vertices(self) -> int:
        return int(self.vertices.shape[0])

    @property
    def num_faces(self) -> int:
        return int(self.faces.shape[0])

    def bounds(self):
        if self.num_vertices == 0:
            raise DegenerateError("mesh has no vertices")
        return self.vertices.min(axis=0), self.vertices.max(axis=0)

    def bbox_diagonal(self) -> float:
        lo, hi = self.bounds()
        return float(np.linalg.norm(hi - lo))

    def triangle_corners(self) -> np.ndarray:
        return self.vertices[self.faces]


def surface_epsilon(mesh: TriangleMesh) -> float:
    """1e-9 x bounding-box diagonal, 0 for an empty mesh (winding.py:193-197)."""
    return 0.0 if mesh.num_vertices == 0 else SURFACE_EPS_FACTOR * mesh.bbox_diagonal()


def _as_res(resolution) -> tuple[int, int, int]:
    if np.ndim(resolution) == 0:
        return (int(resolution),) * 3
    res = tuple(int(r) for r in resolution)
    if len(res) != 3:
        raise ValueError("resolution must be a scalar or a 3-tuple")
    return res


@dataclass(frozen=True, eq=False)
class GridSpec:
    """Lattice spanning [bounds_min, bounds_max]; node (i,j,k) sits at
    ``lo + (hi-lo)*(i/(R-1))`` (midpoint when R == 1); flat index
    ``((i*Ry)+j)*Rz+k``."""

    bounds_min: np.ndarray
    bounds_max: np.ndarray
    resolution: tuple

    def __post_init__(self):
        lo = np.asarray(self.bounds_min, dtype=np.float64).reshape(3)
        hi = np.asarray(self.bounds_max, dtype=np.float64).reshape(3)
        res = _as_res(self.resolution)
        if not np.all(lo < hi):
            raise ValueError(f"bounds_min {lo} must be componentwise below bounds_max {hi}")
        if min(res) < 1:
            raise ValueError(f"resolution must be >= 1 per axis, got {res}")
        object.__setattr__(self, "bounds_min", lo)
        object.__setattr__(self, "bounds_max", hi)
        object.__setattr__(self, "resolution", res)

    def __eq__(self, other):
        if not isinstance(other, GridSpec):
            return NotImplemented
        return (self.resolution == other.resolution
                and np.array_equal(self.bounds_min, other.bounds_min)
                and np.array_equal(self.bounds_max, other.bounds_max))

    def __hash__(self):
        return hash((self.resolution, self.bounds_min.tobytes(), self.bounds_max.tobytes()))

    @property
    def num_nodes(self) -> int:
        rx, ry, rz = self.resolution
        return rx * ry * rz

    def axis_nodes(self, axis: int) -> np.ndarray:
        lo, hi, r = self.bounds_min[axis], self.bounds_max[axis], self.resolution[axis]
        if r == 1:
            return np.array([(lo + hi) / 2.0])
        return lo + (hi - lo) * (np.arange(r, dtype=np.float64) / (r - 1))

    def spacing(self) -> np.ndarray:
        r = np.asarray(self.resolution)
        span = self.bounds_max - self.bounds_min
        return np.where(r > 1, span / np.maximum(r - 1, 1), 0.0)

    def node_coordinates(self) -> np.ndarray:
        axes = [self.axis_nodes(a) for a in range(3)]
        mesh = np.meshgrid(*axes, indexing="ij")
        return np.ascontiguousarray(np.stack(mesh, axis=-1).reshape(-1, 3))


@dataclass(eq=False)
class ScalarField:
    """Values on a GridSpec lattice, stored flat (k fastest)."""

    spec: GridSpec
    values: np.ndarray

    def __post_init__(self):
        v = np.asarray(self.values)
        if v.shape != (self.spec.num_nodes,):
            raise ValueError(
                f"expected {self.spec.num_nodes} flat values for resolution "
                f"{self.spec.resolution}, got shape {v.shape}")
        self.values = v

    def values3(self) -> np.ndarray:
        return self.values.reshape(self.spec.resolution)

    def __eq__(self, other):
        if not isinstance(other, ScalarField):
            return NotImplemented
        return self.spec == other.spec and np.array_equal(self.values, other.values)


@dataclass(frozen=True)
class QueryBatchConfig:
    """Accepted for drop-in compatibility (winding.py:173-190).  On the GPU
    the work decomposition is fixed by the kernels' tiling, so neither field
    changes results (the reference makes the same promise)."""

    chunk_size: int = 2000
    thread_count: int | None = None

    def __post_init__(self):
        if self.chunk_size < 1:
            raise ValueError("chunk_size must be >= 1")
        if self.thread_count is not None and self.thread_count < 1:
            raise ValueError("thread_count must be >= 1 or None")


@dataclass(frozen=True)
class VertexGradients:
    vectors: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "vectors", np.ascontiguousarray(
            np.asarray(self.vectors, dtype=np.float64).reshape(-1, 3)))

    def inf_norm(self) -> float:
        return float(np.abs(self.vectors).max()) if self.vectors.size else 0.0


@dataclass(frozen=True)
class LossReport:
    loss: float
    grads: VertexGradients
    excluded_nodes: int
