"""Open-mesh preprocessing on the device.

``flipped_duplication`` (reference openmesh.py:21-48, paper Algorithm 2)
closes an open surface into a thin shell: an orientation-reversed copy of
the mesh offset by ``-epsilon`` times the area-weighted vertex normals.  The
normals are computed on the GPU (``wv_vertex_normals``) with the reference's
summation order, so the output is bit-identical to the reference.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from .device import _ptr, _stream, device
from .errors import DegenerateError
from .types import TriangleMesh

__all__ = ["vertex_normals", "flipped_duplication"]


def _corner_major_csr(faces: np.ndarray, n_verts: int):
    """Per-vertex slots k*F + f in ascending order (np.add.at's order)."""
    f = np.asarray(faces, dtype=np.int64).reshape(-1, 3)
    flat = f.T.reshape(-1)  # index k*F + f
    slots = np.argsort(flat, kind="stable").astype(np.int64)
    off = np.zeros(n_verts + 1, dtype=np.int64)
    if flat.size:
        np.cumsum(np.bincount(flat, minlength=n_verts), out=off[1:])
    return off, slots


def vertex_normals(mesh: TriangleMesh):
    """(normals (V,3) f64, zero_normal (V,) bool), mesh_io.py:176-195."""
    V, F = mesh.num_vertices, mesh.num_faces
    if V == 0:
        return np.zeros((0, 3)), np.zeros(0, dtype=bool)
    dev = device()
    off, slots = _corner_major_csr(mesh.faces, V)
    v = torch.from_numpy(np.ascontiguousarray(mesh.vertices)).to(dev)
    f = torch.from_numpy(np.ascontiguousarray(mesh.faces, dtype=np.int64)).to(dev)
    to = torch.from_numpy(off).to(dev)
    ts = torch.from_numpy(slots).to(dev)
    n = torch.empty((V, 3), dtype=torch.float64, device=dev)
    z = torch.empty(V, dtype=torch.uint8, device=dev)
    L.check(L.lib().wv_vertex_normals(_ptr(v), V, _ptr(f), F, _ptr(to), _ptr(ts), _ptr(n),
                                      _ptr(z), _stream()), "wv_vertex_normals")
    return n.cpu().numpy(), z.cpu().numpy().astype(bool)


def flipped_duplication(mesh: TriangleMesh, epsilon: float = 0.01) -> TriangleMesh:
    """Append an offset, orientation-reversed copy: vertex i's duplicate is
    V+i at v_i - epsilon*n_i, face (a,b,c) is copied as (a',c',b')."""
    if float(epsilon) <= 0.0:
        raise ValueError(f"epsilon must be positive, got {epsilon}")
    normals, zero = vertex_normals(mesh)
    if mesh.num_vertices == 0 or bool(zero.all()):
        raise DegenerateError("every vertex normal is zero; nothing to offset along")
    shifted = mesh.vertices - float(epsilon) * normals
    flipped = (mesh.faces + mesh.num_vertices)[:, [0, 2, 1]]
    return TriangleMesh(np.concatenate([mesh.vertices, shifted]),
                        np.concatenate([mesh.faces, flipped]))
