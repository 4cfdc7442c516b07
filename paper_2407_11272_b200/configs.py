"""Seeded synthetic workloads of BASELINE.json's five configs.

There is no network, so every mesh is procedural: an icosphere (subdivided
icosahedron projected to the sphere, 20*4^s faces) and a ring torus around
z (2*nu*nv faces), the same primitives the reference ships
(shapes.py:73-139), generated here independently.

  C1  icosphere(3) normalized to [-1,1], grid [-1,1]^3 at 32^3
  C2  torus(0.7,0.3,100,100) with 4 seeded 5x5-quad holes (~19.8k faces,
      open), 128^3; target = binarized exact occupancy of the closed torus
  C3  torus(0.7,0.3,250,200) (100k faces) un-welded into a shuffled soup,
      256^3                                          <- the headline config
  C4  64 x icosphere(4,0.5) with seeded low-frequency radial bumps, 64^3
  C5  torus(0.7,0.3,1000,500) (1M faces), 512^3, forward only
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def icosahedron(radius: float = 1.0):
    t = (1.0 + 5.0 ** 0.5) / 2.0
    v = np.array([(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0),
                  (0, -1, t), (0, 1, t), (0, -1, -t), (0, 1, -t),
                  (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)], dtype=np.float64)
    v *= radius / np.linalg.norm(v[0])
    f = np.array([(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
                  (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
                  (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
                  (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)], dtype=np.int64)
    return v, f


def icosphere(subdivisions: int = 2, radius: float = 1.0):
    """(vertices, faces): each face split 4-to-1 per level, new vertices at
    normalized edge midpoints (vectorized; edge ids via np.unique)."""
    v, f = icosahedron(radius)
    for _ in range(int(subdivisions)):
        e = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]])
        key = np.sort(e, axis=1)
        uniq, inv = np.unique(key, axis=0, return_inverse=True)
        mid = v[uniq[:, 0]] + v[uniq[:, 1]]
        mid *= radius / np.linalg.norm(mid, axis=1, keepdims=True)
        m = len(v) + inv.reshape(3, -1).T  # (F,3): ab, bc, ca
        v = np.concatenate([v, mid])
        a, b, c = f[:, 0], f[:, 1], f[:, 2]
        ab, bc, ca = m[:, 0], m[:, 1], m[:, 2]
        f = np.concatenate([np.stack([a, ab, ca], 1), np.stack([b, bc, ab], 1),
                            np.stack([c, ca, bc], 1), np.stack([ab, bc, ca], 1)])
    return np.ascontiguousarray(v), np.ascontiguousarray(f)


def torus(major: float = 0.7, minor: float = 0.3, nu: int = 48, nv: int = 24):
    """Closed ring torus around z; quad (i,j) -> faces (a,b,c), (a,c,d)."""
    i = np.arange(nu)
    j = np.arange(nv)
    u = 2.0 * np.pi * i / nu
    w = 2.0 * np.pi * j / nv
    ring = major + minor * np.cos(w)[None, :]
    x = ring * np.cos(u)[:, None]
    y = ring * np.sin(u)[:, None]
    z = np.broadcast_to(minor * np.sin(w)[None, :], (nu, nv))
    verts = np.stack([x, y, z], axis=-1).reshape(-1, 3)
    ii, jj = np.meshgrid(i, j, indexing="ij")
    a = ii * nv + jj
    b = ((ii + 1) % nu) * nv + jj
    c = ((ii + 1) % nu) * nv + (jj + 1) % nv
    d = ii * nv + (jj + 1) % nv
    faces = np.concatenate([np.stack([a.ravel(), b.ravel(), c.ravel()], 1),
                            np.stack([a.ravel(), c.ravel(), d.ravel()], 1)])
    return np.ascontiguousarray(verts), np.ascontiguousarray(faces.astype(np.int64))


def normalize_to_unit_cube(verts: np.ndarray) -> np.ndarray:
    lo, hi = verts.min(axis=0), verts.max(axis=0)
    scale = float((hi - lo).max()) / 2.0
    return (verts - (lo + hi) / 2.0) / scale


def torus_with_holes(nu=100, nv=100, holes=4, patch=5, seed=2):
    v, f = torus(0.7, 0.3, nu, nv)
    rng = np.random.default_rng(seed)
    drop = np.zeros(len(f), dtype=bool)
    quads = nu * nv
    for _ in range(holes):
        i0 = int(rng.integers(0, nu))
        j0 = int(rng.integers(0, nv))
        for di in range(patch):
            for dj in range(patch):
                q = ((i0 + di) % nu) * nv + (j0 + dj) % nv
                drop[q] = True
                drop[quads + q] = True
    return v, np.ascontiguousarray(f[~drop])


def soup(verts: np.ndarray, faces: np.ndarray, seed: int = 0):
    """Un-weld into a triangle soup (3 private vertices per face) and shuffle."""
    perm = np.random.default_rng(seed).permutation(len(faces))
    tri = verts[faces[perm]]
    return np.ascontiguousarray(tri.reshape(-1, 3)), np.arange(3 * len(faces),
                                                              dtype=np.int64).reshape(-1, 3)


def random_soup(n_faces: int = 100_000, seed: int = 3, half: float = 0.8, edge: float = 0.05):
    """C3's stress variant: ``n_faces`` independent triangles,
    centres U[-half, half]^3, each an equilateral triangle of edge ~``edge``
    (x U[0.8, 1.2]) in a uniformly random orientation, ``default_rng(seed)``.
    No two faces share a corner position, so nothing welds: the strip
    kernels cannot share distances and the face-ordered kernels run."""
    rng = np.random.default_rng(seed)
    c = rng.uniform(-half, half, size=(n_faces, 3))
    # random orthonormal frames (QR of a Gaussian matrix, sign-fixed -> Haar)
    q, r = np.linalg.qr(rng.normal(size=(n_faces, 3, 3)))
    q = q * np.sign(np.diagonal(r, axis1=1, axis2=2))[:, None, :]
    s = edge * rng.uniform(0.8, 1.2, size=n_faces) / np.sqrt(3.0)   # circumradius
    ang = 2.0 * np.pi * np.arange(3) / 3.0
    loc = np.stack([np.cos(ang), np.sin(ang)], axis=1)                 # (3, 2) in-plane
    tri = c[:, None, :] + s[:, None, None] * np.einsum("kj,fij->fki", loc, q[:, :, :2])
    return np.ascontiguousarray(tri.reshape(-1, 3)), np.arange(3 * n_faces,
                                                             dtype=np.int64).reshape(-1, 3)


def bumpy_icosphere(seed: int, subdivisions: int = 4, radius: float = 0.5):
    v, f = icosphere(subdivisions, radius)
    rng = np.random.default_rng(seed)
    k = rng.normal(size=(3, 3))
    amp = rng.uniform(0.02, 0.06, size=3)
    n = v / np.linalg.norm(v, axis=1, keepdims=True)
    bump = sum(a * np.sin(n @ kk * 3.0) for a, kk in zip(amp, k))
    return v * (1.0 + bump)[:, None], f


@dataclass(frozen=True)
class Workload:
    name: str
    vertices: np.ndarray
    faces: np.ndarray
    lo: tuple
    hi: tuple
    res: tuple

    @property
    def n_nodes(self) -> int:
        return int(np.prod(self.res))

    @property
    def n_faces(self) -> int:
        return int(len(self.faces))

    @property
    def pairs(self) -> int:
        return self.n_nodes * self.n_faces


def make(name: str) -> Workload:
    g = ((-1.0,) * 3, (1.0,) * 3)
    if name == "c1":
        v, f = icosphere(3, 1.0)
        return Workload("c1_icosphere3_32", normalize_to_unit_cube(v), f, *g, (32,) * 3)
    if name == "c2":
        v, f = torus_with_holes()
        return Workload("c2_open_torus_holes_128", v, f, *g, (128,) * 3)
    if name == "c3":
        v, f = soup(*torus(0.7, 0.3, 250, 200), seed=0)
        return Workload("c3_torus100k_soup_256", v, f, *g, (256,) * 3)
    if name == "c3r":  # C3 stress variant: random-triangle soup, nothing welds
        v, f = random_soup(100_000, seed=3)
        return Workload("c3r_random_soup100k_256", v, f, *g, (256,) * 3)
    if name == "c3rs":  # quarter-size c3r for profiling (25k random triangles, 128^3)
        v, f = random_soup(25_000, seed=3)
        return Workload("c3rs_random_soup25k_128", v, f, *g, (128,) * 3)
    if name == "c3s":  # quarter-size C3 for profiling (25k-face soup, 128^3)
        v, f = soup(*torus(0.7, 0.3, 125, 100), seed=0)
        return Workload("c3s_torus25k_soup_128", v, f, *g, (128,) * 3)
    if name == "c5":
        v, f = torus(0.7, 0.3, 1000, 500)
        return Workload("c5_torus1M_512", v, f, *g, (512,) * 3)
    raise KeyError(name)


def c4_batch(n_meshes: int = 64):
    return [bumpy_icosphere(b) for b in range(n_meshes)]
