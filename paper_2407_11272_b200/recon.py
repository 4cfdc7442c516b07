"""Surface reconstruction on the device: marching cubes on
the voxelized grid while it is still in HBM, and uniform Laplacian smoothing.

Mirrors /root/reference/pkg/src/windvox/recon.py:39-140.  Vertices are the
welded lattice-edge crossings, placed by the reference's interpolation and
numbered by the reference's global edge id (axis * N + base node); triangles
come from the classic case table re-indexed into our cell conventions
(``mc_table``), emitted in cell order, slot order within a cell -- so the
vertex AND face arrays are bit-identical to the reference's.

``slab_marching_cubes`` runs the same pipeline on an i-slab-sharded grid
(one rank per GPU): each rank needs only a 1-row halo from the
next rank; per-axis crossing counts and face counts are all-gathered (a few
integers) to turn local prefix sums into the global vertex ids, and the
gathered mesh equals the one-GPU mesh bit for bit.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from .device import _ptr, _stream, device
from .mc_table import EDGE_AXIS, EDGE_BASE, MAX_TRIS, TRI_COUNT, TRI_TABLE
from .morph import uniform_laplacian
from .types import ScalarField, TriangleMesh

__all__ = ["marching_cubes", "marching_cubes_device", "slab_marching_cubes", "laplacian_smooth"]

_TABLES: dict = {}


def _tables(dev):
    t = _TABLES.get(dev)
    if t is None:
        t = (torch.from_numpy(TRI_TABLE.reshape(-1).copy()).to(dev),
             torch.from_numpy(TRI_COUNT.copy()).to(dev),
             torch.from_numpy(EDGE_AXIS.astype(np.int8)).to(dev),
             torch.from_numpy(EDGE_BASE.astype(np.int8).reshape(-1).copy()).to(dev))
        _TABLES[dev] = t
    return t


def _exclusive(x: torch.Tensor) -> tuple[torch.Tensor, int]:
    c = torch.cumsum(x, 0, dtype=torch.int64)
    total = int(c[-1].item()) if c.numel() else 0
    return c - x.to(torch.int64), total


def marching_cubes_device(values: torch.Tensor, grid, iso: float = 0.5):
    """(vertices (M,3) f64, faces (T,3) int64) device tensors for the
    iso-surface of a flat (k fastest) device field on ``grid=(lo, hi, res)``."""
    lib = L.lib()
    lo, hi, res = grid
    if min(int(r) for r in res) < 2:
        raise ValueError("marching cubes needs at least 2 nodes per axis")
    dev = values.device
    v = values.contiguous()
    if v.dtype not in (torch.float32, torch.float64):
        v = v.double()
    f64 = int(v.dtype == torch.float64)
    g = L.make_grid(lo, hi, res)
    rx, ry, rz = (int(r) for r in res)
    n = rx * ry * rz
    cells = (rx - 1) * (ry - 1) * (rz - 1)
    tri_tab, tri_cnt, e_axis, e_base = _tables(dev)
    st = _stream()
    cases = torch.empty(cells, dtype=torch.uint8, device=dev)
    counts = torch.empty(cells, dtype=torch.int32, device=dev)
    L.check(lib.wv_mc_classify(_ptr(v), f64, g, float(iso), _ptr(tri_cnt), _ptr(cases),
                               _ptr(counts), st), "wv_mc_classify")
    flags = torch.empty(3 * n, dtype=torch.int32, device=dev)
    L.check(lib.wv_mc_edges(_ptr(v), f64, g, float(iso), _ptr(flags), st), "wv_mc_edges")
    tri_off, n_tris = _exclusive(counts)
    vidx, n_verts = _exclusive(flags)
    verts = torch.empty((n_verts, 3), dtype=torch.float64, device=dev)
    faces = torch.empty((n_tris, 3), dtype=torch.int64, device=dev)
    if n_tris == 0:
        return verts, faces
    L.check(lib.wv_mc_vertices(_ptr(v), f64, g, float(iso), _ptr(flags), _ptr(vidx), _ptr(verts),
                               st), "wv_mc_vertices")
    L.check(lib.wv_mc_emit(_ptr(cases), _ptr(tri_off), _ptr(tri_tab), MAX_TRIS, _ptr(e_axis),
                           _ptr(e_base), _ptr(vidx), g, _ptr(faces), st), "wv_mc_emit")
    return verts, faces


def slab_marching_cubes(values: torch.Tensor, grid, i0: int, iso: float = 0.5, *,
                        rank: int, world: int, group=None, gather: bool = True):
    """Marching cubes over an i-slab-sharded field.  ``values``: this rank's
    whole i-rows [i0, i0 + rows) of the flat (k fastest) field on
    ``grid=(lo, hi, res)``; ranks own consecutive row ranges in rank order.
    Communication: one all-gather of each rank's first row (the halo the
    previous rank needs), one all-gather of 4 counts per rank, and with
    ``gather`` the pieces of the mesh.  Returns the whole mesh (vertices
    (M,3) f64, faces (T,3) int64) on every rank with ``gather``, else this
    rank's part: (vertices of its own lattice edges, per axis in global id
    order; faces of its cells, with GLOBAL vertex ids; its vertex counts per
    axis; its global face offset)."""
    import torch.distributed as dist
    lib = L.lib()
    lo, hi, res = grid
    rx, ry, rz = (int(r) for r in res)
    if min(rx, ry, rz) < 2:
        raise ValueError("marching cubes needs at least 2 nodes per axis")
    plane = ry * rz
    v = values.contiguous().reshape(-1)
    if v.dtype not in (torch.float32, torch.float64):
        v = v.double()
    if v.numel() % plane:
        raise ValueError("a slab must hold whole i-rows")
    rows = v.numel() // plane
    dev = v.device
    f64 = int(v.dtype == torch.float64)
    # halo: the first row of every rank (the next rank's is ours)
    first = v[:plane].contiguous() if rows else torch.zeros(plane, dtype=v.dtype, device=dev)
    firsts = [torch.empty_like(first) for _ in range(world)]
    dist.all_gather(firsts, first, group=group)
    halo = rank + 1 < world and i0 + rows < rx
    block = torch.cat([v, firsts[rank + 1]]) if halo else v
    nl = rows + int(halo)
    n_loc = nl * plane
    tri_tab, tri_cnt, e_axis, e_base = _tables(dev)
    st = _stream()
    gl = L.make_grid(lo, hi, (nl, ry, rz))
    flags = torch.zeros(3 * n_loc, dtype=torch.int32, device=dev)
    if nl >= 2:
        L.check(lib.wv_mc_edges(_ptr(block), f64, gl, float(iso), _ptr(flags), st), "wv_mc_edges")
    elif nl == 1:  # a lone last row: its axis-1/2 edges only (no cells)
        fl = flags.view(3, plane)
        vr = block.view(ry, rz) <= iso
        fl[1].view(ry, rz)[:-1] = (vr[:-1] != vr[1:]).int()
        fl[2].view(ry, rz)[:, :-1] = (vr[:, :-1] != vr[:, 1:]).int()
    if nl >= 2:
        n_cells = (nl - 1) * (ry - 1) * (rz - 1)
        cases = torch.empty(n_cells, dtype=torch.uint8, device=dev)
        counts = torch.empty(n_cells, dtype=torch.int32, device=dev)
        L.check(lib.wv_mc_classify(_ptr(block), f64, gl, float(iso), _ptr(tri_cnt), _ptr(cases),
                                   _ptr(counts), st), "wv_mc_classify")
        tri_off, n_tris = _exclusive(counts)
    else:
        n_tris = 0
    fl = flags.view(3, nl, plane)
    own = fl[:, :rows].reshape(3, -1)
    cnt = own.sum(dim=1, dtype=torch.int64)
    mine = torch.cat([cnt, torch.tensor([n_tris], dtype=torch.int64, device=dev)])
    allc = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(allc, mine, group=group)
    allc = torch.stack(allc).cpu()                           # (world, 4)
    tot = allc[:, :3].sum(0)
    axis_base = torch.cat([torch.zeros(1, dtype=torch.int64), torch.cumsum(tot, 0)[:2]])
    before = torch.cumsum(allc[:, :3], 0) - allc[:, :3]      # exclusive over ranks
    off = axis_base + before[rank]                           # global id of our first per axis
    vidx = torch.full((3, nl, plane), -1, dtype=torch.int64, device=dev)
    slot = torch.full((3, nl, plane), -1, dtype=torch.int64, device=dev)
    loc_base = 0
    for a in range(3):
        f = own[a]
        ex = torch.cumsum(f, 0, dtype=torch.int64) - f
        vidx[a, :rows] = (ex + int(off[a])).view(rows, plane)
        slot[a, :rows] = (ex + loc_base).view(rows, plane)
        loc_base += int(cnt[a])
        if halo and a > 0:  # the next rank's first-row edges: its ids
            fh = fl[a, rows]
            exh = torch.cumsum(fh, 0, dtype=torch.int64) - fh
            vidx[a, rows] = exh + int(axis_base[a] + before[rank + 1][a])
    n_own = int(cnt.sum())
    verts = torch.empty((n_own, 3), dtype=torch.float64, device=dev)
    if n_own:
        L.check(lib.wv_mc_vertices_slab(_ptr(block), f64, L.make_grid(lo, hi, res), int(i0), nl,
                                        float(iso), _ptr(flags), _ptr(slot), _ptr(verts), st),
                "wv_mc_vertices_slab")
    faces = torch.empty((n_tris, 3), dtype=torch.int64, device=dev)
    if n_tris:
        L.check(lib.wv_mc_emit(_ptr(cases), _ptr(tri_off), _ptr(tri_tab), MAX_TRIS, _ptr(e_axis),
                               _ptr(e_base), _ptr(vidx), gl, _ptr(faces), st), "wv_mc_emit")
    face_off = int(allc[:rank, 3].sum())
    if not gather:
        return verts, faces, cnt.cpu(), face_off
    # gather: vertices per axis in rank order (global ids are axis-major),
    # faces in rank order (cell order)
    def gather_rows(t, counts):
        mx = max(int(c) for c in counts)
        pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
        pad[:t.shape[0]] = t
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
        return [p[:int(c)] for p, c in zip(parts, counts)]
    starts = torch.cat([torch.zeros(1, dtype=torch.int64), torch.cumsum(cnt.cpu(), 0)[:2]])
    per_axis = []
    for a in range(3):
        piece = verts[int(starts[a]):int(starts[a]) + int(cnt[a])]
        per_axis.append(gather_rows(piece, allc[:, a]))
    all_v = torch.cat([p for a in range(3) for p in per_axis[a]])
    all_f = torch.cat(gather_rows(faces, allc[:, 3]))
    return all_v, all_f


def marching_cubes(field: ScalarField, iso: float = 0.5) -> TriangleMesh:
    """Iso-surface of ``field`` as a triangle mesh (outward normals for
    fields where inside means value > iso).  No crossings -> empty mesh."""
    vals = np.ascontiguousarray(field.values)
    dt = torch.float32 if vals.dtype == np.float32 else torch.float64
    t = torch.from_numpy(vals.astype(np.float32 if dt == torch.float32 else np.float64)).to(device())
    spec = field.spec
    v, f = marching_cubes_device(t, (spec.bounds_min, spec.bounds_max, spec.resolution), iso)
    return TriangleMesh(v.cpu().numpy(), f.cpu().numpy())


def laplacian_smooth(mesh: TriangleMesh, lam: float = 0.15, iterations: int = 10) -> TriangleMesh:
    """Uniform (umbrella) Laplacian smoothing, Jacobi updates (recon.py:111-140):
    v <- v + lam (mean(1-ring) - v) for vertices with neighbours, i.e.
    v <- v - lam L v with L = I - D^-1 A; on the device."""
    if iterations < 0:
        raise ValueError("iterations must be >= 0")
    if mesh.num_faces == 0 or iterations == 0 or lam == 0.0:
        return TriangleMesh(mesh.vertices.copy(), mesh.faces.copy())
    dev = device()
    ip, ix, dv = uniform_laplacian(mesh.faces, mesh.num_vertices)
    V = mesh.num_vertices
    lap = torch.sparse_csr_tensor(torch.from_numpy(ip), torch.from_numpy(ix),
                                  torch.from_numpy(dv), size=(V, V),
                                  check_invariants=True).to(dev)
    verts = torch.from_numpy(mesh.vertices.copy()).to(dev)
    for _ in range(int(iterations)):
        verts = verts - lam * (lap @ verts)
    return TriangleMesh(verts.cpu().numpy(), mesh.faces.copy())
