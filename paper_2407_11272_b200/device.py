"""Device-side staging and kernel launches (torch tensors for memory and
streams, the C ABI for every computation).

``DeviceMesh`` holds a mesh resident in HBM, lazily packs the per-kind face
records (``wv_pack_faces``) and keeps the vertex CSR used by the gradient
gather, so a morph loop or repeated voxelize re-packs only when the vertices
change.  Every launch is stream-ordered on torch's current stream; nothing
here synchronises the host.

Precision: ``"f32"`` is the FP32 hot path (north_star), ``"f64"`` the parity
path that mirrors the reference's default f64 kernels.
"""

from __future__ import annotations

import hashlib
from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L

_EXACT = {"f32": L.PACK_EXACT_F32, "f64": L.PACK_EXACT_F64}
_SOFT = {"f32": L.PACK_SOFT_F32, "f64": L.PACK_SOFT_F64}
_SOFTGRAD = {"f32": L.PACK_SOFTGRAD_F32, "f64": L.PACK_SOFTGRAD_F64}
_EXACTGRAD = {"f32": L.PACK_EXACTGRAD_F32, "f64": L.PACK_EXACTGRAD_F64}
_DT = {"f32": torch.float32, "f64": torch.float64}
# exact f32 forwards with at least this many row-aligned lattice nodes use
# the strip-ordered records (wv_strip.cu): its host-side strip builder
# (~0.5 us per face, once per DeviceMesh) pays off from ~2M nodes
STRIP_MIN_NODES = 1 << 21
# ... and only when the mesh actually forms strips: a strip restart costs the
# two extra square roots plus the strip kernel's per-face branch, so above
# this fraction of restarting faces (e.g. a random-triangle soup, where no
# corner position is shared: 100%) the face-ordered kernels are faster
STRIP_MAX_RESTART = 0.25
# the f64 exact backward takes the edge trails (no row alignment needed) from
# this many query points: the host trail builder (~1 us per face, once per
# DeviceMesh) against ~2x fewer f64 edge evaluations per point
TRAIL64_MIN_POINTS = 1 << 16


def strip_order(vertices: np.ndarray, faces: np.ndarray):
    """Face strips of a mesh (wv_strip_order, host code: no GPU needed):
    (perm (F,), window (F,3), flags (F,) u8) -- see include/windvox_b200.h."""
    v = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
    f = np.ascontiguousarray(faces, dtype=np.int64).reshape(-1, 3)
    F = len(f)
    perm = np.empty(F, dtype=np.int64)
    win = np.empty((F, 3), dtype=np.int64)
    fl = np.empty(F, dtype=np.uint8)
    L.check(L.load_library().wv_strip_order(v.ctypes.data, len(v), f.ctypes.data, F,
                                            perm.ctypes.data, win.ctypes.data, fl.ctypes.data),
            "wv_strip_order")
    return perm, win, fl


def edge_trails(vertices: np.ndarray, faces: np.ndarray, dead: np.ndarray | None = None):
    """Edge trails of a mesh for the exact backward (wv_edge_trails, host code:
    no GPU needed): (windows (W,K+1) int64 vertex ids, CSR offsets (V+1,),
    signed CSR slots (S,), representative vertex id per vertex (V,)) -- see
    include/windvox_b200.h and csrc/wv_trail.cu; K = wv_trail_edges()."""
    import ctypes
    lib = L.load_library()
    K = int(lib.wv_trail_edges())
    v = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
    f = np.ascontiguousarray(faces, dtype=np.int64).reshape(-1, 3)
    F, V = len(f), len(v)
    win = np.empty((max(1, 3 * F), K + 1), dtype=np.int64)
    off = np.empty(V + 1, dtype=np.int64)
    slots = np.empty(max(1, 6 * F), dtype=np.int64)
    vrep = np.empty(max(1, V), dtype=np.int64)
    d = None if dead is None else np.ascontiguousarray(dead, dtype=np.uint8).reshape(-1)
    nw, ns = ctypes.c_int64(0), ctypes.c_int64(0)
    L.check(lib.wv_edge_trails(
        v.ctypes.data, V, f.ctypes.data, F, None if d is None else d.ctypes.data,
        win.ctypes.data, ctypes.addressof(nw), off.ctypes.data, slots.ctypes.data,
        ctypes.addressof(ns), vrep.ctypes.data), "wv_edge_trails")
    return win[:nw.value].copy(), off, slots[:ns.value].copy(), vrep[:V].copy()


# Host-side plans (strip order, edge trails, corner sharing) depend only on
# the mesh CONTENT; a caller that rebuilds a DeviceMesh from the same host
# arrays every step (e.g. an end-to-end loop, one per rank) reuses them.
# Keyed by a digest of the f64 vertex and int64 face bytes; a few entries.
_PLANS: OrderedDict = OrderedDict()
_PLANS_MAX = 8


def _digest(*arrays) -> bytes:
    h = hashlib.sha256()  # SHA extensions: ~1 GB/s on the host
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(f"{a.dtype.str}{a.shape}".encode())
        h.update(memoryview(a).cast("B"))
    return h.digest()


def _plan(kind: str, key: bytes, build):
    k = (kind, key)
    hit = _PLANS.get(k)
    if hit is None:
        hit = build()  # (callers treat plan arrays as read-only)
        _PLANS[k] = hit
        while len(_PLANS) > _PLANS_MAX:
            _PLANS.popitem(last=False)
    else:
        _PLANS.move_to_end(k)
    return hit


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def device() -> torch.device:
    L.lib()
    return torch.device("cuda", torch.cuda.current_device())


def _check_precision(precision: str) -> None:
    if precision not in _DT:
        raise ValueError(f"precision must be 'f64' or 'f32', got {precision!r}")


def vertex_csr(faces: np.ndarray, n_verts: int) -> tuple[np.ndarray, np.ndarray]:
    """(offsets (V+1,), slots (3F,)) with slot = 3*f + corner, grouped by
    vertex in stable (face, corner) order -- the fixed summation order of
    the face->vertex gather."""
    flat = np.ascontiguousarray(faces, dtype=np.int64).reshape(-1)
    slots = np.argsort(flat, kind="stable").astype(np.int64)
    counts = np.bincount(flat, minlength=n_verts) if flat.size else np.zeros(n_verts, np.int64)
    off = np.zeros(n_verts + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    return off, slots


def exact_edge_weights(faces: np.ndarray, dead: np.ndarray | None = None):
    """Active faces and net directed-edge weights for the exact backward.

    d(Omega_f)/dv is a sum of per-edge terms T(P->Q) with T(Q->P) = -T(P->Q),
    so over the whole mesh only the NET multiplicity of each undirected edge
    matters: k = #(min->max) - #(max->min).  The first occurrence (face order)
    of each edge carries weight k*dir (dir = +1 if it runs min->max), every
    other occurrence 0; faces whose three weights vanish are inactive.
    Degenerate faces (dropped by the reference forward, winding.py:264) are
    excluded.  Returns (active (A,) int64, weights (A,3) float32)."""
    f = np.ascontiguousarray(faces, dtype=np.int64).reshape(-1, 3)
    nf = len(f)
    if nf == 0:
        return np.zeros(0, np.int64), np.zeros((0, 3), np.float32)
    live = np.ones(nf, bool) if dead is None else ~np.asarray(dead, bool)
    u = f.reshape(-1)                        # corner k of face i -> edge (k, k+1)
    v = f[:, [1, 2, 0]].reshape(-1)
    lo = np.minimum(u, v)
    hi = np.maximum(u, v)
    sgn = np.where(u < v, 1, -1)
    sgn[u == v] = 0                          # self-loop edges carry nothing
    sgn = sgn * np.repeat(live, 3)
    key = lo * (int(f.max()) + 1) + hi
    # group by edge; within a group live (sgn != 0) occurrences first, so the
    # weight lands on a face that actually contributes
    order = np.lexsort(((sgn == 0).astype(np.int8), key))
    ks = key[order]
    start = np.ones(len(ks), bool)
    start[1:] = ks[1:] != ks[:-1]
    grp = np.cumsum(start) - 1
    net = np.zeros(int(grp[-1]) + 1, np.int64)
    np.add.at(net, grp, sgn[order])
    first = order[start]                     # first occurrence of each edge
    w = np.zeros(len(u), np.float32)
    w[first] = (net * sgn[first]).astype(np.float32)   # sgn[first] in {+1,-1,0}
    w = w.reshape(nf, 3)
    active = np.flatnonzero(np.any(w != 0, axis=1)).astype(np.int64)
    # unit-weight faces first: the kernel takes a warp-uniform fast path when
    # all 32 faces of a warp have unit weights
    unit = np.all(w[active] == 1, axis=1)
    active = np.concatenate([active[unit], active[~unit]])
    return active, np.ascontiguousarray(w[active])


def strip_pairs(vertices: np.ndarray, faces: np.ndarray, weights: np.ndarray, order=None):
    """Pair consecutive faces of each strip (strip_order) for the exact
    backward's pair kernel: returns (rows (2P,3) int64 vertex ids with
    corners in window order, row weights (2P,3) f32, valid (2P,) bool).
    ``order``: a precomputed ``strip_order(vertices, faces)``.
    Rows 2i, 2i+1 are a pair F1 = (A,B,C), F2 = (B',C',D); an unpaired face
    gets a zero-weight partner (B,C,A) (valid False).  Window edge weights:
    edge AB of a window is the face's directed edge between those corners,
    negated when the window reflects the face's orientation."""
    f = np.ascontiguousarray(faces, dtype=np.int64).reshape(-1, 3)
    w = np.asarray(weights, dtype=np.float32).reshape(-1, 3)
    A = len(f)
    if A == 0:
        return np.zeros((0, 3), np.int64), np.zeros((0, 3), np.float32), np.zeros(0, bool)
    perm, win, fl = strip_order(vertices, f) if order is None else order
    fo, wo = f[perm], w[perm]
    pos = np.stack([np.argmax(fo == win[:, c:c + 1], axis=1) for c in range(3)], axis=1)
    refl = (fl & 2) != 0
    ar = np.arange(A)
    ww = np.empty((A, 3), np.float32)
    for e in range(3):  # window edge (e, e+1)
        p0, p1 = pos[:, e], pos[:, (e + 1) % 3]
        ww[:, e] = np.where(refl, -wo[ar, p1], wo[ar, p0])
    restart = (fl & 1) != 0
    start = np.maximum.accumulate(np.where(restart, ar, 0))
    idx = ar - start                               # position within the strip
    first = np.flatnonzero(idx % 2 == 0)           # pair heads
    has2 = np.zeros(len(first), bool)
    nxt = first + 1
    ok = nxt < A
    has2[ok] = ~restart[nxt[ok]]
    P = len(first)
    rows = np.empty((2 * P, 3), np.int64)
    rw = np.zeros((2 * P, 3), np.float32)
    valid = np.zeros(2 * P, bool)
    rows[0::2] = win[first]
    rw[0::2] = ww[first]
    valid[0::2] = True
    h = first[has2]
    rows[1::2][has2] = win[h + 1]
    rw[1::2][has2] = ww[h + 1]
    valid[1::2][has2] = True
    s = first[~has2]
    rows[1::2][~has2] = win[s][:, [1, 2, 0]]       # zero-weight partner (B, C, A)
    return rows, rw, valid


def vertex_csr_rows(rows: np.ndarray, valid: np.ndarray, n_verts: int):
    """vertex_csr over the valid rows only (slots keep their row indices)."""
    flat = np.ascontiguousarray(rows, dtype=np.int64).reshape(-1)
    ids = np.flatnonzero(np.repeat(np.asarray(valid, bool), 3))
    vals = flat[ids]
    slots = ids[np.argsort(vals, kind="stable")].astype(np.int64)
    counts = np.bincount(vals, minlength=n_verts) if vals.size else np.zeros(n_verts, np.int64)
    off = np.zeros(n_verts + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    return off, slots


def dead_faces(vertices: np.ndarray, faces: np.ndarray) -> np.ndarray:
    """|N| == 0 in f64, the reference's degenerate-face test (winding.py:262-264)."""
    v = np.asarray(vertices, dtype=np.float64).reshape(-1, 3)
    f = np.asarray(faces, dtype=np.int64).reshape(-1, 3)
    if len(f) == 0:
        return np.zeros(0, bool)
    t = v[f]
    return ~(np.linalg.norm(np.cross(t[:, 1] - t[:, 0], t[:, 2] - t[:, 0]), axis=1) > 0.0)


def _dead_faces_dev(vertices: torch.Tensor, faces: torch.Tensor) -> torch.Tensor:
    """``dead_faces`` on the device: |N| == 0 in f64 (same expression order)."""
    t = vertices.to(torch.float64)[faces.long()]
    u, w = t[:, 1] - t[:, 0], t[:, 2] - t[:, 0]
    n = torch.stack([u[:, 1] * w[:, 2] - u[:, 2] * w[:, 1], u[:, 2] * w[:, 0] - u[:, 0] * w[:, 2],
                     u[:, 0] * w[:, 1] - u[:, 1] * w[:, 0]], dim=1)
    return ~(torch.sqrt((n * n).sum(1)) > 0.0)


@dataclass
class DeviceMesh:
    """Mesh resident on the GPU.  ``vertices`` (V,3) f32/f64 and ``faces``
    (F,3) int32/int64, contiguous CUDA tensors."""

    vertices: torch.Tensor
    faces: torch.Tensor
    _packs: dict = field(default_factory=dict, repr=False)
    _version: int = field(default=-1, repr=False)
    _csr: tuple | None = field(default=None, repr=False)

    @classmethod
    def from_numpy(cls, vertices: np.ndarray, faces: np.ndarray, dev=None,
                   dtype=torch.float64) -> "DeviceMesh":
        dev = dev or device()
        v = torch.from_numpy(np.ascontiguousarray(np.asarray(vertices), dtype=np.float64)
                             ).reshape(-1, 3).to(dtype)
        f = torch.from_numpy(np.ascontiguousarray(np.asarray(faces), dtype=np.int64)).reshape(-1, 3)
        v = v.pin_memory().to(dev, non_blocking=True)
        f = f.pin_memory().to(dev, non_blocking=True)
        m = cls(v.contiguous(), f.contiguous())
        m._faces_np = np.ascontiguousarray(np.asarray(faces), dtype=np.int64).reshape(-1, 3)
        m._verts_np = np.ascontiguousarray(np.asarray(vertices), dtype=np.float64).reshape(-1, 3)
        return m

    @property
    def num_vertices(self) -> int:
        return int(self.vertices.shape[0])

    @property
    def num_faces(self) -> int:
        return int(self.faces.shape[0])

    def invalidate(self) -> None:
        self._packs.clear()

    def set_vertices(self, vertices: torch.Tensor) -> None:
        """Replace the vertex positions (same connectivity); re-packs lazily.
        The exact backward's active faces and edge weights exclude faces that
        are degenerate at the CURRENT positions (the reference re-drops them
        on every call, winding.py:262-264): if a move changes that set, the
        cached setups are rebuilt from the new positions."""
        self.vertices = vertices.contiguous()
        self._packs.clear()
        tr = getattr(self, "_exact_trail", None)
        if tr is not None:
            # the trail records evaluate every vertex of a welded position at
            # its representative's coordinates: rebuild when a move splits a weld
            ids, reps = tr[3]
            if ids.numel():
                v32 = self.vertices.detach().float()
                if not torch.equal(v32[ids], v32[reps]):
                    self._verts_np = self.vertices.detach().double().cpu().numpy()
                    self._exact_trail = None
        dead0 = getattr(self, "_dead_dev", None)
        if dead0 is not None:
            dead = _dead_faces_dev(self.vertices, self.faces)
            if not torch.equal(dead, dead0):
                self._verts_np = self.vertices.detach().double().cpu().numpy()
                self._exact_grad = None
                self._exact_pair = None
                self._exact_trail = None
                self._dead_dev = None

    def packed(self, kind: int) -> torch.Tensor:
        ver = (id(self.vertices), self.vertices._version)
        if ver != self._version:
            self._packs.clear()
            self._version = ver
        buf = self._packs.get(kind)
        if buf is not None:
            return buf
        lib = L.lib()
        v, f = self.vertices, self.faces
        if not (v.is_cuda and f.is_cuda):
            raise ValueError("DeviceMesh tensors must live on a CUDA device")
        if v.dtype not in (torch.float32, torch.float64):
            raise TypeError("vertices must be float32 or float64")
        if f.dtype not in (torch.int32, torch.int64):
            raise TypeError("faces must be int32 or int64")
        v = v.contiguous()
        f = f.contiguous()
        nbytes = int(lib.wv_packed_bytes(kind, self.num_faces))
        buf = torch.empty(nbytes, dtype=torch.uint8, device=v.device)
        if kind == L.PACK_EXACTSTRIP_F64:
            perm, win, fl = self.strip_setup()
            L.check(lib.wv_pack_exact_strip_f64(_ptr(v), int(v.dtype == torch.float64),
                                                self.num_vertices, _ptr(f),
                                                int(f.dtype == torch.int64), self.num_faces,
                                                _ptr(perm), _ptr(win), _ptr(fl), _ptr(buf),
                                                _stream()), "wv_pack_exact_strip_f64")
        elif kind == L.PACK_EXACTSTRIP_F32:
            perm, win, fl = self.strip_setup()
            L.check(lib.wv_pack_exact_strip(_ptr(v), int(v.dtype == torch.float64),
                                            self.num_vertices, _ptr(f),
                                            int(f.dtype == torch.int64), self.num_faces,
                                            _ptr(perm), _ptr(win), _ptr(fl), _ptr(buf),
                                            _stream()), "wv_pack_exact_strip")
        else:
            L.check(lib.wv_pack_faces(kind, _ptr(v), int(v.dtype == torch.float64),
                                      self.num_vertices, _ptr(f), int(f.dtype == torch.int64),
                                      self.num_faces, _ptr(buf), _stream()), "wv_pack_faces")
        self._packs[kind] = buf
        return buf

    def strip_setup(self):
        """Device copies of the face strips (strip_order), built once from the
        positions at setup time.  Later vertex moves may break the welds;
        the packer then restarts the strip there (always correct)."""
        st = getattr(self, "_strip", None)
        if st is None:
            vnp = getattr(self, "_verts_np", None)
            if vnp is None:
                vnp = self.vertices.detach().double().cpu().numpy()
            fnp = self.faces_np()
            perm, win, fl = _plan("strip", self._plan_key(vnp),
                                  lambda: strip_order(vnp, fnp))
            dev = self.vertices.device
            st = tuple(torch.from_numpy(a).to(dev) for a in (perm, win, fl))
            self._strip = st
            self._strip_host = (perm, win, fl)
        return st

    def strip_restart_fraction(self) -> float:
        """Fraction of faces that start a strip in ``strip_setup``'s order
        (builds the order on first use)."""
        self.strip_setup()
        fl = self._strip_host[2]
        return float(np.count_nonzero(fl & 1)) / max(1, len(fl))

    def _plan_key(self, vnp: np.ndarray) -> bytes:
        """Digest of (vnp, faces) for the host-plan cache, once per array."""
        k = getattr(self, "_pkey", None)
        if k is None or k[0] is not vnp:
            k = (vnp, _digest(vnp, self.faces_np()))
            self._pkey = k
        return k[1]

    def shared_corner_fraction(self) -> float:
        """1 - (distinct corner positions) / (3F): ~5/6 for a closed surface
        (welded or un-welded soup alike: the copies are bitwise equal), 0 for
        a soup of independent triangles.  Positions are hashed from their f64
        bit patterns (a collision can only overstate sharing, which the strip
        builder then measures exactly)."""
        vnp = getattr(self, "_verts_np", None)
        if vnp is None:
            vnp = self.vertices.detach().double().cpu().numpy()
        fnp = self.faces_np()

        def frac():
            bits = np.ascontiguousarray(vnp, dtype=np.float64).view(np.uint64).reshape(-1, 3)
            with np.errstate(over="ignore"):
                h = (bits[:, 0] * np.uint64(0x9E3779B97F4A7C15)
                     ^ bits[:, 1] * np.uint64(0xC2B2AE3D27D4EB4F)
                     ^ bits[:, 2] * np.uint64(0x165667B19E3779F9))
            corners = h[fnp.reshape(-1)]
            if corners.size == 0:
                return 0.0
            return 1.0 - np.unique(corners).size / corners.size

        return _plan("share", self._plan_key(vnp), frac)

    def strips_pay(self) -> bool:
        """Whether the strip-ordered kernels beat the face-ordered ones on this
        mesh (restart fraction <= STRIP_MAX_RESTART); decided once."""
        sp = getattr(self, "_strips_pay", None)
        if sp is None:
            # cheap reject first: when most face corners have a position no
            # other corner shares (a random soup), no strip can form and the
            # strip builder's sorts are not worth running
            sp = (self.num_faces > 0 and self.shared_corner_fraction() >= 0.5
                  and self.strip_restart_fraction() <= STRIP_MAX_RESTART)
            self._strips_pay = sp
        return sp

    def faces_np(self) -> np.ndarray:
        fn = getattr(self, "_faces_np", None)
        if fn is None:
            fn = self.faces.detach().cpu().numpy().astype(np.int64)  # connectivity is static
            self._faces_np = fn
        return fn

    def csr(self) -> tuple[torch.Tensor, torch.Tensor]:
        if self._csr is None:
            off, slots = vertex_csr(self.faces_np(), self.num_vertices)
            dev = self.vertices.device
            self._csr = (torch.from_numpy(off).to(dev), torch.from_numpy(slots).to(dev))
        return self._csr

    def exact_grad_setup(self):
        """(active (A,) int64 dev, weights (A,3) f32 dev, CSR over active
        corners).  Connectivity-only, computed once (dead faces from the
        vertex positions at setup time)."""
        eg = getattr(self, "_exact_grad", None)
        if eg is None:
            vnp = getattr(self, "_verts_np", None)
            if vnp is None:
                vnp = self.vertices.detach().double().cpu().numpy()
            fnp = self.faces_np()
            dead = dead_faces(vnp, fnp)
            self._dead_dev = torch.from_numpy(dead).to(self.vertices.device)
            active, w = exact_edge_weights(fnp, dead)
            off, slots = vertex_csr(fnp[active], self.num_vertices)
            dev = self.vertices.device
            eg = (torch.from_numpy(active).to(dev), torch.from_numpy(w).to(dev),
                  (torch.from_numpy(off).to(dev), torch.from_numpy(slots).to(dev)))
            self._exact_grad = eg
        return eg

    def exact_pair_setup(self):
        """Strip pairs of the active faces for the exact f32 backward
        (wv_exact_pair_bwd_*): (faces (2P,3) int64 dev in pair order with
        window-ordered corners, weights (2P,3) f32 dev, CSR over the real
        rows, row ids 0..2P-1 for the packer).  Connectivity-only, built once from the setup-time positions
        (a pair whose welds later break is evaluated face by face)."""
        ps = getattr(self, "_exact_pair", None)
        if ps is None:
            vnp = getattr(self, "_verts_np", None)
            if vnp is None:
                vnp = self.vertices.detach().double().cpu().numpy()
            fnp = self.faces_np()
            dead = dead_faces(vnp, fnp)
            self._dead_dev = torch.from_numpy(dead).to(self.vertices.device)
            active, w = exact_edge_weights(fnp, dead)
            # every face active in face order (soups): the forward's strips apply
            order = getattr(self, "_strip_host", None)
            if order is not None and not np.array_equal(active, np.arange(len(fnp))):
                order = None
            rows_f, rows_w, valid = strip_pairs(vnp, fnp[active], w, order)
            off, slots = vertex_csr_rows(rows_f, valid, self.num_vertices)
            dev = self.vertices.device
            ps = (torch.from_numpy(rows_f).to(dev), torch.from_numpy(rows_w).to(dev),
                  (torch.from_numpy(off).to(dev), torch.from_numpy(slots).to(dev)),
                  torch.arange(len(rows_f), dtype=torch.int64, device=dev))
            self._exact_pair = ps
        return ps

    def packed_exact_pair(self) -> torch.Tensor:
        key = "exact_pair_f32"
        ver = (id(self.vertices), self.vertices._version)
        if ver != self._version:
            self._packs.clear()
            self._version = ver
        buf = self._packs.get(key)
        if buf is not None:
            return buf
        rows_f, rows_w, _, idx = self.exact_pair_setup()
        lib = L.lib()
        v = self.vertices.contiguous()
        n = int(rows_f.shape[0])
        kind = L.PACK_EXACTGRAD_F32
        buf = torch.empty(int(lib.wv_packed_bytes(kind, n)), dtype=torch.uint8, device=v.device)
        L.check(lib.wv_pack_exact_grad(kind, _ptr(v), int(v.dtype == torch.float64),
                                       self.num_vertices, _ptr(rows_f), 1, _ptr(idx),
                                       _ptr(rows_w), n, _ptr(buf), _stream()),
                "wv_pack_exact_grad (strip pairs)")
        self._packs[key] = buf
        return buf

    def abs_max(self) -> float:
        """Largest |vertex coordinate| (setup-time positions, cached: the
        trail-scale screen it feeds has a 1024x margin)."""
        am = getattr(self, "_abs_max", None)
        if am is None:
            vnp = getattr(self, "_verts_np", None)
            if vnp is None:
                vnp = self.vertices.detach().double().cpu().numpy()
            am = float(np.abs(vnp).max()) if vnp.size else 0.0
            self._abs_max = am
        return am

    def trails_pay(self) -> bool:
        """Whether the edge-trail backward beats the face kernels: corner
        positions must be shared (a closed surface, welded or a soup); a
        random soup of independent triangles has nothing to share."""
        tp = getattr(self, "_trails_pay", None)
        if tp is None:
            tp = self.num_faces > 0 and self.shared_corner_fraction() >= 0.5
            self._trails_pay = tp
        return tp

    def exact_trail_setup(self):
        """Edge trails for the exact f32 backward (wv_exact_trail_bwd_*):
        (windows (W,K+1) int64 dev, CSR (off, signed slots) dev, W, (ids, reps)
        dev: vertices that share a representative's position).  Built from
        the positions at setup time; ``set_vertices`` rebuilds it when a move
        splits a weld."""
        ts = getattr(self, "_exact_trail", None)
        if ts is None:
            vnp = getattr(self, "_verts_np", None)
            if vnp is None:
                vnp = self.vertices.detach().double().cpu().numpy()
            fnp = self.faces_np()

            def build():
                dead = dead_faces(vnp, fnp)
                return (*edge_trails(vnp, fnp, dead), dead)

            win, off, slots, vrep, dead = _plan("trail", self._plan_key(vnp), build)
            self._dead_dev = torch.from_numpy(dead).to(self.vertices.device)
            dev = self.vertices.device
            ids = np.flatnonzero(vrep != np.arange(len(vrep))).astype(np.int64)
            ts = (torch.from_numpy(win).to(dev),
                  (torch.from_numpy(off).to(dev), torch.from_numpy(slots).to(dev)),
                  len(win),
                  (torch.from_numpy(ids).to(dev), torch.from_numpy(vrep[ids]).to(dev)))
            self._exact_trail = ts
        return ts

    def packed_exact_trail(self, precision: str = "f32") -> torch.Tensor:
        key = f"exact_trail_{precision}"
        ver = (id(self.vertices), self.vertices._version)
        if ver != self._version:
            self._packs.clear()
            self._version = ver
        buf = self._packs.get(key)
        if buf is not None:
            return buf
        win, _, W, _ = self.exact_trail_setup()
        lib = L.lib()
        v = self.vertices.contiguous()
        kind, fn = ((L.PACK_EXACTTRAIL_F32, lib.wv_pack_exact_trail) if precision == "f32"
                    else (L.PACK_EXACTTRAIL_F64, lib.wv_pack_exact_trail_f64))
        buf = torch.empty(int(lib.wv_packed_bytes(kind, W)), dtype=torch.uint8, device=v.device)
        L.check(fn(_ptr(v), int(v.dtype == torch.float64), self.num_vertices, _ptr(win), W,
                   _ptr(buf), _stream()), "wv_pack_exact_trail")
        self._packs[key] = buf
        return buf

    def packed_exact_grad(self, precision: str) -> torch.Tensor:
        kind = _EXACTGRAD[precision]
        ver = (id(self.vertices), self.vertices._version)
        if ver != self._version:
            self._packs.clear()
            self._version = ver
        buf = self._packs.get(kind)
        if buf is not None:
            return buf
        active, w, _ = self.exact_grad_setup()
        lib = L.lib()
        v = self.vertices.contiguous()
        f = self.faces.contiguous()
        A = int(active.shape[0])
        buf = torch.empty(int(lib.wv_packed_bytes(kind, A)), dtype=torch.uint8, device=v.device)
        L.check(lib.wv_pack_exact_grad(kind, _ptr(v), int(v.dtype == torch.float64),
                                       self.num_vertices, _ptr(f), int(f.dtype == torch.int64),
                                       _ptr(active), _ptr(w), A, _ptr(buf), _stream()),
                "wv_pack_exact_grad")
        self._packs[kind] = buf
        return buf


def _points_arg(points, dev, dtype):
    pts = torch.as_tensor(points).to(device=dev, dtype=dtype).contiguous().reshape(-1, 3)
    return pts, int(pts.shape[0])


def _grid_count(grid, n0, count):
    lo, hi, res = grid
    total = int(res[0]) * int(res[1]) * int(res[2])
    return total - int(n0) if count is None else int(count)


def lattice_paths(mesh: DeviceMesh, mode: str, precision: str, grid, n0: int, count: int):
    """Which records the automatic choice takes for a lattice node range:
    (forward over strips, exact backward over strip pairs).  Strips need a
    large range (STRIP_MIN_NODES, the host strip builder's break-even), a mesh
    that forms strips (``strips_pay``) and, for the f32 row kernel, 8-node
    aligned k-rows; strip pairs exist for the exact f32 backward only."""
    if mode != "exact" or count < STRIP_MIN_NODES or mesh.num_faces == 0:
        return False, False
    if precision == "f32" and not (int(grid[2][2]) % 8 == 0 and int(n0) % 8 == 0
                                   and count % 8 == 0):
        fwd = False
    else:
        fwd = mesh.strips_pay()
    return fwd, precision == "f32" and mesh.strips_pay()


def backward_path(mesh: DeviceMesh, mode: str, precision: str, grid, n0: int, count: int) -> str:
    """The records face_grad's automatic choice takes for a lattice range:
    "trails", "pairs", "faces" (exact) or "soft"."""
    if mode != "exact":
        return "soft"
    if precision == "f64":
        return "trails" if count >= TRAIL64_MIN_POINTS and mesh.trails_pay() else "faces"
    big = precision == "f32" and count >= STRIP_MIN_NODES and mesh.num_faces > 0
    if big and trail_rows_ok(grid, n0) and mesh.trails_pay() and trail_scale_ok(mesh, grid):
        return "trails"
    if big and mesh.strips_pay():
        return "pairs"
    return "faces"


def forward(mesh: DeviceMesh, mode: str, precision: str, *, grid=None, n0: int = 0,
            count: int | None = None, points=None, policy: int = L.POLICY_RAW,
            use_atan2: bool = True, out: torch.Tensor | None = None,
            flags: torch.Tensor | None = None, strip: bool | None = None):
    """Winding numbers on the device.  ``grid=(lo, hi, res)`` with the node
    range [n0, n0+count), or ``points`` (n,3).  Returns (values, flags u8).
    ``strip`` (exact only): strip-ordered records; None = automatic (lattice
    ranges of >= STRIP_MIN_NODES nodes, row-aligned for f32)."""
    _check_precision(precision)
    if mode not in ("exact", "soft"):
        raise ValueError(f"mode must be 'exact' or 'soft', got {mode!r}")
    lib = L.lib()
    dev = mesh.vertices.device
    dt = _DT[precision]
    kind = (_EXACT if mode == "exact" else _SOFT)[precision]
    if points is not None:
        pts, count = _points_arg(points, dev, dt)
    else:
        count = _grid_count(grid, n0, count)
    out = torch.empty(count, dtype=dt, device=dev) if out is None else out
    flags = torch.empty(count, dtype=torch.uint8, device=dev) if flags is None else flags
    if count == 0:
        return out, flags
    F = mesh.num_faces
    st = _stream()
    if precision == "f32":
        if not use_atan2:
            raise ValueError("the single-argument arctan branch exists only at precision='f64'")
        if strip is None:
            strip = points is None and lattice_paths(mesh, mode, precision, grid, n0, count)[0]
        if strip and mode != "exact":
            raise ValueError("strip records exist for the exact forward only")
        if strip:
            kind = L.PACK_EXACTSTRIP_F32
        packed = mesh.packed(kind)
        wsb = int(lib.wv_fwd_workspace_bytes(kind, F, count))
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev) if wsb else None
        if strip:
            if points is not None:
                rc = lib.wv_exact_strip_fwd_points_f32(_ptr(packed), F, _ptr(pts), count, policy,
                                                       _ptr(out), _ptr(flags), _ptr(ws), wsb, st)
            else:
                rc = lib.wv_exact_strip_fwd_grid_f32(_ptr(packed), F, L.make_grid(*grid),
                                                     int(n0), count, policy, _ptr(out),
                                                     _ptr(flags), _ptr(ws), wsb, st)
        elif points is not None:
            fn = lib.wv_exact_fwd_points_f32 if mode == "exact" else lib.wv_soft_fwd_points_f32
            rc = fn(_ptr(packed), F, _ptr(pts), count, policy, _ptr(out), _ptr(flags), _ptr(ws),
                    wsb, st)
        else:
            fn = lib.wv_exact_fwd_grid_f32 if mode == "exact" else lib.wv_soft_fwd_grid_f32
            rc = fn(_ptr(packed), F, L.make_grid(*grid), int(n0), count, policy, _ptr(out),
                    _ptr(flags), _ptr(ws), wsb, st)
    else:
        if strip is None:
            strip = points is None and lattice_paths(mesh, mode, precision, grid, n0, count)[0]
        if strip and mode != "exact":
            raise ValueError("strip records exist for the exact forward only")
        if strip:
            kind = L.PACK_EXACTSTRIP_F64
        packed = mesh.packed(kind)
        if strip:
            if points is not None:
                rc = lib.wv_exact_strip_fwd_points_f64(_ptr(packed), F, _ptr(pts), count,
                                                       int(bool(use_atan2)), policy, _ptr(out),
                                                       _ptr(flags), st)
            else:
                rc = lib.wv_exact_strip_fwd_grid_f64(_ptr(packed), F, L.make_grid(*grid),
                                                     int(n0), count, int(bool(use_atan2)),
                                                     policy, _ptr(out), _ptr(flags), st)
        elif mode == "exact":
            if points is not None:
                rc = lib.wv_exact_fwd_points_f64(_ptr(packed), F, _ptr(pts), count,
                                                 int(bool(use_atan2)), policy, _ptr(out),
                                                 _ptr(flags), st)
            else:
                rc = lib.wv_exact_fwd_grid_f64(_ptr(packed), F, L.make_grid(*grid), int(n0),
                                               count, int(bool(use_atan2)), policy, _ptr(out),
                                               _ptr(flags), st)
        else:
            if points is not None:
                rc = lib.wv_soft_fwd_points_f64(_ptr(packed), F, _ptr(pts), count, policy,
                                                _ptr(out), _ptr(flags), st)
            else:
                rc = lib.wv_soft_fwd_grid_f64(_ptr(packed), F, L.make_grid(*grid), int(n0), count,
                                              policy, _ptr(out), _ptr(flags), st)
    L.check(rc, f"{mode} forward ({precision})")
    return out, flags


def exact_forward_f32(mesh: DeviceMesh, **kw):
    return forward(mesh, "exact", "f32", **kw)


def trail_rows_ok(grid, n0: int) -> bool:
    """The edge-trail backward runs on lattice rows only: k-rows of >= 16
    nodes, an even row length and an even range start."""
    rz = int(grid[2][2])
    return rz >= 16 and rz % 2 == 0 and int(n0) % 2 == 0


# The f32 trail kernel shares ONE reciprocal among four edge denominators
# (~|x|^8 in the power-of-two frame where the lattice's largest coordinate is
# in [1, 2)); meshes reaching beyond this many lattice extents keep the
# face kernels (3-fold products), so the product stays far inside f32 range.
TRAIL_MAX_MESH_EXTENT = 1024.0


def trail_scale_ok(mesh: "DeviceMesh", grid) -> bool:
    ext = max(max(abs(float(x)) for x in grid[0]), max(abs(float(x)) for x in grid[1]))
    return ext > 0.0 and mesh.abs_max() <= TRAIL_MAX_MESH_EXTENT * ext


def face_grad(mesh: DeviceMesh, mode: str, precision: str, coefs: torch.Tensor, *, grid=None,
              n0: int = 0, count: int | None = None, points=None, coef_scale: float = 1.0,
              pairs: bool | None = None, trails: bool | None = None):
    """Per-face corner gradients sum_p coef_scale*coefs[p]*dW_p/dv, f64.
    Returns (corner_grad (A,3,3), csr) where the rows are all faces (soft) or
    the active faces of the exact edge form (exact) -- or, for the edge-trail
    backward, the (2KW,3) end vectors of the trail windows' edges with a
    signed CSR; feed both to ``vertex_grad``.  Exact mode expects coefs == 0
    at flagged points.  ``trails`` / ``pairs``: force (True) or forbid (False)
    those records; None = automatic (large row-aligned lattice ranges of a
    mesh whose corner positions are shared take the trails)."""
    _check_precision(precision)
    lib = L.lib()
    dev = mesh.vertices.device
    dt = _DT[precision]
    if points is not None:
        n_pts = int(torch.as_tensor(points).reshape(-1, 3).shape[0])
    else:
        n_pts = _grid_count(grid, n0, count)
    exact32 = mode == "exact" and precision == "f32"
    exact64 = mode == "exact" and precision == "f64"
    if trails is None:
        trails = pairs is None and (
            (exact32 and points is None and n_pts >= STRIP_MIN_NODES
             and trail_rows_ok(grid, n0) and mesh.trails_pay() and trail_scale_ok(mesh, grid))
            or (exact64 and n_pts >= TRAIL64_MIN_POINTS and mesh.trails_pay()))
    if trails:
        if not (exact64 or (exact32 and points is None and trail_rows_ok(grid, n0))):
            raise ValueError("edge trails exist for the exact backward (f32: lattice rows only)")
        return _trail_grad(mesh, coefs, precision, grid, n0, n_pts, points, coef_scale)
    if pairs is None:
        pairs = (exact32 and n_pts >= STRIP_MIN_NODES and mesh.num_faces > 0
                 and mesh.strips_pay())
    if pairs and not exact32:
        raise ValueError("strip pairs exist for the exact f32 backward only")
    if pairs:
        kind = None
        packed = mesh.packed_exact_pair()
        rows_f, _, csr, _ = mesh.exact_pair_setup()
        F = int(rows_f.shape[0])
    elif mode == "exact":
        kind = _EXACTGRAD[precision]
        packed = mesh.packed_exact_grad(precision)
        active, _, csr = mesh.exact_grad_setup()
        F = int(active.shape[0])
    elif mode == "soft":
        kind = _SOFTGRAD[precision]
        packed = mesh.packed(kind)
        csr = mesh.csr()
        F = mesh.num_faces
    else:
        raise ValueError(f"mode must be 'exact' or 'soft', got {mode!r}")
    if points is not None:
        pts, count = _points_arg(points, dev, dt)
    else:
        count = _grid_count(grid, n0, count)
    cf = coefs.to(device=dev, dtype=dt).contiguous().reshape(-1)
    if cf.numel() != count:
        raise ValueError(f"coefs has {cf.numel()} entries for {count} query points")
    out = torch.empty((F, 3, 3), dtype=torch.float64, device=dev)
    if F == 0:
        return out, csr
    if pairs:
        wsb = int(lib.wv_exact_pair_bwd_workspace_bytes(F, count))
    else:
        wsb = int(lib.wv_bwd_workspace_bytes(kind, F, count))
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev) if wsb else None
    st = _stream()
    name = f"wv_{mode}_bwd_{'points' if points is not None else 'grid'}_{precision}"
    if pairs:
        name = f"wv_exact_pair_bwd_{'points' if points is not None else 'grid'}_f32"
    fn = getattr(lib, name)
    if points is not None:
        rc = fn(_ptr(packed), F, _ptr(pts), count, _ptr(cf), float(coef_scale), _ptr(out),
                _ptr(ws), wsb, st)
    else:
        rc = fn(_ptr(packed), F, L.make_grid(*grid), int(n0), count, _ptr(cf), float(coef_scale),
                _ptr(out), _ptr(ws), wsb, st)
    L.check(rc, name)
    return out, csr


def _trail_grad(mesh: DeviceMesh, coefs: torch.Tensor, precision: str, grid, n0: int,
                count: int, points, coef_scale: float):
    """face_grad over edge trails: (end vectors (2KW,3) f64, signed CSR)."""
    lib = L.lib()
    dev = mesh.vertices.device
    dt = _DT[precision]
    packed = mesh.packed_exact_trail(precision)
    win, csr, W, _ = mesh.exact_trail_setup()
    cf = coefs.to(device=dev, dtype=dt).contiguous().reshape(-1)
    if cf.numel() != count:
        raise ValueError(f"coefs has {cf.numel()} entries for {count} query points")
    out = torch.empty((2 * (int(win.shape[1]) - 1) * W, 3), dtype=torch.float64, device=dev)
    if W == 0:
        return out, csr
    sfx = "" if precision == "f32" else "_f64"
    wsb = int(getattr(lib, f"wv_exact_trail_bwd_workspace_bytes{sfx}")(W, count))
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev) if wsb else None
    if points is not None:
        pts, _ = _points_arg(points, dev, dt)
        name = "wv_exact_trail_bwd_points_f64"
        rc = lib.wv_exact_trail_bwd_points_f64(_ptr(packed), W, _ptr(pts), count, _ptr(cf),
                                               float(coef_scale), _ptr(out), _ptr(ws), wsb,
                                               _stream())
    else:
        name = f"wv_exact_trail_bwd_grid_{precision}"
        rc = getattr(lib, name)(_ptr(packed), W, L.make_grid(*grid), int(n0), count, _ptr(cf),
                                float(coef_scale), _ptr(out), _ptr(ws), wsb, _stream())
    L.check(rc, name)
    return out, csr


def vertex_grad(mesh: DeviceMesh, fgrad, *, scale: torch.Tensor | None = None,
                dtype=torch.float64, out: torch.Tensor | None = None,
                accumulate: bool = False) -> torch.Tensor:
    """(V,3) vertex gradients from ``face_grad``'s (corner_grad, csr)."""
    lib = L.lib()
    dev = mesh.vertices.device
    fg, (off, slots) = fgrad
    V = mesh.num_vertices
    if out is None:
        out = torch.zeros((V, 3), dtype=dtype, device=dev)
    o64 = out if out.dtype == torch.float64 else None
    o32 = out if out.dtype == torch.float32 else None
    L.check(lib.wv_face_to_vertex(_ptr(fg), _ptr(off), _ptr(slots), V, _ptr(scale),
                                  int(accumulate), _ptr(o64), _ptr(o32), _stream()),
            "wv_face_to_vertex")
    return out


def loss_terms(values: torch.Tensor, flags: torch.Tensor, targets: torch.Tensor,
               weights: torch.Tensor | None = None):
    """(coefs = 2 w r, sums[8]) on the device (see include/windvox_b200.h)."""
    lib = L.lib()
    dev = values.device
    n = int(values.numel())
    dt = values.dtype
    tg = targets.to(device=dev, dtype=dt).contiguous()
    wt = None if weights is None else weights.to(device=dev, dtype=dt).contiguous()
    coefs = torch.empty_like(values)
    sums = torch.zeros(8, dtype=torch.float64, device=dev)
    wsb = int(lib.wv_loss_workspace_bytes(n))
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    fn = lib.wv_loss_terms_f32 if dt == torch.float32 else lib.wv_loss_terms_f64
    L.check(fn(_ptr(values), _ptr(flags), _ptr(tg), _ptr(wt), n, _ptr(coefs), _ptr(sums),
               _ptr(ws), wsb, _stream()), "wv_loss_terms")
    return coefs, sums


def loss_finalize(sums: torch.Tensor) -> torch.Tensor:
    L.check(L.lib().wv_loss_finalize(_ptr(sums), _stream()), "wv_loss_finalize")
    return sums
