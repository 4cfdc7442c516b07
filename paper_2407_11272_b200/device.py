"""Device-side staging and kernel launches (torch tensors for memory and
streams, the C ABI for every computation).

``DeviceMesh`` holds a mesh resident in HBM and lazily packs the per-kind
face records (``wv_pack_faces``), so a morph loop or a multi-call voxelize
re-packs only when the vertices change.  Every launch is stream-ordered on
torch's current stream; nothing here synchronises the host.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def device() -> torch.device:
    L.lib()
    return torch.device("cuda", torch.cuda.current_device())


@dataclass
class DeviceMesh:
    """Mesh resident on the GPU.  ``vertices`` (V,3) f32/f64, ``faces``
    (F,3) int32/int64, both contiguous CUDA tensors."""

    vertices: torch.Tensor
    faces: torch.Tensor
    _packs: dict = field(default_factory=dict, repr=False)
    _version: int = field(default=-1, repr=False)

    @classmethod
    def from_numpy(cls, vertices: np.ndarray, faces: np.ndarray, dev=None,
                   dtype=torch.float64) -> "DeviceMesh":
        dev = dev or device()
        v = torch.as_tensor(np.ascontiguousarray(vertices), dtype=dtype).reshape(-1, 3)
        f = torch.as_tensor(np.ascontiguousarray(faces, dtype=np.int64)).reshape(-1, 3)
        if dev.type == "cuda":
            v = v.pin_memory().to(dev, non_blocking=True)
            f = f.pin_memory().to(dev, non_blocking=True)
        return cls(v.contiguous(), f.contiguous())

    @property
    def num_vertices(self) -> int:
        return int(self.vertices.shape[0])

    @property
    def num_faces(self) -> int:
        return int(self.faces.shape[0])

    def invalidate(self) -> None:
        self._packs.clear()

    def packed(self, kind: int) -> torch.Tensor:
        ver = self.vertices._version
        if ver != self._version:
            self._packs.clear()
            self._version = ver
        buf = self._packs.get(kind)
        if buf is not None:
            return buf
        lib = L.lib()
        if not (self.vertices.is_cuda and self.faces.is_cuda):
            raise ValueError("DeviceMesh tensors must live on a CUDA device")
        v = self.vertices.contiguous()
        f = self.faces.contiguous()
        if v.dtype not in (torch.float32, torch.float64):
            raise TypeError("vertices must be float32 or float64")
        if f.dtype not in (torch.int32, torch.int64):
            raise TypeError("faces must be int32 or int64")
        nbytes = int(lib.wv_packed_bytes(kind, self.num_faces))
        buf = torch.empty(nbytes, dtype=torch.uint8, device=v.device)
        L.check(lib.wv_pack_faces(kind, _ptr(v), int(v.dtype == torch.float64),
                                  self.num_vertices, _ptr(f), int(f.dtype == torch.int64),
                                  self.num_faces, _ptr(buf), _stream()), "wv_pack_faces")
        self._packs[kind] = buf
        return buf


def _workspace(kind: int, n_faces: int, count: int, dev) -> tuple[torch.Tensor | None, int]:
    nbytes = int(L.lib().wv_fwd_workspace_bytes(kind, n_faces, count))
    if nbytes == 0:
        return None, 0
    return torch.empty(nbytes, dtype=torch.uint8, device=dev), nbytes


def exact_forward_f32(mesh: DeviceMesh, *, grid=None, n0: int = 0, count: int | None = None,
                      points: torch.Tensor | None = None, policy: int = L.POLICY_RAW,
                      out: torch.Tensor | None = None, flags: torch.Tensor | None = None):
    """FP32 exact winding numbers.  Either ``grid=(lo, hi, res)`` with the
    node range [n0, n0+count), or ``points`` (n,3) float32 on the device.
    Returns (values f32, flags u8) device tensors."""
    lib = L.lib()
    dev = mesh.vertices.device
    packed = mesh.packed(L.PACK_EXACT_F32)
    if points is not None:
        pts = points.to(device=dev, dtype=torch.float32).contiguous().reshape(-1, 3)
        count = int(pts.shape[0])
    else:
        lo, hi, res = grid
        if count is None:
            count = int(res[0]) * int(res[1]) * int(res[2]) - n0
    out = torch.empty(count, dtype=torch.float32, device=dev) if out is None else out
    flags = torch.empty(count, dtype=torch.uint8, device=dev) if flags is None else flags
    if count == 0:
        return out, flags
    ws, wsb = _workspace(L.PACK_EXACT_F32, mesh.num_faces, count, dev)
    if points is not None:
        rc = lib.wv_exact_fwd_points_f32(_ptr(packed), mesh.num_faces, _ptr(pts), count,
                                         policy, _ptr(out), _ptr(flags), _ptr(ws), wsb,
                                         _stream())
    else:
        rc = lib.wv_exact_fwd_grid_f32(_ptr(packed), mesh.num_faces, L.make_grid(lo, hi, res),
                                       int(n0), count, policy, _ptr(out), _ptr(flags),
                                       _ptr(ws), wsb, _stream())
    L.check(rc, "wv_exact_fwd")
    return out, flags
