"""Batched occupancy loss over many meshes sharing one grid (config C4, the
"mesh-morphing training batch": 64 meshes x ~5k faces at 64^3).

``BatchOccupancyLoss`` is a torch.autograd.Function over a (B,V,3) batch of
vertex positions with fixed connectivity: its forward runs, per mesh, the
device path of ``occupancy_loss_grad`` -- soft (or exact) forward, fused loss
terms, backward and vertex gather, all on the GPU -- and keeps the gradients;
its backward only scales them by the incoming per-mesh loss gradients.  So a
deformation network upstream gets d loss / d vertices for every mesh at the
cost of one fused pass, and nothing but the B loss scalars ever reaches the
host.  Per-mesh semantics are the reference's (grad.py:71-127): weighted MSE
over unflagged nodes, normalised by the weight sum.
"""

from __future__ import annotations

import torch

from . import _lib as L
from .device import DeviceMesh, _ptr, _stream
from .grad import device_loss_grad

__all__ = ["BatchOccupancyLoss", "batch_occupancy_loss", "DeformationNet"]


# meshes are independent: round-robin them over a few streams so one mesh's
# kernels fill the wave tails of another's (each mesh alone is ~1 ms of work)
N_STREAMS = 4
_STREAMS: dict = {}


def _side_streams(dev):
    st = _STREAMS.get(dev)
    if st is None:
        st = [torch.cuda.Stream(device=dev) for _ in range(N_STREAMS)]
        _STREAMS[dev] = st
    return st


def _grid_count(grid) -> int:
    r = grid[2]
    return int(r[0]) * int(r[1]) * int(r[2])


def batched_soft_loss_grad_f32(verts: torch.Tensor, faces: torch.Tensor, grid,
                               targets: torch.Tensor, csr):
    """Soft occupancy loss and its vertex gradients for a (B,V,3) batch with
    one connectivity, by ONE forward and ONE backward launch for the whole
    batch (include/windvox_b200.h "batched grid kernels"; blockIdx.z = mesh),
    with batched packing, loss terms and CSR gathers around them (about ten
    launches per batch instead of seven per mesh).  Returns
    (losses (B,) f64, grads (B,V,3) f32, sums (B,8) f64); every mesh's
    numbers equal the single-mesh path's (``device_loss_grad``)."""
    lib = L.lib()
    dev = verts.device
    B, V, _ = verts.shape
    F = int(faces.shape[0])
    N = _grid_count(grid)
    g = L.make_grid(*grid)
    st = _stream()
    v32 = verts.detach().to(torch.float32).contiguous()
    f64i = faces.to(torch.int64).contiguous()

    def pack(kind):
        stride = (int(lib.wv_packed_bytes(kind, F)) + 15) // 16 * 16
        buf = torch.empty(B * stride, dtype=torch.uint8, device=dev)
        L.check(lib.wv_pack_faces_batch(kind, _ptr(v32), 0, V, _ptr(f64i), 1, F, B, _ptr(buf),
                                        stride, st), "wv_pack_faces_batch")
        return buf, stride

    fbuf, fstride = pack(L.PACK_SOFT_F32)
    gbuf, gstride = pack(L.PACK_SOFTGRAD_F32)
    vals = torch.empty((B, N), dtype=torch.float32, device=dev)
    flags = torch.empty((B, N), dtype=torch.uint8, device=dev)
    wsb = max(int(lib.wv_fwd_workspace_bytes_batch(L.PACK_SOFT_F32, F, N, B)),
              int(lib.wv_bwd_workspace_bytes_batch(L.PACK_SOFTGRAD_F32, F, N, B)))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    L.check(lib.wv_fwd_grid_f32_batch(L.PACK_SOFT_F32, _ptr(fbuf), fstride, F, g, 0, N, B,
                                      L.POLICY_RAW, _ptr(vals), _ptr(flags), _ptr(ws), wsb, st),
            "wv_fwd_grid_f32_batch")
    tg = targets.to(device=dev, dtype=torch.float32).reshape(B, N).contiguous()
    coefs = torch.empty((B, N), dtype=torch.float32, device=dev)
    sums = torch.zeros((B, 8), dtype=torch.float64, device=dev)
    lwsb = B * int(lib.wv_loss_workspace_bytes(N))
    lws = torch.empty(max(lwsb, 1), dtype=torch.uint8, device=dev)
    L.check(lib.wv_loss_terms_f32_batch(_ptr(vals), _ptr(flags), _ptr(tg), None, N, B,
                                        _ptr(coefs), _ptr(sums), _ptr(lws), lwsb, st),
            "wv_loss_terms_f32_batch")
    fg = torch.empty((B, F, 3, 3), dtype=torch.float64, device=dev)
    L.check(lib.wv_bwd_grid_f32_batch(L.PACK_SOFTGRAD_F32, _ptr(gbuf), gstride, F, g, 0, N, B,
                                      _ptr(coefs), 1.0, _ptr(fg), _ptr(ws), wsb, st),
            "wv_bwd_grid_f32_batch")
    grads = torch.empty((B, V, 3), dtype=torch.float32, device=dev)
    off, slots = csr
    # 1/sum(w) (sums[b][3]) applied on the device by the gather
    L.check(lib.wv_face_to_vertex_batch(_ptr(fg), F, _ptr(off), _ptr(slots), V, B,
                                        _ptr(sums) + 3 * 8, 8, 0, None, _ptr(grads), st),
            "wv_face_to_vertex_batch")
    return sums[:, 4].clone(), grads, sums


class BatchOccupancyLoss(torch.autograd.Function):
    @staticmethod
    def forward(ctx, verts, faces, grid, targets, mode, precision, csr):
        B = verts.shape[0]
        if mode == "soft" and precision == "f32" and verts.dtype == torch.float32:
            losses, grads, _ = batched_soft_loss_grad_f32(verts, faces, grid, targets, csr)
            ctx.save_for_backward(grads)
            return losses
        losses = torch.empty(B, dtype=torch.float64, device=verts.device)
        grads = torch.empty((B,) + tuple(verts.shape[1:]), dtype=verts.dtype,
                            device=verts.device)
        main = torch.cuda.current_stream(verts.device)
        side = _side_streams(verts.device)
        for s in side:
            s.wait_stream(main)
        for b in range(B):
            with torch.cuda.stream(side[b % len(side)]):
                m = DeviceMesh(verts[b].detach().contiguous(), faces, _csr=csr)
                sums, g = device_loss_grad(m, grid, targets[b], None, mode=mode,
                                           precision=precision)
                losses[b] = sums[4]
                grads[b] = (g * sums[3]).to(verts.dtype)
        for s in side:
            main.wait_stream(s)
        ctx.save_for_backward(grads)
        return losses

    @staticmethod
    def backward(ctx, grad_losses):
        (grads,) = ctx.saved_tensors
        return (grads * grad_losses.to(grads.dtype)[:, None, None], None, None, None, None, None,
                None)


def batch_occupancy_loss(verts: torch.Tensor, faces: torch.Tensor, grid, targets: torch.Tensor,
                         *, mode: str = "soft", precision: str = "f32", csr=None):
    """Per-mesh occupancy losses (B,) with autograd to ``verts`` (B,V,3)."""
    if csr is None:
        csr = DeviceMesh(verts[0].detach(), faces).csr()
    return BatchOccupancyLoss.apply(verts, faces, grid, targets, mode, precision, csr)


class DeformationNet(torch.nn.Module):
    """MLP [xyz + per-mesh latent] -> displacement (hidden
    128 x 2, 32-d latent)."""

    def __init__(self, n_meshes: int, latent: int = 32, hidden: int = 128):
        super().__init__()
        self.latent = torch.nn.Parameter(torch.zeros(n_meshes, latent))
        self.mlp = torch.nn.Sequential(
            torch.nn.Linear(3 + latent, hidden), torch.nn.ReLU(),
            torch.nn.Linear(hidden, hidden), torch.nn.ReLU(),
            torch.nn.Linear(hidden, 3))
        with torch.no_grad():  # start near the identity map
            self.mlp[-1].weight.mul_(0.01)
            self.mlp[-1].bias.zero_()

    def forward(self, template: torch.Tensor, mesh_ids: torch.Tensor) -> torch.Tensor:
        """template (B,V,3) -> deformed (B,V,3)."""
        B, V, _ = template.shape
        z = self.latent[mesh_ids][:, None, :].expand(B, V, self.latent.shape[1])
        return template + self.mlp(torch.cat([template, z], dim=-1))
