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

from .device import DeviceMesh
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


class BatchOccupancyLoss(torch.autograd.Function):
    @staticmethod
    def forward(ctx, verts, faces, grid, targets, mode, precision, csr):
        B = verts.shape[0]
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
