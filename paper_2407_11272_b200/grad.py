"""Reference-compatible gradient API on the B200 kernels.

Mirrors /root/reference/pkg/src/windvox/grad.py:
  soft_winding_vertex_jacobian (:54-68), occupancy_loss_grad (:71-127).
Adds the exact-mode counterpart the reference deliberately leaves out
(grad.py:9-12): ``exact_loss_grad`` differentiates the same loss through the
closed-form d(Omega)/dv of the Van Oosterom-Strackee solid angle.

Everything after the host->device copy of the mesh and targets stays on the
GPU: forward -> fused loss terms -> backward -> CSR vertex gather, with the
1/sum(w) normalisation read on the device.  ``precision="f64"`` (default,
as the reference) runs the f64 parity kernels; ``"f32"`` the FP32 hot path.
"""

from __future__ import annotations

import numpy as np
import torch

from .device import DeviceMesh, face_grad, forward, loss_terms, vertex_grad
from .errors import OnSurfaceError
from .types import LossReport, QueryBatchConfig, ScalarField, TriangleMesh, VertexGradients

__all__ = ["VertexGradients", "LossReport", "soft_winding_vertex_jacobian",
           "occupancy_loss_grad", "exact_loss_grad", "device_loss_grad"]


def soft_winding_vertex_jacobian(mesh: TriangleMesh, q, *,
                                 precision: str = "f64") -> VertexGradients:
    """dW_soft(q)/dV, shape (V,3); raises OnSurfaceError on a face centroid."""
    dmesh = DeviceMesh.from_numpy(mesh.vertices, mesh.faces)
    dt = torch.float64 if precision == "f64" else torch.float32
    pt = torch.as_tensor(np.asarray(q, dtype=np.float64).reshape(1, 3), dtype=dt,
                         device=dmesh.vertices.device)
    _, flags = forward(dmesh, "soft", precision, points=pt)
    if bool(flags[0].item()):
        raise OnSurfaceError("query point lies on a face centroid")
    coefs = torch.ones(1, dtype=dt, device=pt.device)
    fg = face_grad(dmesh, "soft", precision, coefs, points=pt)
    return VertexGradients(vertex_grad(dmesh, fg).cpu().numpy())


def device_loss_grad(dmesh: DeviceMesh, grid, targets: torch.Tensor,
                     weights: torch.Tensor | None = None, *, mode: str = "soft",
                     precision: str = "f32", n0: int = 0, count: int | None = None,
                     grad_out: torch.Tensor | None = None):
    """Device-resident loss + gradient over the node range [n0, n0+count) of
    ``grid``: returns (sums[8] f64 device tensor, vertex gradient numerator
    (V,3) f64, i.e. NOT yet divided by sum(w)).  The multi-GPU driver
    all-reduces both before normalising; single-GPU callers use
    ``normalize``."""
    vals, flags = forward(dmesh, mode, precision, grid=grid, n0=n0, count=count)
    coefs, sums = loss_terms(vals, flags, targets, weights)
    fg = face_grad(dmesh, mode, precision, coefs, grid=grid, n0=n0, count=count)
    g = vertex_grad(dmesh, fg, out=grad_out)
    return sums, g


def _loss_grad(mesh, targets: ScalarField, weights, mode: str, precision: str) -> LossReport:
    if mesh.num_faces == 0:
        raise ValueError("cannot evaluate occupancy loss for an empty mesh")
    n = targets.spec.num_nodes
    if weights is not None:
        w = np.asarray(weights, dtype=np.float64).reshape(n)
        if np.any(w < 0):
            raise ValueError("weights must be non-negative")
    dmesh = DeviceMesh.from_numpy(mesh.vertices, mesh.faces)
    dev = dmesh.vertices.device
    dt = torch.float64 if precision == "f64" else torch.float32
    tg = torch.as_tensor(np.asarray(targets.values, dtype=np.float64), dtype=dt).to(dev)
    wt = None if weights is None else torch.as_tensor(w, dtype=dt).to(dev)
    spec = targets.spec
    grid = (spec.bounds_min, spec.bounds_max, spec.resolution)
    sums, g = device_loss_grad(dmesh, grid, tg, wt, mode=mode, precision=precision)
    s = sums.cpu().numpy()
    if s[1] == 0.0:
        raise ValueError("no usable grid nodes: all excluded or zero-weighted")
    grads = g.cpu().numpy() * s[3]
    return LossReport(loss=float(s[4]), grads=VertexGradients(grads), excluded_nodes=int(s[2]))


def occupancy_loss_grad(mesh: TriangleMesh, targets: ScalarField,
                        weights: np.ndarray | None = None,
                        batch: QueryBatchConfig | None = None, *,
                        precision: str = "f64") -> LossReport:
    """Weighted MSE between the soft winding number and ``targets`` over the
    target grid's unflagged nodes, with its exact vertex gradient."""
    return _loss_grad(mesh, targets, weights, "soft", precision)


def exact_loss_grad(mesh: TriangleMesh, targets: ScalarField,
                    weights: np.ndarray | None = None,
                    batch: QueryBatchConfig | None = None, *,
                    precision: str = "f64") -> LossReport:
    """Same loss on the EXACT winding number, differentiated through the
    closed-form d(Omega)/dv (nonzero only where the surface sweeps past
    nodes' solid angles, e.g. near open rims)."""
    return _loss_grad(mesh, targets, weights, "exact", precision)
