"""torch.autograd binding of the winding-number kernels.

The reference has no autograd layer (its "differentiable" API returns numpy
gradients, grad.py:54-127); this is the torch surface north_star asks for:

    W, flags = winding_number(vertices, faces, grid=(lo, hi, res))   # or points=
    loss = ((W - target) ** 2).mean(); loss.backward()               # -> vertices.grad

backward(grad_W) = sum_p grad_W[p] * dW_p/dV: exactly the reference's
``soft_grad_accum`` with ``coefs = grad_W`` in soft mode (_kernels.py:161-232)
and the closed-form d(Omega)/dv in exact mode.  Pairs the forward skipped
(on-surface) carry no gradient, as in the reference (_kernels.py:182-184,
203-204).  FP32 vertices run the FP32 kernels, FP64 vertices the f64 parity
kernels.  Everything stays on the device.
"""

from __future__ import annotations

import torch

from . import _lib as L
from .device import DeviceMesh, face_grad, forward, vertex_grad


def _precision(vertices: torch.Tensor, precision: str | None) -> str:
    if precision is not None:
        return precision
    return "f64" if vertices.dtype == torch.float64 else "f32"


class _WindingNumberFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, vertices, layer, points):
        mesh = layer._mesh_for(vertices.detach())
        prec = layer.precision_for(vertices)
        if points is not None:
            W, flags = forward(mesh, layer.mode, prec, points=points.detach(),
                               policy=layer.policy)
        else:
            W, flags = forward(mesh, layer.mode, prec, grid=layer.grid, n0=layer.n0,
                               count=layer.count, policy=layer.policy)
        ctx.layer = layer
        ctx.mesh = mesh
        ctx.prec = prec
        ctx.vdtype = vertices.dtype
        ctx.save_for_backward(points if points is not None else torch.empty(0), flags)
        ctx.has_points = points is not None
        ctx.mark_non_differentiable(flags)
        return W, flags

    @staticmethod
    def backward(ctx, grad_W, _grad_flags):
        if grad_W is None or not ctx.needs_input_grad[0]:
            return None, None, None
        points, flags = ctx.saved_tensors
        layer = ctx.layer
        coefs = grad_W.contiguous()
        if layer.policy == L.POLICY_HALF or layer.mode == "exact":
            # voxelize policy: flagged nodes hold the constant 0.5; exact mode:
            # W jumps across the surface, so on-surface nodes have no derivative
            coefs = torch.where(flags.bool(), torch.zeros_like(coefs), coefs)
        if ctx.has_points:
            fg = face_grad(ctx.mesh, layer.mode, ctx.prec, coefs, points=points)
        else:
            fg = face_grad(ctx.mesh, layer.mode, ctx.prec, coefs, grid=layer.grid, n0=layer.n0,
                           count=layer.count)
        g = vertex_grad(ctx.mesh, fg, dtype=ctx.vdtype)
        return g, None, None


class WindingNumber(torch.nn.Module):
    """Differentiable winding-number field of a mesh with fixed connectivity.

    ``faces`` (F,3) int tensor; either ``grid=(lo, hi, res)`` (optionally the
    node range [n0, n0+count) for slab sharding) or per-call ``points``.
    Calling the module with vertex positions (V,3) returns (W, flags)."""

    def __init__(self, faces: torch.Tensor, *, grid=None, n0: int = 0, count: int | None = None,
                 mode: str = "exact", precision: str | None = None, voxelize: bool = False):
        super().__init__()
        if mode not in ("exact", "soft"):
            raise ValueError(f"mode must be 'exact' or 'soft', got {mode!r}")
        self.faces = faces
        self.grid = grid
        self.n0 = int(n0)
        self.count = count
        self.mode = mode
        self.precision = precision
        self.policy = L.POLICY_HALF if voxelize else L.POLICY_RAW
        self._mesh: DeviceMesh | None = None

    def precision_for(self, vertices):
        return _precision(vertices, self.precision)

    def _mesh_for(self, vertices: torch.Tensor) -> DeviceMesh:
        """A fresh DeviceMesh snapshot per call (a later forward must not
        change what an earlier graph's backward sees), sharing the static
        connectivity and its vertex CSR."""
        if self._mesh is None or self._mesh.vertices.device != vertices.device:
            faces = self.faces.to(vertices.device).contiguous()
            self._mesh = DeviceMesh(vertices.contiguous(), faces)
            self._mesh.csr()
            if self.mode == "exact":
                self._mesh.exact_grad_setup()
        m = DeviceMesh(vertices.contiguous(), self._mesh.faces, _csr=self._mesh._csr)
        m._faces_np = self._mesh._faces_np
        if self.mode == "exact":
            m._exact_grad = self._mesh._exact_grad
        return m

    def forward(self, vertices: torch.Tensor, points: torch.Tensor | None = None):
        if points is None and self.grid is None:
            raise ValueError("give either a grid at construction or points per call")
        return _WindingNumberFn.apply(vertices, self, points)


def winding_number(vertices: torch.Tensor, faces: torch.Tensor, *, grid=None, points=None,
                   mode: str = "exact", precision: str | None = None, voxelize: bool = False):
    """Functional form: (W, flags) with autograd to ``vertices``."""
    layer = WindingNumber(faces, grid=grid, mode=mode, precision=precision, voxelize=voxelize)
    return layer(vertices, points)
