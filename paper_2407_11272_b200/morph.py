"""Occupancy-supervised mesh morphing with every loss/gradient evaluation on
the GPU -- the "mesh-morphing loop" caller of the hot path.

Same algorithm, configuration and report as the reference
(/root/reference/pkg/src/windvox/morph.py:35-207): gradient descent with
momentum, step-halving backtracking that only accepts non-increasing steps
(8 momentum trials, then 12 plain ones), and a uniform-Laplacian smoothness
term ``smooth_weight * sum_v |v - mean(nbrs)|^2``.  What changes is where
the state lives: vertices, the target grid, the packed face records, the
vertex CSR and the Laplacian stay in HBM across iterations; each trial is a
soft forward + fused loss (2-21 per iteration, forward only) and each
accepted step one soft forward + backward + gather.  The only host traffic
per trial is the scalar loss needed by the accept rule.

``precision="f64"`` (default) runs the f64 parity kernels, so the trace
matches the reference's to rounding (tests/test_gpu_morph.py); ``"f32"``
runs the FP32 path.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .device import DeviceMesh, face_grad, forward, loss_terms, vertex_grad
from .errors import DivergedError
from .types import GridSpec, QueryBatchConfig, ScalarField, TriangleMesh

__all__ = ["MorphConfig", "MorphReport", "morph", "uniform_laplacian"]

_MOMENTUM_HALVINGS = 8
_PLAIN_HALVINGS = 12


@dataclass(frozen=True)
class MorphConfig:
    """Optimizer settings (reference morph.py:35-62)."""

    step_size: float = 0.05
    momentum: float = 0.9
    iterations: int = 300
    smooth_weight: float = 1e-3
    grid: GridSpec | None = None
    log_every: int = 1
    batch: QueryBatchConfig = field(default_factory=QueryBatchConfig)

    def __post_init__(self):
        if self.step_size < 0.0:
            raise ValueError("step_size must be >= 0")
        if not 0.0 <= self.momentum < 1.0:
            raise ValueError("momentum must be in [0, 1)")
        if self.iterations < 0:
            raise ValueError("iterations must be >= 0")
        if self.smooth_weight < 0.0:
            raise ValueError("smooth_weight must be >= 0")
        if self.log_every < 1:
            raise ValueError("log_every must be >= 1")


@dataclass
class MorphReport:
    """{iter, loss, grad_inf_norm} entries for iteration 0, every
    ``log_every``-th iteration and the final one."""

    entries: list = field(default_factory=list)
    final_mesh_path: str | None = None


def uniform_laplacian(faces: np.ndarray, n_verts: int):
    """L = I - D^-1 A over the undirected edge graph, restricted to vertices
    that have neighbours (zero rows elsewhere), as (indptr, indices, data)
    CSR arrays -- the reference's construction (morph.py:78-92), built once
    on the host since the connectivity never changes."""
    import scipy.sparse as sp
    f = np.asarray(faces, dtype=np.int64).reshape(-1, 3)
    e = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]])
    e = np.unique(np.sort(e, axis=1), axis=0)
    both = (np.concatenate([e[:, 0], e[:, 1]]), np.concatenate([e[:, 1], e[:, 0]]))
    adj = sp.csr_matrix((np.ones(len(both[0])), both), shape=(n_verts, n_verts))
    deg = np.asarray(adj.sum(axis=1)).ravel()
    has = deg > 0
    inv = np.where(has, 1.0 / np.where(has, deg, 1.0), 0.0)
    lap = (sp.diags(has.astype(np.float64)) - sp.diags(inv) @ adj).tocsr()
    lap.sort_indices()
    return (lap.indptr.astype(np.int64), lap.indices.astype(np.int64),
            lap.data.astype(np.float64))


class _DeviceProblem:
    """Everything the loop touches, resident on the GPU."""

    def __init__(self, template: TriangleMesh, target: ScalarField, cfg: MorphConfig,
                 precision: str):
        self.prec = precision
        self.dt = torch.float64 if precision == "f64" else torch.float32
        self.cfg = cfg
        self.mesh = DeviceMesh.from_numpy(template.vertices, template.faces, dtype=self.dt)
        self.mesh.csr()
        dev = self.mesh.vertices.device
        spec = target.spec
        self.grid = (spec.bounds_min, spec.bounds_max, spec.resolution)
        self.targets = torch.as_tensor(np.asarray(target.values, dtype=np.float64),
                                       dtype=self.dt).to(dev)
        ip, ix, dv = uniform_laplacian(template.faces, template.num_vertices)
        V = template.num_vertices
        self.L = torch.sparse_csr_tensor(torch.from_numpy(ip), torch.from_numpy(ix),
                                         torch.from_numpy(dv), size=(V, V),
                                         check_invariants=True).to(dev, self.dt)
        self.LT = self.L.to_sparse_coo().t().coalesce().to_sparse_csr()

    def _occupancy(self, verts: torch.Tensor):
        self.mesh.set_vertices(verts)
        vals, flags = forward(self.mesh, "soft", self.prec, grid=self.grid)
        coefs, sums = loss_terms(vals, flags, self.targets)
        return coefs, sums

    def _smooth(self, verts):
        lv = self.L @ verts
        return (lv * lv).sum(), lv

    def loss_only(self, verts: torch.Tensor) -> float:
        _, sums = self._occupancy(verts)
        e, _ = self._smooth(verts)
        s = torch.stack([sums[1], sums[4], e.to(torch.float64)]).cpu().numpy()
        if s[0] == 0.0:
            return float("inf")
        return float(s[1] + self.cfg.smooth_weight * s[2])

    def full_eval(self, verts: torch.Tensor):
        coefs, sums = self._occupancy(verts)
        fg = face_grad(self.mesh, "soft", self.prec, coefs, grid=self.grid)
        g = vertex_grad(self.mesh, fg, scale=sums[3:4], dtype=self.dt)
        e, lv = self._smooth(verts)
        g = g + self.cfg.smooth_weight * 2.0 * (self.LT @ lv)
        s = torch.stack([sums[1], sums[4], e.to(torch.float64)]).cpu().numpy()
        loss = float("inf") if s[0] == 0.0 else float(s[1] + self.cfg.smooth_weight * s[2])
        return loss, g


def morph(template: TriangleMesh, target: ScalarField, cfg: MorphConfig | None = None, *,
          precision: str = "f64") -> tuple[TriangleMesh, MorphReport]:
    """Fit ``template``'s soft occupancy to ``target``; returns (mesh, report).
    Raises DivergedError if the loss turns non-finite."""
    cfg = cfg or MorphConfig()
    if template.num_faces == 0:
        raise ValueError("template mesh has no faces")
    if cfg.grid is not None and cfg.grid != target.spec:
        raise ValueError("cfg.grid, when given, must equal the target field's grid")
    lo, hi = template.bounds()
    if np.any(lo < target.spec.bounds_min) or np.any(hi > target.spec.bounds_max):
        raise ValueError("target grid bounds must contain the template bounding box")

    P = _DeviceProblem(template, target, cfg, precision)
    verts = P.mesh.vertices.clone()
    report = MorphReport()
    loss, grad = P.full_eval(verts)
    if not np.isfinite(loss):
        raise DivergedError(f"initial loss is not finite ({loss})")

    def log(iteration: int) -> None:
        report.entries.append({"iter": iteration, "loss": float(loss),
                               "grad_inf_norm": float(grad.abs().max().item())})

    log(0)
    faces = np.asarray(template.faces).copy()
    if cfg.step_size == 0.0 or cfg.iterations == 0:
        return TriangleMesh(verts.double().cpu().numpy(), faces), report

    velocity = torch.zeros_like(verts)
    for it in range(1, cfg.iterations + 1):
        accepted = False
        step = cfg.step_size
        for _ in range(_MOMENTUM_HALVINGS):
            trial_velocity = cfg.momentum * velocity - step * grad
            trial = verts + trial_velocity
            trial_loss = P.loss_only(trial)
            if np.isfinite(trial_loss) and trial_loss <= loss:
                accepted = True
                break
            step *= 0.5
        if not accepted:
            step = cfg.step_size
            for _ in range(_PLAIN_HALVINGS):
                trial_velocity = -step * grad
                trial = verts + trial_velocity
                trial_loss = P.loss_only(trial)
                if np.isfinite(trial_loss) and trial_loss <= loss:
                    accepted = True
                    break
                step *= 0.5
        if accepted:
            verts = trial
            velocity = trial_velocity
            loss = trial_loss  # the accepted backtracking loss is authoritative
            _, grad = P.full_eval(verts)
        else:
            velocity = torch.zeros_like(verts)
        if not np.isfinite(loss):
            log(it)
            raise DivergedError(f"loss became non-finite at iteration {it}")
        if it % cfg.log_every == 0 or it == cfg.iterations:
            log(it)
    return TriangleMesh(verts.double().cpu().numpy(), faces), report
