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


def _padded(ip: np.ndarray, ix: np.ndarray, dv: np.ndarray, n: int):
    """CSR rows as padded (n, width) column / value arrays; padding points at
    the extra zero row n, so a row product is a fixed-order gather + sum."""
    cnt = np.diff(ip)
    width = max(1, int(cnt.max()) if n else 1)
    cols = np.full((n, width), n, dtype=np.int64)
    vals = np.zeros((n, width), dtype=np.float64)
    r = np.repeat(np.arange(n), cnt)
    k = np.arange(len(ix)) - np.repeat(ip[:-1], cnt)
    cols[r, k] = ix
    vals[r, k] = dv
    return cols, vals


class _Laplacian:
    """y = L x and y = L^T x for the uniform Laplacian as padded gathers
    (each row's CSR entries in column order, then a sum over the row): the
    same terms as the sparse CSR product, in a fixed order, and capturable
    in a CUDA graph (the sparse-library path is not)."""

    def __init__(self, faces, n_verts: int, dev, dt):
        import scipy.sparse as sp
        ip, ix, dv = uniform_laplacian(faces, n_verts)
        lt = sp.csr_matrix((dv, ix, ip), shape=(n_verts, n_verts)).T.tocsr()
        lt.sort_indices()
        self.n = n_verts
        c, v = _padded(ip, ix, dv, n_verts)
        self.cols, self.vals = torch.from_numpy(c).to(dev), torch.from_numpy(v).to(dev, dt)
        c, v = _padded(lt.indptr.astype(np.int64), lt.indices.astype(np.int64),
                       lt.data.astype(np.float64), n_verts)
        self.tcols, self.tvals = torch.from_numpy(c).to(dev), torch.from_numpy(v).to(dev, dt)

    def _apply(self, cols, vals, x):
        xe = torch.cat([x, torch.zeros_like(x[:1])])
        return (vals.unsqueeze(-1) * xe[cols]).sum(dim=1)

    def mv(self, x):
        return self._apply(self.cols, self.vals, x)

    def tmv(self, x):
        return self._apply(self.tcols, self.tvals, x)


class _DeviceProblem:
    """Everything the loop touches, resident on the GPU.  With ``graphs`` the
    two evaluations (a trial's loss; the accepted step's loss + gradient) are
    captured once as CUDA graphs over a static vertex buffer and replayed:
    every kernel still runs per evaluation (pack, forward, loss terms,
    backward, gather, smoothing), only the per-launch host overhead goes --
    at the reference's own morph sizes (hundreds of faces, 32^3) that
    overhead, not the kernels, is the evaluation's cost."""

    def __init__(self, template: TriangleMesh, target: ScalarField, cfg: MorphConfig,
                 precision: str, graphs: bool = True):
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
        self.lap = _Laplacian(template.faces, template.num_vertices, dev, self.dt)
        self.graphs = graphs
        self._g = None

    def _occupancy(self, verts: torch.Tensor):
        self.mesh.set_vertices(verts)
        vals, flags = forward(self.mesh, "soft", self.prec, grid=self.grid)
        coefs, sums = loss_terms(vals, flags, self.targets)
        return coefs, sums

    def _smooth(self, verts):
        lv = self.lap.mv(verts)
        return (lv * lv).sum(), lv

    def _loss_body(self, verts):
        _, sums = self._occupancy(verts)
        e, _ = self._smooth(verts)
        return torch.stack([sums[1], sums[4], e.to(torch.float64)])

    def _full_body(self, verts):
        coefs, sums = self._occupancy(verts)
        fg = face_grad(self.mesh, "soft", self.prec, coefs, grid=self.grid)
        g = vertex_grad(self.mesh, fg, scale=sums[3:4], dtype=self.dt)
        e, lv = self._smooth(verts)
        g = g + self.cfg.smooth_weight * 2.0 * self.lap.tmv(lv)
        return torch.stack([sums[1], sums[4], e.to(torch.float64)]), g

    def _capture(self):
        v0 = self.mesh.vertices
        self.v_in = v0.clone()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm-up on a side stream before capture
            self._loss_body(self.v_in)
            self._full_body(self.v_in)
        torch.cuda.current_stream().wait_stream(side)
        self._gl, self._gf = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(self._gl):
            self._out_l = self._loss_body(self.v_in)
        with torch.cuda.graph(self._gf):
            self._out_f = self._full_body(self.v_in)
        self._g = True

    def _loss_value(self, s) -> float:
        s = s.cpu().numpy()
        if s[0] == 0.0:
            return float("inf")
        return float(s[1] + self.cfg.smooth_weight * s[2])

    def loss_only(self, verts: torch.Tensor) -> float:
        if not self.graphs:
            return self._loss_value(self._loss_body(verts))
        if self._g is None:
            self._capture()
        self.v_in.copy_(verts)
        self._gl.replay()
        return self._loss_value(self._out_l)

    def full_eval(self, verts: torch.Tensor):
        if not self.graphs:
            s, g = self._full_body(verts)
            return self._loss_value(s), g
        if self._g is None:
            self._capture()
        self.v_in.copy_(verts)
        self._gf.replay()
        return self._loss_value(self._out_f[0]), self._out_f[1].clone()


def morph(template: TriangleMesh, target: ScalarField, cfg: MorphConfig | None = None, *,
          precision: str = "f64", graphs: bool = True) -> tuple[TriangleMesh, MorphReport]:
    """Fit ``template``'s soft occupancy to ``target``; returns (mesh, report).
    Raises DivergedError if the loss turns non-finite.  ``graphs``: replay
    the evaluations as CUDA graphs (same kernels, same results)."""
    cfg = cfg or MorphConfig()
    if template.num_faces == 0:
        raise ValueError("template mesh has no faces")
    if cfg.grid is not None and cfg.grid != target.spec:
        raise ValueError("cfg.grid, when given, must equal the target field's grid")
    lo, hi = template.bounds()
    if np.any(lo < target.spec.bounds_min) or np.any(hi > target.spec.bounds_max):
        raise ValueError("target grid bounds must contain the template bounding box")

    P = _DeviceProblem(template, target, cfg, precision, graphs=graphs)
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
