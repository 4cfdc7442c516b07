"""Slab-sharded multi-GPU driver (one process per GPU, torch.distributed).

The grid shards into contiguous ranges of the flat node index -- i-slabs,
since the flat order is k fastest, i slowest (winding.py:75-76) -- with the
mesh replicated on every rank (<= 48 MB packed even at 1M faces).  This is
the multi-device form of the reference's chunked driver (_parallel.py:39-53):
independent node ranges, each written by exactly one worker.

* forward: no communication; optionally an all-gather of the slabs into the
  full grid (occupancy output);
* loss + backward: every rank computes its partial loss sums and its vertex
  gradient numerator over its slab; ONE all-reduce of a packed buffer
  [grad numerator (V*3) | sum w r^2 | sum w | n_flagged] (f64), then the
  1/sum(w) normalisation (the gradient is linear in the coefficients, so
  scaling after the reduce avoids a second collective; cf. grad.py:103-110).

The compute is behind a small evaluator interface so the collective logic
is exercised on CPU (gloo, world_size 2) in tests with the oracle as the
evaluator; the product evaluator is ``CudaSlabEvaluator`` (the C ABI).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


def slab_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """[n0, n0+count) owned by ``rank``: equal contiguous slabs (the last
    one shorter when world does not divide n_total)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    per = (n_total + world - 1) // world
    n0 = min(n_total, rank * per)
    return n0, max(0, min(n_total, n0 + per) - n0)


class CudaSlabEvaluator:
    """Product evaluator: the sm_100a kernels through the C ABI."""

    def __init__(self, dmesh, grid, mode: str = "exact", precision: str = "f32"):
        self.dmesh = dmesh
        self.grid = grid
        self.mode = mode
        self.precision = precision

    def forward(self, n0: int, count: int, policy: int):
        from .device import forward
        return forward(self.dmesh, self.mode, self.precision, grid=self.grid, n0=n0,
                       count=count, policy=policy)

    def loss_grad_partial(self, n0: int, count: int, targets, weights=None):
        from .grad import device_loss_grad
        return device_loss_grad(self.dmesh, self.grid, targets, weights, mode=self.mode,
                                precision=self.precision, n0=n0, count=count)


@dataclass
class SlabDriver:
    evaluator: object
    n_total: int
    rank: int = 0
    world: int = 1
    group: object = None

    @property
    def slab(self) -> tuple[int, int]:
        return slab_range(self.n_total, self.rank, self.world)

    def forward(self, policy: int = 1, gather: bool = False):
        """This rank's slab (values, flags); with ``gather`` the full grid on
        every rank (all-gather of equal padded slabs)."""
        n0, cnt = self.slab
        vals, flags = self.evaluator.forward(n0, cnt, policy)
        if not gather or self.world == 1:
            return vals, flags
        per = (self.n_total + self.world - 1) // self.world
        pv = torch.zeros(per, dtype=vals.dtype, device=vals.device)
        pf = torch.zeros(per, dtype=flags.dtype, device=flags.device)
        pv[:cnt] = vals
        pf[:cnt] = flags
        out_v = [torch.empty_like(pv) for _ in range(self.world)]
        out_f = [torch.empty_like(pf) for _ in range(self.world)]
        dist.all_gather(out_v, pv, group=self.group)
        dist.all_gather(out_f, pf, group=self.group)
        return (torch.cat(out_v)[: self.n_total], torch.cat(out_f)[: self.n_total])

    def loss_grad(self, targets_slab, weights_slab=None):
        """(loss, grads (V,3) f64, excluded_nodes) over the whole grid.
        ``targets_slab`` / ``weights_slab`` cover this rank's slab only."""
        n0, cnt = self.slab
        sums, gnum = self.evaluator.loss_grad_partial(n0, cnt, targets_slab, weights_slab)
        V = gnum.shape[0]
        buf = torch.cat([gnum.reshape(-1).to(torch.float64), sums[:3].to(torch.float64)])
        if self.world > 1:
            dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.group)
        s = buf[-3:]
        wsum = s[1]
        # every rank holds the same reduced sums, so every rank raises alike
        # (the reference's check, grad.py:108-109)
        if float(wsum) == 0.0:
            raise ValueError("no usable grid nodes: all excluded or zero-weighted")
        grads = buf[:-3].reshape(V, 3) / wsum
        loss = s[0] / wsum
        return loss, grads, s[2], wsum
