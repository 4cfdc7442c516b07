"""Accuracy report of the FP32 hot path against the f64 oracle on the
BASELINE configs, through the lattice kernels the bench runs (strip-ordered
forward, edge-trail row backward): a seeded set of whole k-rows of each grid is
evaluated with grid launches (node range = one row) and compared with the
oracle on the same f32-rounded nodes.

The oracle evaluates the same f32-rounded nodes AND vertices the kernels see
(the reference's f32 path rounds both, winding.py:362-387).  Forward: max /
p99.99 |dW| over every unflagged node (north_star: 1e-5), flag and
binarized-occupancy mismatches (|w - 0.5| < 1e-3 excluded).  Backward
(exact): vertex gradients of sum_p c_p W_p for seeded coefficients at every
unflagged node, max |dg| / max |g| (north_star: 1e-4).  Prints one JSON line (``-s``);
profiles/r01_error_report_*.txt are its output."""

import json

import numpy as np
import pytest

from oracle import oracle as orc
from test_gpu_fuzz import r32

pytestmark = pytest.mark.gpu

ROWS = 16


def test_error_report(cuda_device):
    import torch
    from paper_2407_11272_b200 import configs, device
    out = {}
    for name in ("c1", "c2", "c3", "c3r", "c5"):
        w = configs.make(name)
        rx, ry, rz = w.res
        rows = np.sort(np.random.default_rng(7).choice(rx * ry, size=min(ROWS, rx * ry),
                                                       replace=False))
        grid = (w.lo, w.hi, w.res)
        ax = [orc.axis_nodes(w.lo[a], w.hi[a], w.res[a]) for a in range(3)]
        pts = np.concatenate([np.stack([np.full(rz, ax[0][r // ry]), np.full(rz, ax[1][r % ry]),
                                        ax[2]], axis=1) for r in rows])
        p32 = pts.astype(np.float32).astype(np.float64)
        dm = device.DeviceMesh.from_numpy(w.vertices, w.faces)
        vals, flags = [], []
        for r in rows:
            v, f = device.forward(dm, "exact", "f32", grid=grid, n0=int(r) * rz, count=rz,
                                  strip=name != "c3r")
            vals.append(v.double().cpu().numpy())
            flags.append(f.cpu().numpy().astype(bool))
        got, gf = np.concatenate(vals), np.concatenate(flags)
        v32 = r32(w.vertices)
        ref, rf = orc.winding_number_batch(v32, w.faces, p32)
        err = np.abs(got - ref)
        err[rf] = 0.0
        amb = (np.abs(ref - 0.5) < 1e-3) | (np.abs(got - 0.5) < 1e-3)
        rep = {"nodes": int(len(pts)), "max_abs_err": float(err.max()),
               "p9999_abs_err": float(np.quantile(err[~rf], 0.9999)),
               "flag_mismatch": int((gf != rf).sum()),
               "binarize_mismatch": int(((got > 0.5) != (ref > 0.5))[~amb].sum())}
        assert rep["flag_mismatch"] == 0 and rep["binarize_mismatch"] == 0, (name, rep)
        assert rep["max_abs_err"] <= 1e-5, (name, rep)
        if name != "c5":  # the 1M-face oracle gradient is too slow for a report
            c = np.random.default_rng(11).normal(size=len(pts))
            c[rf | gf] = 0.0
            c32 = c.astype(np.float32).astype(np.float64)
            g = torch.zeros((dm.num_vertices, 3), dtype=torch.float64, device="cuda")
            for i, r in enumerate(rows):
                cr = torch.from_numpy(c32[i * rz:(i + 1) * rz]).float().cuda()
                kw = {"pairs": False} if name == "c3r" else {"trails": True}
                fg = device.face_grad(dm, "exact", "f32", cr, grid=grid, n0=int(r) * rz,
                                      count=rz, **kw)
                device.vertex_grad(dm, fg, out=g, accumulate=True)
            gr = orc.exact_grad(v32, w.faces, p32, c32)
            if dm.exact_trail_setup()[2] == 0:
                # closed mesh: the exact gradient is identically zero (every edge
                # cancels); the oracle's face-wise sum shows its rounding noise
                rep["exact_grad_abs"] = float(np.abs(g.cpu().numpy()).max())
                rep["oracle_grad_noise"] = float(np.abs(gr).max())
                assert rep["exact_grad_abs"] <= max(1e-9, 10 * rep["oracle_grad_noise"])
            else:
                scale = max(np.abs(gr).max(), 1e-300)
                rep["exact_grad_rel_err"] = float(np.abs(g.cpu().numpy() - gr).max() / scale)
                assert rep["exact_grad_rel_err"] <= 1e-4, (name, rep)
        out[name] = rep
        print(name, rep, flush=True)
    print(json.dumps(out))
