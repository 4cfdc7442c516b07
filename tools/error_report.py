"""Accuracy report of the FP32 exact forward against the f64 oracle on the
BASELINE configs (seeded node subsets): max / p99.99 |dW| on unflagged nodes,
flag and binarized-occupancy mismatches.  Run on a GPU box:

    python tools/error_report.py [--nodes N]
"""

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nodes", type=int, default=4096)
    args = ap.parse_args()
    import torch
    from oracle import oracle as orc
    from paper_2407_11272_b200 import configs, device

    out = {}
    for name, n in (("c1", None), ("c2", args.nodes), ("c3", args.nodes // 2),
                    ("c5", args.nodes // 16)):
        w = configs.make(name)
        if n is None or n >= w.n_nodes:
            idx = np.arange(w.n_nodes)
        else:
            idx = np.sort(np.random.default_rng(7).choice(w.n_nodes, size=n, replace=False))
        i, rem = np.divmod(idx, w.res[1] * w.res[2])
        j, k = np.divmod(rem, w.res[2])
        ax = [orc.axis_nodes(w.lo[a], w.hi[a], w.res[a]) for a in range(3)]
        pts = np.stack([ax[0][i], ax[1][j], ax[2][k]], axis=1)
        dm = device.DeviceMesh.from_numpy(w.vertices, w.faces)
        got, gf = device.forward(dm, "exact", "f32",
                                 points=torch.as_tensor(pts, dtype=torch.float32))
        got = got.double().cpu().numpy()
        gf = gf.cpu().numpy().astype(bool)
        ref, rf = orc.winding_number_batch(w.vertices, w.faces,
                                           pts.astype(np.float32).astype(np.float64))
        err = np.abs(got - ref)[~rf]
        amb = (np.abs(ref - 0.5) < 1e-3) | (np.abs(got - 0.5) < 1e-3)
        out[name] = {"nodes": int(len(idx)), "max_abs_err": float(err.max()),
                     "p9999_abs_err": float(np.quantile(err, 0.9999)),
                     "flag_mismatch": int((gf != rf).sum()),
                     "binarize_mismatch": int(((got > 0.5) != (ref > 0.5))[~amb].sum())}
        print(name, out[name], flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
