"""CUDA-event time of one kernel path on a BASELINE config's full lattice
(re-pack included, as a step does), min over reps -- for A/B variant builds:

    WV_LIB_PATH=scratch/variants/X/lib.so python tools/fwd_time.py --config c3r [--bwd]
"""

import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3r")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--bwd", action="store_true")
    ap.add_argument("--precision", default="f32", choices=["f32", "f64"])
    ap.add_argument("--path", default="auto", choices=["auto", "trails", "pairs", "faces"],
                    help="backward records (--bwd)")
    a = ap.parse_args()
    import torch
    from paper_2407_11272_b200 import configs, device
    w = configs.make(a.config)
    grid = (w.lo, w.hi, w.res)
    dm = device.DeviceMesh.from_numpy(w.vertices, w.faces)
    v, f = device.forward(dm, "exact", a.precision, grid=grid)
    coefs = torch.where(f.bool(), 0.0, 2.0 * (v - (v > 0.5).to(v.dtype)))

    def run():
        dm.invalidate()
        if a.bwd:
            kw = {"auto": {}, "trails": {"trails": True}, "pairs": {"pairs": True},
                  "faces": {"pairs": False}}[a.path]
            device.face_grad(dm, "exact", a.precision, coefs, grid=grid, **kw)
        else:
            device.forward(dm, "exact", a.precision, grid=grid)

    run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(json.dumps({"lib": os.environ.get("WV_LIB_PATH", "default"), "config": a.config,
                      "bwd": a.bwd, "path": a.path, "precision": a.precision, "ms": min(ts), "all": ts}))


if __name__ == "__main__":
    main()
