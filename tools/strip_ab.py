"""A/B of the exact f32 forward: face-ordered vs strip-ordered records on a
BASELINE configuration's full lattice (CUDA-event timing, after warm-up).

    python tools/strip_ab.py [--config c3] [--reps 3]
"""

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--bwd", action="store_true", help="A/B the exact backward (pairs)")
    ap.add_argument("--f64", action="store_true", help="A/B the f64 parity forward")
    args = ap.parse_args()
    import time
    import torch
    from paper_2407_11272_b200 import configs, device, _lib as L
    w = configs.make(args.config)
    grid = (w.lo, w.hi, w.res)
    dm = device.DeviceMesh.from_numpy(w.vertices, w.faces)
    t0 = time.perf_counter()
    dm.strip_setup()
    host = time.perf_counter() - t0
    if args.bwd:
        return bwd_ab(args, w, grid, dm)
    res = {}
    outs = {}
    prec = "f64" if args.f64 else "f32"
    for strip in (False, True, False, True):
        v, f = device.forward(dm, "exact", prec, grid=grid, policy=L.POLICY_RAW, strip=strip)
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.reps):
            dm.invalidate()  # include the re-pack, as a step does
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            v, f = device.forward(dm, "exact", prec, grid=grid, policy=L.POLICY_RAW,
                                  strip=strip)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res.setdefault(strip, []).append(min(ts))
        outs[strip] = (v.double(), f)
    d = (outs[True][0] - outs[False][0]).abs()
    ok = outs[True][1] == 0
    print({"config": args.config, "face_order_ms": res[False], "strip_ms": res[True],
           "speedup": min(res[False]) / min(res[True]), "strip_host_s": host,
           "max_abs_diff": float(d[ok].max()),
           "flag_mismatch": int((outs[True][1] != outs[False][1]).sum())})


def bwd_ab(args, w, grid, dm):
    import time
    import torch
    from paper_2407_11272_b200 import device
    t0 = time.perf_counter()
    dm.exact_pair_setup()
    host = time.perf_counter() - t0
    n = w.n_nodes
    g = torch.Generator(device="cuda").manual_seed(0)
    coefs = torch.randn(n, device="cuda", generator=g)
    _, flags = device.forward(dm, "exact", "f32", grid=grid)
    coefs[flags.bool()] = 0.0
    res, outs = {}, {}
    for pairs in (False, True, False, True):
        fg = device.face_grad(dm, "exact", "f32", coefs, grid=grid, pairs=pairs)
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.reps):
            dm.invalidate()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fg = device.face_grad(dm, "exact", "f32", coefs, grid=grid, pairs=pairs)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res.setdefault(pairs, []).append(min(ts))
        outs[pairs] = device.vertex_grad(dm, fg)
    d = (outs[True] - outs[False]).abs().max().item()
    print({"config": args.config, "single_ms": res[False], "pairs_ms": res[True],
           "speedup": min(res[False]) / min(res[True]), "pair_host_s": host,
           "max_rel_diff": d / outs[False].abs().max().item()})


if __name__ == "__main__":
    main()
