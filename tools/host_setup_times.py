"""Host-side setup costs of one DeviceMesh on a BASELINE config (the parts of
bench.py's e2e step that are not kernels).

    python tools/host_setup_times.py [--config c3]
"""

import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    args = ap.parse_args()
    import torch
    from paper_2407_11272_b200 import configs, device
    w = configs.make(args.config)
    torch.cuda.synchronize()
    for rep in range(2):
        t = {}
        t0 = time.perf_counter()
        dm = device.DeviceMesh.from_numpy(w.vertices, w.faces)
        torch.cuda.synchronize()
        t["from_numpy"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        perm, win, fl = device.strip_order(w.vertices, w.faces)
        t["strip_order"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        dm.strip_setup()
        t["strip_setup"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        a, wt = device.exact_edge_weights(w.faces, device.dead_faces(w.vertices, w.faces))
        t["edge_weights"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        dm.exact_pair_setup()
        t["pair_setup"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        dm.csr()
        t["csr"] = time.perf_counter() - t0
        print(rep, {k: round(v * 1e3, 1) for k, v in t.items()}, "ms")


if __name__ == "__main__":
    main()
