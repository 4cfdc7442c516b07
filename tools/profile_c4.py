"""Where a C4 training step spends its time (torch.profiler, CUDA activity):
per-kernel GPU time and the GPU-busy fraction of the step's wall time.

    python tools/profile_c4.py [--meshes 64] [--res 64] [--steps 2]

A profiling aid (numbers under the profiler are not bench values).
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2407_11272_b200 import configs, device  # noqa: E402
from paper_2407_11272_b200.batch import DeformationNet, batch_occupancy_loss  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--meshes", type=int, default=64)
    ap.add_argument("--res", type=int, default=64)
    ap.add_argument("--steps", type=int, default=2)
    a = ap.parse_args()
    dev = torch.device("cuda")
    B, R = a.meshes, a.res
    grid = ((-1.0,) * 3, (1.0,) * 3, (R, R, R))
    meshes = configs.c4_batch(B)
    faces = torch.from_numpy(meshes[0][1]).to(dev)
    tmpl = torch.stack([torch.from_numpy(m[0]) for m in meshes]).to(dev, torch.float32)
    tg = []
    for b in range(B):
        cv, cf = configs.icosphere(3, 1.0)
        cv = cv * np.random.default_rng(1000 + b).uniform(0.3, 0.6, size=3)
        w, _ = device.forward(device.DeviceMesh.from_numpy(cv, cf, dev), "exact", "f32", grid=grid)
        tg.append((w > 0.5).float())
    targets = torch.stack(tg)
    torch.manual_seed(0)
    net = DeformationNet(B).to(dev)
    opt = torch.optim.Adam(net.parameters(), lr=1e-4)
    mid = torch.arange(B, device=dev)
    csr = device.DeviceMesh(tmpl[0], faces).csr()

    def step():
        opt.zero_grad(set_to_none=True)
        loss = batch_occupancy_loss(net(tmpl, mid), faces, grid, targets, csr=csr).mean()
        loss.backward()
        opt.step()

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        for _ in range(a.steps):
            step()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / a.steps
    ev = [e for e in prof.key_averages() if e.device_time_total > 0]
    gpu = sum(e.self_device_time_total for e in ev) / a.steps / 1e3
    print(f"wall {wall * 1e3:.1f} ms/step, GPU kernel time {gpu:.1f} ms/step "
          f"({100 * gpu / (wall * 1e3):.0f}% busy)")
    print(prof.key_averages().table(sort_by="self_cuda_time_total", row_limit=18))


if __name__ == "__main__":
    main()
