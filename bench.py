"""Benchmark of the winding-number hot path (BASELINE.json metric:
point-triangle solid-angle evaluations/s, forward and forward+backward, plus
256^3 voxelize ms).

Workload (N=1 default): config C3 -- a 100k-face triangle soup (torus
(0.7,0.3,250,200) un-welded and shuffled, seeded) voxelized on [-1,1]^3 at
256^3.  A step = one pass of the hot path over the node slab this rank owns
(contiguous i-slabs).  Inputs are synthetic (no network).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun (N>1) every rank times its slab on its own GPU; the reported
time is the max over ranks and ``value`` is the whole-job pair rate.
``--impl reference`` times the reference's CPU algorithm (the bit-exact C
port in oracle/, all host threads) on a bounded node sample of the same
workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

EXACT_FWD_FLOPS = 63      # SURVEY.md 8d / Appendix A.1 (VOS formula as written)
EXACT_BWD_FLOPS = 170     # Appendix A.4
FP32_PEAK_NOMINAL = None  # computed from MEASURED_PEAKS sm_max_mhz below


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c3")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target duration of the CPU-baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    sm_mhz = 1965.0
    out = {"source": "nominal"}
    if p.exists():
        d = json.loads(p.read_text())
        sm_mhz = float(d.get("sm_max_mhz", sm_mhz))
        out.update(d)
        out["source"] = "MEASURED_PEAKS.json sm_max_mhz"
    # FP32 CUDA-core peak: 148 SMs x 128 lanes x 2 FLOP/FMA x clock
    out["fp32_tflops_nominal"] = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12
    return out


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 4 + i and s[4 + i].lower() == "active"})
        pw = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "power_w_median": statistics.median(pw) if pw else None,
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# reference arm / CPU baseline (oracle = bit-exact C port of the reference)

def cpu_sample_rate(w, seconds: float, threads: int, seed: int = 0):
    """Exact f64 forward of the reference algorithm on a seeded node sample
    sized to take about `seconds` on `threads` host threads."""
    from oracle import oracle as orc

    nodes_all = int(np.prod(w.res))
    rng = np.random.default_rng(seed)
    probe = max(threads * 2, 16)
    idx = rng.choice(nodes_all, size=probe, replace=False)
    pts = _nodes(w, idx)
    t0 = time.perf_counter()
    orc.winding_number_batch(w.vertices, w.faces, pts, chunk=1, threads=threads)
    dt = max(time.perf_counter() - t0, 1e-6)
    rate = probe * w.n_faces / dt
    n = int(min(nodes_all, max(threads * 8, rate * seconds / w.n_faces)))
    idx = np.sort(rng.choice(nodes_all, size=n, replace=False))
    pts = _nodes(w, idx)
    chunk = max(1, min(2000, n // (threads * 4) or 1))
    t0 = time.perf_counter()
    orc.winding_number_batch(w.vertices, w.faces, pts, chunk=chunk, threads=threads)
    dt = time.perf_counter() - t0
    return n * w.n_faces / dt, n, dt


def _nodes(w, idx):
    from oracle import oracle as orc
    rx, ry, rz = w.res
    i, rem = np.divmod(idx, ry * rz)
    j, k = np.divmod(rem, rz)
    ax = [orc.axis_nodes(w.lo[a], w.hi[a], w.res[a]) for a in range(3)]
    return np.stack([ax[0][i], ax[1][j], ax[2][k]], axis=1)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as orc
    from paper_2407_11272_b200 import configs

    w = configs.make(args.config)
    threads = orc.default_threads()
    per = max(2.0, args.cpu_seconds / max(1, args.steps))
    for _ in range(args.warmup if args.warmup < 1 else 1):
        cpu_sample_rate(w, 0.5, threads, seed=99)
    rates, samples = [], []
    t_all = time.perf_counter()
    for k in range(args.steps):
        r, n, dt = cpu_sample_rate(w, per, threads, seed=k)
        rates.append(r)
        samples.append(n)
    wall = time.perf_counter() - t_all
    rate = statistics.median(rates)
    line = {
        "impl": "reference", "metric": "point-triangle solid-angle evals/sec (exact fwd, f64 CPU reference)",
        "value": rate, "unit": "pairs/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": wall * 1e3 / max(1, args.steps),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": w.name, "faces": w.n_faces,
                                        "grid": list(w.res), "mode": "exact"},
        "cpu_baseline": {"value": rate, "unit": "pairs/s", "cores": threads, "kind": "port",
                         "sample": f"{samples} seeded random nodes of the {w.res[0]}^3 grid x "
                                   f"{w.n_faces} faces per step (bit-exact C port of "
                                   "_kernels.exact_batch, oracle/windvox_oracle.c)"},
        "e2e": {"value": rate, "unit": "pairs/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "extrapolated_full_forward_s": w.pairs / rate,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm

def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2407_11272_b200 as wvb
    from paper_2407_11272_b200 import configs, device

    dev = torch.device("cuda", local)
    w = configs.make(args.config)
    n_total = w.n_nodes
    per_rank = (n_total + world - 1) // world
    n0 = rank * per_rank
    cnt = max(0, min(n_total, n0 + per_rank) - n0)
    grid = (w.lo, w.hi, w.res)

    dmesh = device.DeviceMesh.from_numpy(w.vertices, w.faces, dev)
    out = torch.empty(cnt, dtype=torch.float32, device=dev)
    flags = torch.empty(cnt, dtype=torch.uint8, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step():
        # one pass of the hot path over this rank's slab: face staging +
        # exact forward (every kernel of the path runs each step)
        dmesh.invalidate()
        device.exact_forward_f32(dmesh, grid=grid, n0=n0, count=cnt, out=out, flags=flags)

    launches_per_step = 2 + 1  # surface-eps + pack + forward
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # --- timed region -----------------------------------------------------
    stream = torch.cuda.current_stream()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            flush.zero_()
            step()
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / args.steps
    pairs_step = w.pairs  # all ranks together cover the whole grid once per step
    value = pairs_step / (ms_step / 1e3)

    # --- roofline: the forward kernel alone, CUDA events on its stream ----
    kev0 = torch.cuda.Event(enable_timing=True)
    kev1 = torch.cuda.Event(enable_timing=True)
    dmesh.packed(1)
    torch.cuda.synchronize()
    reps = max(1, args.steps)
    kev0.record(stream)
    for _ in range(reps):
        device.exact_forward_f32(dmesh, grid=grid, n0=n0, count=cnt, out=out, flags=flags)
    kev1.record(stream)
    torch.cuda.synchronize()
    k_ms = kev0.elapsed_time(kev1) / reps
    pk = peaks()
    achieved = EXACT_FWD_FLOPS * cnt * w.n_faces / (k_ms / 1e3) / 1e12

    # --- e2e: public API, host buffers in, host result out ----------------
    mesh_np = wvb.TriangleMesh(w.vertices, w.faces)
    spec = wvb.GridSpec(w.lo, w.hi, w.res)
    e2e_value = None
    h2d = w.vertices.nbytes + w.faces.nbytes
    d2h = n_total * 4
    if world == 1:
        wvb.voxelize(mesh_np, spec, precision="f32")  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_steps = max(1, min(args.steps, 3))
        for _ in range(e2e_steps):
            field = wvb.voxelize(mesh_np, spec, precision="f32")
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        e2e_value = w.pairs / e2e_s
        del field

    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            from oracle import oracle as orc
            thr = orc.default_threads()
            r, n, dt = cpu_sample_rate(w, args.cpu_seconds, thr)
            cpu = {"value": r, "unit": "pairs/s", "cores": thr, "kind": "port",
                   "sample": f"{n} seeded random nodes of the {w.res[0]}^3 grid x {w.n_faces} "
                             f"faces, exact f64 forward, {dt:.1f} s (bit-exact C port of "
                             "_kernels.exact_batch)"}
        line = {
            "metric": "point-triangle solid-angle evals/sec (exact fwd; fwd+bwd pending); "
                      "256^3 voxelize ms",
            "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": w.name, "faces": w.n_faces, "grid": list(w.res),
                       "mode": "exact", "step": "pack + exact forward over the rank's i-slab",
                       "l2": "256 MiB buffer zeroed between timed steps (> 126 MB L2)",
                       "parallelism": f"i-slabs x{world}"},
            "voxelize_ms": ms_step,
            "fwd_pairs_per_s": value,
            "roofline": {"bound": "fp32", "achieved": achieved,
                         "peak": pk["fp32_tflops_nominal"], "unit": "TFLOP/s",
                         "frac": achieved / pk["fp32_tflops_nominal"], "traffic": None,
                         "kernel": "exact_fwd_f32_kernel<GridSrc>",
                         "kernel_ms": k_ms,
                         "flops_per_pair": EXACT_FWD_FLOPS,
                         "peak_source": "148 SM x 128 FP32 lanes x 2 x sm_max_mhz ("
                                        + pk["source"] + ")"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "pairs/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "api": "paper_2407_11272_b200.voxelize(mesh, spec, precision='f32')"},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
