"""Benchmark of the winding-number hot path (BASELINE.json metric:
point-triangle solid-angle evaluations/s, forward and forward+backward, plus
256^3 voxelize ms).

Workload (default, N=1): config C3 -- a 100k-face triangle soup (torus
(0.7,0.3,250,200) un-welded and shuffled with a fixed seed) on [-1,1]^3 at
256^3 = 16.8M lattice nodes, 1.68e12 point-triangle pairs per pass.  A step
is one forward+backward training pass of the occupancy loss in exact mode on
the FP32 path: pack the (moved) mesh, exact forward over the rank's i-slab,
fused loss terms against a fixed target occupancy, exact backward, vertex
gather, and (N>1) one all-reduce of [grad numerator | loss sums].  Synthetic
inputs (no network); the target is the binarized exact occupancy of the same
soup scaled by 1.03, computed once before timing.  At this size both
directions run over face strips (strip-ordered forward, strip-pair backward;
DESIGN.md 3.1b / 3.3b).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun each rank owns 1/N of the grid (weak scaling in pairs per
GPU is NOT what this is: total work is fixed, so scaling is "strong"); time
is the max over ranks.  ``--impl reference`` times the reference's CPU
algorithm (the bit-exact C port in oracle/, all host threads) on a bounded
node sample of the same workload, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# algorithmic work per point-triangle pair
EXACT_FWD_FLOPS = 63
EXACT_BWD_FLOPS = 170
# What the kernels actually EXECUTE per pair, from the SASS of their inner
# loops (tools/sass_loop_mix.py; FMA = 2 FLOPs; MUFU = XU-pipe ops).  The
# lattice-row kernels hoist the x/y parts of every pair term out of the pair
# loop, and the backward's edge (Biot-Savart) form is cheaper than the pinned
# face-wise closed form, so they execute FEWER FLOPs than the pinned
# algorithmic counts above: the algorithmic-FLOP rate can exceed the FP32
# peak, and the executed-work fractions below are the pipe utilisation.
# strip-ordered forward (the lattice default from 2M nodes): measured from the
# ncu executed-instruction mix on the full C3 lattice (tools/sass_exec_mix.py;
# 4.3% strip restarts); the face-ordered kernel executed 42.25 / 4 MUFU
EXACT_FWD_EXEC_FLOPS = 25.7    # fwd_f32_kernel<ExactStripPol,RowSrc> (profiles/r01_ncu_c3_fwd_v73_summary.txt)
EXACT_FWD_FACE_ORDER_EXEC_FLOPS = 42.25  # fwd_f32_kernel<ExactPol,RowSrc>, all-common fast path
# strip-pair backward (the lattice default from 2M nodes), ncu executed mix on
# c3s; the single-face kernel executed 60.5 / 4 MUFU (static SASS count)
EXACT_BWD_EXEC_FLOPS = 49.0    # bwd_f32_kernel<ExactEdgeBwdPair,RowSrc>
EXACT_FWD_MUFU = 2.09  # 1 sqrt (+2 per strip restart) + 1 rcp; face-ordered: 4
SOFT_STEP_FLOPS = 15 + 72  # soft forward + soft backward, pinned
EXACT_BWD_MUFU = 3.1  # 2 rsqrt + 1 rcp per face and pair (+ rare paths)


def traffic(workload: str, kernel: str):
    """DRAM bytes per launch of ``kernel`` from a committed ncu capture."""
    try:
        t = json.loads((ROOT / "profiles" / "traffic.json").read_text()).get(workload)
    except (OSError, ValueError):
        return None
    if not t or t["kernel"].split("<")[0] not in kernel:
        return None
    return t["read"] + t["write"]


# FMA-pipe lane-ops per pair (one per lane of every FFMA/FADD/FMUL, two per
# packed f32x2 op), from the same ncu executed-instruction mixes: the FMA
# pipe issues 128 lane-ops per clock per SM whatever the op, so this (not the
# FLOP count, where an add is half an FMA) is what bounds the kernels.
EXACT_FWD_LANE_OPS = 17.4   # strip forward (C3 mix, v73: row parts carried, two faces per decision)
EXACT_BWD_LANE_OPS = 31.7   # strip-pair backward (c3s mix)


def executed(alg_tf, alg_flops, exec_flops, mufu, ms, peak, clk_mhz, lane_ops=None):
    """Roofline of one kernel: pinned-algorithmic rate plus the utilisation of
    the two pipes it actually runs on (FP32 FMA pipe, XU/MUFU pipe at 16 ops
    per clock per SM)."""
    pairs_s = alg_tf * 1e12 / alg_flops
    xu_peak = 148 * 16 * clk_mhz * 1e6
    r = {"achieved": alg_tf, "frac": alg_tf / peak, "kernel_ms": ms,
         "executed_flops_per_pair": exec_flops, "mufu_per_pair": mufu,
         "fma_frac": pairs_s * exec_flops / 1e12 / peak,
         "xu_frac": pairs_s * mufu / xu_peak}
    if lane_ops:
        r["fma_lane_ops_per_pair"] = lane_ops
        r["fma_pipe_frac"] = pairs_s * lane_ops / (148 * 128 * clk_mhz * 1e6)
    return r


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
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def init_dist(local: int, world: int):
    """One process per GPU; NCCL over NVLink.  WV_BENCH_BACKEND=gloo (with
    ranks wrapped onto the visible GPUs) exercises the N>1 code path on a
    single GPU -- a functional check only, never a reported number."""
    import torch
    import torch.distributed as dist
    gpu = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        backend = os.environ.get("WV_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    return dev


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    sm_mhz, src = 1965.0, "nominal 1965 MHz"
    if p.exists():
        d = json.loads(p.read_text())
        sm_mhz = float(d.get("sm_max_mhz", sm_mhz))
        src = "MEASURED_PEAKS.json sm_max_mhz"
    # FP32 CUDA-core peak: 148 SMs x 128 FP32 lanes x 2 FLOP/FMA x clock
    return 148 * 128 * 2 * sm_mhz * 1e6 / 1e12, src


def measured_fp32_peak():
    """FP32 FMA throughput measured on this GPU by tools/ffma2_probe (16
    independent FMA chains per thread, FFMA and packed FFMA2), TFLOP/s."""
    import subprocess
    exe = ROOT / "tools" / "ffma2_probe"
    if not exe.exists():
        return None
    try:
        out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60).stdout
        vals = [float(line.split()[-2]) for line in out.splitlines() if "TFLOP/s" in line]
        return max(vals) if vals else None
    except Exception:
        return None


class ClockSampler:
    """SM clock / throttle reasons sampled (NVML) DURING the timed region."""

    def __init__(self, index: int, period: float = 0.25):
        self.index, self.period = index, period
        self.samples = []
        self._stop = threading.Event()
        self._first = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                pw = N.nvmlDeviceGetPowerUsage(h) / 1000.0
                self.samples.append((sm, mx, r, pw))
                self._first.set()
                self._stop.wait(self.period)
        except Exception as e:  # pragma: no cover - reported in the JSON line
            self.error = repr(e)
        self._first.set()

    def __enter__(self):
        # NVML is initialised and the first sample taken before the timed
        # region opens, so even a millisecond-long region has a reading
        self._t.start()
        self._first.wait(timeout=10)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None,
                    "reasons": ["unsampled: " + getattr(self, "error", "no samples")]}
        import pynvml as N
        bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
        reasons = sorted({k for s in self.samples for k, b in bits.items() if s[2] & b})
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "power_w_median": statistics.median(s[3] for s in self.samples),
                "samples": len(self.samples), "source": "nvml"}


# ---------------------------------------------------------------------------
# CPU side: the reference algorithm (bit-exact C port, oracle/) on a sample

def _nodes(w, idx):
    from oracle import oracle as orc
    i, rem = np.divmod(idx, w.res[1] * w.res[2])
    j, k = np.divmod(rem, w.res[2])
    ax = [orc.axis_nodes(w.lo[a], w.hi[a], w.res[a]) for a in range(3)]
    return np.stack([ax[0][i], ax[1][j], ax[2][k]], axis=1)


def cpu_fwd_bwd_rate(w, seconds: float, threads: int, seed: int = 0):
    """Exact f64 forward (reference exact_batch, bit-exact port) + exact f64
    gradient (closed-form oracle; the reference has no exact-gradient kernel)
    on a seeded node sample sized for ~`seconds` on `threads` threads.
    Returns (fwd+bwd pairs/s, fwd pairs/s, nodes, wall s)."""
    from oracle import oracle as orc
    rng = np.random.default_rng(seed)
    probe = max(threads * 32, 64)  # large enough that per-call staging does not dominate
    pts = _nodes(w, rng.choice(w.n_nodes, size=probe, replace=False))
    t0 = time.perf_counter()
    orc.winding_number_batch(w.vertices, w.faces, pts, chunk=1, threads=threads)
    orc.exact_grad(w.vertices, w.faces, pts, np.ones(probe), chunk=1, threads=threads)
    rate = probe * w.n_faces / max(time.perf_counter() - t0, 1e-6)
    n = int(min(w.n_nodes, max(threads * 4, rate * seconds / w.n_faces)))
    pts = _nodes(w, np.sort(rng.choice(w.n_nodes, size=n, replace=False)))
    chunk = max(1, n // (threads * 4))
    t0 = time.perf_counter()
    vals, flags = orc.winding_number_batch(w.vertices, w.faces, pts, chunk=chunk, threads=threads)
    t_f = time.perf_counter() - t0
    coefs = np.where(flags, 0.0, 2.0 * (vals - (vals > 0.5)))
    # one (V,3) buffer per chunk in the reference's merge (grad.py:113-127)
    gchunk = max(chunk, n // threads)
    t1 = time.perf_counter()
    orc.exact_grad(w.vertices, w.faces, pts, coefs, chunk=gchunk, threads=threads)
    t_b = time.perf_counter() - t1
    return n * w.n_faces / (t_f + t_b), n * w.n_faces / t_f, n, t_f + t_b


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as orc
    from paper_2407_11272_b200 import configs
    w = configs.make(args.config)
    threads = orc.default_threads()
    per = max(3.0, args.cpu_seconds / max(1, args.steps))
    for _ in range(min(1, args.warmup)):
        cpu_fwd_bwd_rate(w, 0.5, threads, seed=99)
    rates, fwd, samples = [], [], []
    t_all = time.perf_counter()
    for k in range(args.steps):
        r, rf, n, _ = cpu_fwd_bwd_rate(w, per, threads, seed=k)
        rates.append(r)
        fwd.append(rf)
        samples.append(n)
    wall = time.perf_counter() - t_all
    rate = statistics.median(rates)
    line = {
        "impl": "reference",
        "metric": "point-triangle solid-angle evals/sec, exact fwd+bwd (256^3 voxelize ms in "
                  "extrapolated_voxelize_ms)",
        "value": rate, "unit": "pairs/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": wall * 1e3 / max(1, args.steps),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": w.name, "faces": w.n_faces, "grid": list(w.res), "mode": "exact",
                   "step": "bounded node sample: exact forward + exact gradient"},
        "fwd_pairs_per_s": statistics.median(fwd),
        "extrapolated_voxelize_ms": w.pairs / statistics.median(fwd) * 1e3,
        "cpu_baseline": {"value": rate, "unit": "pairs/s", "cores": threads, "kind": "port",
                         "sample": f"{samples} seeded random nodes of the {w.res[0]}^3 grid x "
                                   f"{w.n_faces} faces per step; forward = bit-exact C port of "
                                   "_kernels.exact_batch, backward = closed-form oracle "
                                   "(no reference exact-gradient kernel exists)"},
        "e2e": {"value": rate, "unit": "pairs/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm

def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    dev = init_dist(local, world)
    local = dev.index
    from paper_2407_11272_b200 import configs, device
    from paper_2407_11272_b200 import _lib as L
    from paper_2407_11272_b200.distributed import SlabDriver, slab_range

    w = configs.make(args.config)
    n0, cnt = slab_range(w.n_nodes, rank, world)
    grid = (w.lo, w.hi, w.res)

    # fixed target: binarized exact occupancy of the soup scaled by 1.03 (untimed)
    tmesh = device.DeviceMesh.from_numpy(w.vertices * 1.03, w.faces, dev)
    tv, _ = device.forward(tmesh, "exact", "f32", grid=grid, n0=n0, count=cnt)
    targets = (tv > 0.5).to(torch.float32)
    del tmesh, tv

    dmesh = device.DeviceMesh.from_numpy(w.vertices, w.faces, dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream()
    ev = {k: [] for k in ("f0", "f1", "b0", "b1")}

    def step(record=False):
        def mark(k):
            if record:
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                ev[k].append(e)
        dmesh.invalidate()  # the vertices moved: re-stage every kernel's records
        mark("f0")
        vals, flags = device.forward(dmesh, "exact", "f32", grid=grid, n0=n0, count=cnt)
        mark("f1")
        coefs, sums = device.loss_terms(vals, flags, targets)
        mark("b0")
        fg = device.face_grad(dmesh, "exact", "f32", coefs, grid=grid, n0=n0, count=cnt)
        mark("b1")
        g = device.vertex_grad(dmesh, fg)
        buf = torch.cat([g.reshape(-1), sums[:3]])
        if world > 1:
            dist.all_reduce(buf)
        return buf[:-3].reshape(-1, 3) / buf[-2], buf[-3] / buf[-2]

    F = w.n_faces
    active = int(dmesh.exact_grad_setup()[0].shape[0])
    # per step: [surface eps + pack + forward (+ split finalize)] + [loss terms +
    # loss final] + [surface eps + pack + backward (+ split reduce)] + gather.
    # Large lattices take the strip forward and the strip-pair backward
    # (device.STRIP_MIN_NODES), whose split plans decide the optional launches.
    strip_path = cnt >= device.STRIP_MIN_NODES
    if strip_path:
        n_rows = int(dmesh.exact_pair_setup()[0].shape[0])
        fws = L.lib().wv_fwd_workspace_bytes(L.PACK_EXACTSTRIP_F32, F, cnt)
        bws = L.lib().wv_exact_pair_bwd_workspace_bytes(n_rows, cnt)
    else:
        fws = L.lib().wv_fwd_workspace_bytes(L.PACK_EXACT_F32, F, cnt)
        bws = L.lib().wv_bwd_workspace_bytes(L.PACK_EXACTGRAD_F32, active, cnt)
    bwd_launches = (3 + (1 if bws else 0)) if active > 0 else 1  # no active face: eps only
    launches = 3 + (1 if fws else 0) + 2 + bwd_launches + 1

    fp32_meas = measured_fp32_peak() if rank == 0 else None
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    e_start = torch.cuda.Event(enable_timing=True)
    e_stop = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e_start.record(stream)
        for _ in range(args.steps):
            flush.zero_()
            grads, loss = step(record=True)
        e_stop.record(stream)
        barrier()
    ms = e_start.elapsed_time(e_stop)
    fwd_ms = statistics.mean(a.elapsed_time(b) for a, b in zip(ev["f0"], ev["f1"]))
    bwd_ms = statistics.mean(a.elapsed_time(b) for a, b in zip(ev["b0"], ev["b1"]))
    t = torch.tensor([ms, fwd_ms, bwd_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t[0]) / args.steps
    fwd_ms, bwd_ms = float(t[1]), float(t[2])
    value = w.pairs / (ms_step / 1e3)

    # --- e2e: host numpy in (mesh + this rank's target slab), host grads out
    e2e = None
    if not args.no_e2e:
        tgt_host = targets.cpu().numpy()
        h2d = w.vertices.nbytes + w.faces.nbytes + tgt_host.nbytes
        d2h = w.vertices.nbytes + 8

        def e2e_step():
            m = device.DeviceMesh.from_numpy(w.vertices, w.faces, dev)
            tg = torch.from_numpy(tgt_host).pin_memory().to(dev, non_blocking=True)
            drv = SlabDriver(_E(m, grid), w.n_nodes, rank, world)
            lo, gr, _, _ = drv.loss_grad(tg)
            return gr.cpu().numpy(), float(lo)

        e2e_step()
        barrier()
        t0 = time.perf_counter()
        e2e_steps = max(1, min(args.steps, 2))
        for _ in range(e2e_steps):
            e2e_step()
        barrier()
        dt = torch.tensor([(time.perf_counter() - t0) / e2e_steps], device=dev,
                          dtype=torch.float64)
        if world > 1:
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e = {"value": w.pairs / float(dt), "unit": "pairs/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h,
               "api": "DeviceMesh.from_numpy + SlabDriver(CudaSlabEvaluator).loss_grad "
                      "(grad.exact_loss_grad's device path), numpy in / numpy grads out"}

    if rank == 0:
        peak, peak_src = peaks()
        fwd_tf = EXACT_FWD_FLOPS * cnt * F / (fwd_ms / 1e3) / 1e12
        # the exact backward launches only faces with a non-cancelling edge
        # (all of them for a soup): count the pairs it actually evaluates
        bwd_tf = EXACT_BWD_FLOPS * cnt * active / (bwd_ms / 1e3) / 1e12
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            from oracle import oracle as orc
            thr = orc.default_threads()
            r, rf, n, dt = cpu_fwd_bwd_rate(w, args.cpu_seconds, thr)
            cpu = {"value": r, "unit": "pairs/s", "cores": thr, "kind": "port",
                   "fwd_pairs_per_s": rf,
                   "sample": f"{n} seeded random nodes of the {w.res[0]}^3 grid x {F} faces, "
                             f"exact f64 fwd (bit-exact C port of _kernels.exact_batch) + exact "
                             f"f64 grad (closed-form oracle), {dt:.1f} s"}
        if strip_path:  # strip forward + strip-pair backward (device.STRIP_MIN_NODES)
            kf, kb = "fwd_f32_kernel<ExactStripPol,RowSrc>", "bwd_f32_kernel<ExactEdgeBwdPair,RowSrc>"
            xf = (EXACT_FWD_EXEC_FLOPS, EXACT_FWD_MUFU, EXACT_FWD_LANE_OPS)
            xb = (EXACT_BWD_EXEC_FLOPS, EXACT_BWD_MUFU, EXACT_BWD_LANE_OPS)
        else:
            kf, kb = "fwd_f32_kernel<ExactPol,RowSrc>", "bwd_f32_kernel<ExactEdgeBwd,RowSrc>"
            xf = (EXACT_FWD_FACE_ORDER_EXEC_FLOPS, 4, 26.75)
            xb = (60.5, 4, 34.7)
        dom = (f"exact_bwd ({kb})", bwd_ms, bwd_tf) if bwd_ms >= fwd_ms \
            else (f"exact_fwd ({kf})", fwd_ms, fwd_tf)
        clk_mhz = clk.summary().get("sm_mhz") or 1965.0
        rfwd = executed(fwd_tf, EXACT_FWD_FLOPS, xf[0], xf[1], fwd_ms, peak, clk_mhz, xf[2])
        rbwd = executed(bwd_tf, EXACT_BWD_FLOPS, xb[0], xb[1], bwd_ms, peak, clk_mhz, xb[2])
        step_tf = (EXACT_FWD_FLOPS * cnt * F + EXACT_BWD_FLOPS * cnt * active) \
            / (ms_step / 1e3) / 1e12
        line = {
            "metric": "point-triangle solid-angle evals/sec fwd & fwd+bwd; 256^3 voxelize ms",
            "value": value, "unit": "pairs/s (exact fwd+bwd)", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": w.name, "faces": F, "grid": list(w.res), "mode": "exact",
                       "step": "pack + exact fwd + loss + exact bwd + vertex gather"
                               + (" + all-reduce" if world > 1 else ""),
                       "l2": "256 MiB buffer zeroed between timed steps (> 126 MB L2)",
                       "parallelism": f"i-slabs x{world}", "active_bwd_faces": active},
            "fwd_pairs_per_s": w.pairs / (fwd_ms / 1e3),
            "bwd_pairs_per_s": w.pairs / (bwd_ms / 1e3),
            "voxelize_ms": fwd_ms,
            "loss": float(loss),
            "roofline": {"bound": "fp32", "achieved": dom[2], "peak": peak, "unit": "TFLOP/s",
                         "frac": dom[2] / peak, "traffic": traffic(w.name, dom[0]),
                         "traffic_unit": "bytes per launch", "kernel": dom[0],
                         "kernel_ms": dom[1],
                         "flops_per_pair": EXACT_BWD_FLOPS if dom[0].startswith("exact_bwd")
                         else EXACT_FWD_FLOPS,
                         # the pipe that bounds the kernel: FMA-pipe lane-ops actually
                         # issued per pair (ncu mix) against 128 per clock per SM
                         "fma_pipe_frac": (rbwd if dom[0].startswith("exact_bwd")
                                           else rfwd)["fma_pipe_frac"],
                         "peak_source": f"FP32 CUDA-core peak 148 SM x 128 lanes x 2 x clock "
                                        f"({peak_src}); MEASURED_PEAKS has no FP32 entry",
                         "peak_measured": fp32_meas,
                         "peak_measured_source": "tools/ffma2_probe (FFMA/FFMA2 chains, this "
                                                 "GPU, before the timed region)",
                         "traffic_note": "dram read+write bytes per launch of this kernel "
                                         "from one ncu --set full capture "
                                         "(profiles/traffic.json); null if not captured for "
                                         "this workload",
                         "frac_note": "achieved uses the pinned algorithmic FLOPs/pair (SURVEY "
                                      "8d); the kernels execute fewer (roofline_fwd/bwd "
                                      "executed_flops_per_pair), so frac may exceed 1 -- "
                                      "fma_frac / xu_frac there are the pipe utilisation"},
            "roofline_fwd": rfwd,
            "roofline_bwd": rbwd,
            "roofline_step": {"achieved": step_tf, "frac": step_tf / peak,
                              "note": "whole step: 63 FLOP per forward pair + 170 per "
                                      "backward pair actually evaluated (active faces)"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


class _E:
    """CudaSlabEvaluator in exact/f32 mode (the product evaluator)."""

    def __new__(cls, dmesh, grid):
        from paper_2407_11272_b200.distributed import CudaSlabEvaluator
        return CudaSlabEvaluator(dmesh, grid, mode="exact", precision="f32")


def run_c4(args):
    """Config C4: a mesh-morphing training batch -- 64 meshes (icosphere(4),
    5120 faces, seeded radial bumps) deformed by a random-init MLP
    [xyz + 32-d latent -> 3, hidden 128x2], soft occupancy loss against
    seeded primitive targets at 64^3; a step = net forward, fused soft
    fwd+loss+bwd for every mesh, net backward, Adam step.  Multi-GPU: the
    meshes shard over ranks, MLP gradients are all-reduced (DP)."""
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    dev = init_dist(local, world)
    local = dev.index
    from paper_2407_11272_b200 import configs, device
    from paper_2407_11272_b200.batch import DeformationNet, batch_occupancy_loss

    B, R = 64, 64
    grid = ((-1.0,) * 3, (1.0,) * 3, (R, R, R))
    per = B // world
    ids = list(range(rank * per, (rank + 1) * per))
    meshes = configs.c4_batch(B)
    faces = torch.from_numpy(meshes[0][1]).to(dev)
    tmpl = torch.stack([torch.from_numpy(meshes[b][0]) for b in ids]).to(dev, torch.float32)
    # targets: exact occupancy of seeded primitives (cube / ellipsoid / torus)
    tg = []
    for b in ids:
        rng = np.random.default_rng(1000 + b)
        kind = b % 3
        if kind == 0:
            h = rng.uniform(0.3, 0.55)
            cv = np.array([[x, y, z] for x in (-h, h) for y in (-h, h) for z in (-h, h)])
            cf = np.array([[0, 2, 3], [0, 3, 1], [4, 5, 7], [4, 7, 6], [0, 1, 5], [0, 5, 4],
                           [2, 6, 7], [2, 7, 3], [0, 4, 6], [0, 6, 2], [1, 3, 7], [1, 7, 5]])
        elif kind == 1:
            cv, cf = configs.icosphere(3, 1.0)
            cv = cv * rng.uniform(0.3, 0.6, size=3)
        else:
            cv, cf = configs.torus(rng.uniform(0.4, 0.55), rng.uniform(0.12, 0.2), 48, 24)
        dm = device.DeviceMesh.from_numpy(cv, cf, dev)
        w, _ = device.forward(dm, "exact", "f32", grid=grid)
        tg.append((w > 0.5).float())
    targets = torch.stack(tg)
    torch.manual_seed(0)
    net = DeformationNet(B).to(dev)
    opt = torch.optim.Adam(net.parameters(), lr=1e-4)  # soft-W MSE is spiky: 1e-3 oscillates
    mid = torch.tensor(ids, device=dev)
    csr = device.DeviceMesh(tmpl[0], faces).csr()

    def step():
        opt.zero_grad(set_to_none=True)
        verts = net(tmpl, mid)
        losses = batch_occupancy_loss(verts, faces, grid, targets, csr=csr)
        loss = losses.mean()
        loss.backward()
        if world > 1:
            for p in net.parameters():
                if p.grad is not None:
                    dist.all_reduce(p.grad)
                    p.grad /= world
        opt.step()
        return loss

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        losses = [step() for _ in range(args.steps)]
        e1.record(stream)
        barrier()
    t = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t) / args.steps
    n_faces = int(faces.shape[0])
    pairs = B * R ** 3 * n_faces
    if rank == 0:
        line = {
            "metric": "point-triangle solid-angle evals/sec (C4: soft fwd+bwd training step)",
            "value": pairs / (ms_step / 1e3), "unit": "pairs/s (soft fwd+bwd)", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": "c4_64x_icosphere4_64", "meshes": B, "faces_per_mesh": n_faces,
                       "grid": [R] * 3, "mode": "soft", "parallelism": f"mesh DP x{world}",
                       "step": "MLP fwd + fused soft fwd/loss/bwd per mesh + MLP bwd + Adam"},
            "loss_first": float(losses[0].detach()), "loss_last": float(losses[-1].detach()),
            "roofline": {"bound": "fp32", "unit": "TFLOP/s", "peak": peaks()[0],
                         "achieved": SOFT_STEP_FLOPS * pairs / (ms_step / 1e3) / 1e12,
                         "frac": SOFT_STEP_FLOPS * pairs / (ms_step / 1e3) / 1e12 / peaks()[0],
                         "flops_per_pair": SOFT_STEP_FLOPS, "traffic": None,
                         "note": "whole training step at the pinned soft fwd 15 + bwd 72 "
                                 "FLOP/pair (SURVEY 8d); MLP/Adam time included"},
            # per batch: 2 packs x (eps + pack), 1 forward (+ split finalize),
            # 2 loss kernels, 1 backward (+ split reduce), 1 gather
            "gpu_launches": args.steps * 11,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_c5(args):
    """Config C5: 1M-face torus, exact forward only (voxelize,
    flagged -> 0.5) at 512^3 = 1.34e14 pairs, i-slabs over ranks.  One step
    takes minutes on one GPU, so this is an explicit measurement
    (``--config c5``), not the default line."""
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    dev = init_dist(local, world)
    local = dev.index
    from paper_2407_11272_b200 import _lib as L, configs, device
    from paper_2407_11272_b200.distributed import slab_range

    w = configs.make("c5")
    n0, cnt = slab_range(w.n_nodes, rank, world)
    grid = (w.lo, w.hi, w.res)
    dmesh = device.DeviceMesh.from_numpy(w.vertices, w.faces, dev)
    out = torch.empty(cnt, dtype=torch.float32, device=dev)
    flags = torch.empty(cnt, dtype=torch.uint8, device=dev)

    def step():
        dmesh.invalidate()
        device.forward(dmesh, "exact", "f32", grid=grid, n0=n0, count=cnt,
                       policy=L.POLICY_HALF, out=out, flags=flags)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        barrier()
    t = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t) / args.steps
    if rank == 0:
        peak, peak_src = peaks()
        clocks = clk.summary()
        clk_mhz = clocks.get("sm_mhz") or 1965.0
        F = w.n_faces
        fwd_tf = EXACT_FWD_FLOPS * cnt * F / (ms_step / 1e3) / 1e12
        rf = executed(fwd_tf, EXACT_FWD_FLOPS, EXACT_FWD_EXEC_FLOPS, EXACT_FWD_MUFU, ms_step,
                      peak, clk_mhz, EXACT_FWD_LANE_OPS)
        line = {
            "metric": "point-triangle solid-angle evals/sec (C5: exact forward / voxelize)",
            "value": w.pairs / (ms_step / 1e3), "unit": "pairs/s (exact fwd)", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": w.name, "faces": F, "grid": list(w.res), "mode": "exact",
                       "step": "pack + exact forward (voxelize, flagged -> 0.5)",
                       "l2": "inputs (48 MB records) L2-resident by design; outputs 537 MB",
                       "parallelism": f"i-slabs x{world}"},
            "voxelize_ms": ms_step,
            "roofline": dict(rf, bound="xu+fp32", peak=peak, unit="TFLOP/s",
                             kernel="exact_fwd (fwd_f32_kernel<ExactStripPol,RowSrc>)",
                             peak_source=peak_src, traffic=None),
            "clocks": clocks,
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
    if args.config == "c4":
        return run_c4(args)
    if args.config == "c5":
        return run_c5(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
