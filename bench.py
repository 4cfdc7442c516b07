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
soup scaled by 1.03, computed once before timing.  ``value`` is the
fwd+bwd pair rate of the whole step; the forward (= the 256^3 voxelize) and
backward rates and ``voxelize_ms`` ride along.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c3|c3r|c1|c2|c3s|c3rs|c4|c5] [--precision f32|f64]

``--gpus N`` without torchrun re-launches itself under
``torch.distributed.run`` with N ranks (one per GPU, NCCL); each rank owns
1/N of the grid (total work fixed: "strong" scaling), time is the max over
ranks.  ``--impl reference`` times the reference's CPU algorithm (the
bit-exact C port in oracle/, all host threads) on a bounded node sample of the
same workload, rank 0 only, and prints the SAME metric / unit / config.

Roofline: ``achieved``/``frac`` are the dominant kernel's EXECUTED FLOP rate
(per-pair counts from the committed ncu capture profiles/exec_mix.json)
against the FP32 (FP64 for --precision f64) CUDA-core peak;
``algorithmic_achieved``/``algorithmic_frac`` use SURVEY 8d's pinned FLOPs per
pair (which the lattice-row / strip / edge-form kernels undercut, so that
figure can exceed 1); ``fma_pipe_frac`` / ``xu_frac`` are the two pipes'
utilisation.
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

# BASELINE.json's metric, printed verbatim by BOTH arms (the driver pairs the
# lines by metric + unit); the per-direction figures ride in extra keys
METRIC = "point-triangle solid-angle evals/sec fwd & fwd+bwd; 256^3 voxelize ms"
UNIT = "pairs/s"

# algorithmic work per point-triangle pair
PINNED = {"exact_fwd": 63, "exact_bwd": 170, "soft_fwd": 15, "soft_bwd": 72}

# the kernels each path launches (names as in the ncu launch list / exec_mix.json)
KERNELS = {
    ("f32", "fwd", True): "fwd_f32_kernel<ExactStripPol,RowSrc>",
    ("f32", "fwd", False): "fwd_f32_kernel<ExactPol,RowSrc>",
    ("f32", "bwd", "trails"): "bwd_f32_kernel<ExactEdgeBwdTrail,RowSrc>",
    ("f32", "bwd", "pairs"): "bwd_f32_kernel<ExactEdgeBwdPair,RowSrc>",
    ("f32", "bwd", "faces"): "bwd_f32_kernel<ExactEdgeBwd,RowSrc>",
    ("f64", "fwd", True): "fwd_f64_strip_kernel<GridSrc>",
    ("f64", "fwd", False): "fwd_f64_kernel<ExactF64Pol,GridSrc>",
    ("f64", "bwd", "faces"): "bwd_f64_kernel<ExactBwd64,GridSrc>",
    ("f64", "bwd", "trails"): "bwd_f64_kernel<ExactTrail64,GridSrc>",
}


def fwd_kernel(prec: str, strip: bool, grid, n0: int, cnt: int) -> str:
    """The forward kernel a lattice range launches: the warp-row variant
    (RowSrcW) when every warp's 256 nodes lie in one k-row (wv_fwd.cuh)."""
    k = KERNELS[(prec, "fwd", strip)]
    if prec == "f32" and int(grid[2][2]) % 256 == 0 and n0 % 256 == 0 and cnt % 256 == 0:
        k = k.replace(",RowSrc>", ",RowSrcW>")
    return k


def exec_mix(kernel: str, workload: str):
    """Executed work per pair of ``kernel`` from profiles/exec_mix.json: the
    entry for this workload, else the kernel's first entry (None if absent)."""
    try:
        ents = json.loads((ROOT / "profiles" / "exec_mix.json").read_text())["entries"]
    except (OSError, ValueError, KeyError):
        return None
    hits = [e for e in ents if e["kernel"] == kernel]
    if not hits and ",RowSrcW>" in kernel:  # the row-kernel capture, if the warp-row one is absent
        hits = [e for e in ents if e["kernel"] == kernel.replace(",RowSrcW>", ",RowSrc>")]
    exact = [e for e in hits if e["workload"] == workload]
    return (exact or hits or [None])[0]


def traffic(workload: str, kernel: str):
    """DRAM bytes per launch of ``kernel`` from a committed ncu capture."""
    try:
        t = json.loads((ROOT / "profiles" / "traffic.json").read_text()).get(workload)
    except (OSError, ValueError):
        return None
    if not t or t["kernel"] != kernel:
        return None
    return t["read"] + t["write"]


def peaks(precision: str = "f32"):
    """CUDA-core peak, TFLOP/s: 148 SMs x lanes x 2 FLOP/FMA x max clock
    (FP32 128 lanes, FP64 64 lanes per SM); MEASURED_PEAKS.json has no
    FP32/FP64 entry, only the clock."""
    p = ROOT / "MEASURED_PEAKS.json"
    sm_mhz, src = 1965.0, "nominal 1965 MHz"
    if p.exists():
        d = json.loads(p.read_text())
        sm_mhz = float(d.get("sm_max_mhz", sm_mhz))
        src = "MEASURED_PEAKS.json sm_max_mhz"
    lanes = 128 if precision == "f32" else 64
    return 148 * lanes * 2 * sm_mhz * 1e6 / 1e12, \
        f"{'FP32' if lanes == 128 else 'FP64'} CUDA-core peak 148 SM x {lanes} lanes x 2 x " \
        f"clock ({src})"


def measured_peaks():
    """FP32 (FFMA/FFMA2) and FP64 (DFMA) throughput measured on this GPU by
    tools/ffma2_probe, TFLOP/s: {"f32": x, "f64": y} (None if unavailable)."""
    exe = ROOT / "tools" / "ffma2_probe"
    out = {"f32": None, "f64": None}
    if not exe.exists():
        return out
    try:
        txt = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60).stdout
    except Exception:
        return out
    f32 = [float(ln.split()[-2]) for ln in txt.splitlines() if "TFLOP/s" in ln
           and ln.startswith("FFMA")]
    f64 = [float(ln.split()[-2]) for ln in txt.splitlines() if ln.startswith("DFMA")]
    out["f32"] = max(f32) if f32 else None
    out["f64"] = max(f64) if f64 else None
    return out


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c3")
    ap.add_argument("--precision", choices=["f32", "f64"], default="f32")
    ap.add_argument("--cpu-nodes", type=int, default=65536,
                    help="lattice nodes in the CPU-baseline sample (SURVEY 8d: 65,536)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                    help="replay the step as a CUDA graph (auto: one rank and < 2^20 nodes, "
                         "where launch overhead matters)")
    return ap.parse_args(argv)


def spawn_ranks(args) -> int:
    """``--gpus N`` outside torchrun: re-launch this command under
    torch.distributed.run with N ranks on 127.0.0.1 (one process per GPU)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", str(ROOT / "bench.py"), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


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


class ClockSampler:
    """SM clock / throttle reasons sampled (NVML) DURING the timed region."""

    def __init__(self, index: int, period: float = 0.1):
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


def count_launches(fn) -> int | None:
    """Kernels of OUR library (namespace wv::) one call of ``fn`` launches,
    counted by the CUDA activity trace (torch.profiler/CUPTI) on an untimed
    call; None if the tracer is unavailable."""
    import torch
    if os.environ.get("CUDA_INJECTION64_PATH"):  # under ncu: CUPTI has one subscriber
        return None
    try:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        n = sum(1 for e in prof.events()
                if e.device_type.name == "CUDA" and "wv::" in e.name)
        return n or None
    except Exception:
        return None


def roofline(kernel: str, workload: str, pairs: float, ms: float, alg_flops: float,
             precision: str, clk_mhz: float, bound: str):
    """Roofline of one kernel launch: executed FLOP rate (committed ncu mix)
    against the CUDA-core peak, the pinned-algorithm rate beside it, and the
    FMA / XU pipe utilisation."""
    peak, peak_src = peaks(precision)
    pairs_s = pairs / (ms / 1e3)
    alg = alg_flops * pairs_s / 1e12
    e = exec_mix(kernel, workload)
    r = {"bound": bound, "unit": "TFLOP/s", "peak": peak, "kernel": kernel, "kernel_ms": ms,
         "pairs_per_launch": pairs, "algorithmic_flops_per_pair": alg_flops,
         "algorithmic_achieved": alg, "algorithmic_frac": alg / peak, "peak_source": peak_src}
    if e is None:
        r.update(achieved=None, frac=None, exec_mix_source=None)
        return r
    fl = e["flops"] if precision == "f32" else e.get("dflops") or e["flops"]
    r.update(achieved=fl * pairs_s / 1e12, frac=fl * pairs_s / 1e12 / peak,
             executed_flops_per_pair=fl,
             exec_mix_source=f"{e['source']} [{e['workload']}]")
    if e.get("lane_ops"):
        r["fma_pipe_frac"] = pairs_s * e["lane_ops"] / (148 * 128 * clk_mhz * 1e6)
        r["fma_lane_ops_per_pair"] = e["lane_ops"]
    if e.get("mufu"):
        r["xu_frac"] = pairs_s * e["mufu"] / (148 * 16 * clk_mhz * 1e6)
        r["mufu_per_pair"] = e["mufu"]
    return r


# ---------------------------------------------------------------------------
# CPU side: the reference algorithm (bit-exact C port, oracle/) on a sample

def _nodes(w, idx):
    from oracle import oracle as orc
    i, rem = np.divmod(idx, w.res[1] * w.res[2])
    j, k = np.divmod(rem, w.res[2])
    ax = [orc.axis_nodes(w.lo[a], w.hi[a], w.res[a]) for a in range(3)]
    return np.stack([ax[0][i], ax[1][j], ax[2][k]], axis=1)


def cpu_fwd_bwd(vertices, faces, w, n: int, threads: int, mode: str = "exact", seed: int = 0,
                precision: str = "f64"):
    """Reference CPU algorithm on ``n`` seeded random lattice nodes: forward
    (bit-exact C port of _kernels.exact_batch / soft_batch) + gradient
    (exact: closed-form oracle -- the reference has no exact-gradient kernel;
    soft: port of _kernels.soft_grad_accum with the reference's per-chunk
    buffers, grad.py:113-127).  Returns (fwd+bwd pairs/s, fwd pairs/s, wall s)."""
    from oracle import oracle as orc
    rng = np.random.default_rng(seed)
    pts = _nodes(w, np.sort(rng.choice(w.n_nodes, size=n, replace=False)))
    if precision == "f32":
        pts = pts.astype(np.float32).astype(np.float64)
    F = len(faces)
    chunk = max(1, n // (threads * 4))
    t0 = time.perf_counter()
    vals, flags = orc.winding_number_batch(vertices, faces, pts, mode=mode, chunk=chunk,
                                           threads=threads)
    t_f = time.perf_counter() - t0
    coefs = np.where(flags, 0.0, 2.0 * (vals - (vals > 0.5)))
    gchunk = max(chunk, n // threads)
    gfn = orc.exact_grad if mode == "exact" else orc.soft_grad
    t1 = time.perf_counter()
    gfn(vertices, faces, pts, coefs, chunk=gchunk, threads=threads)
    t_b = time.perf_counter() - t1
    return n * F / (t_f + t_b), n * F / t_f, t_f + t_b


def cpu_fwd(vertices, faces, w, n: int, threads: int, seed: int = 0):
    """Exact forward only (C5 is forward-only)."""
    from oracle import oracle as orc
    rng = np.random.default_rng(seed)
    pts = _nodes(w, np.sort(rng.choice(w.n_nodes, size=n, replace=False)))
    t0 = time.perf_counter()
    orc.winding_number_batch(vertices, faces, pts, chunk=max(1, n // (threads * 4)),
                             threads=threads)
    dt = time.perf_counter() - t0
    return n * len(faces) / dt, dt


def cpu_desc(threads: int, n: int, what: str, dt: float):
    return {"unit": UNIT, "cores": threads, "cpu_model": cpu_model(), "kind": "port",
            "sample": f"{n} seeded random lattice nodes x all faces: {what}; {dt:.1f} s"}


# ---------------------------------------------------------------------------
# workload descriptions shared by both arms

def exact_config(w, precision: str, world: int, active: int | None = None):
    c = {"workload": w.name, "faces": w.n_faces, "grid": list(w.res), "mode": "exact",
         "precision": precision,
         "step": "pack + exact fwd + loss + exact bwd + vertex gather"
                 + (" + all-reduce" if world > 1 else ""),
         "l2": "256 MiB buffer zeroed between timed steps (> 126 MB L2; outside the "
               "per-step CUDA events)",
         "parallelism": f"i-slabs x{world}"}
    if active is not None:
        c["active_bwd_faces"] = active
    return c


def c4_config(world: int, B=64, R=64, n_faces=5120):
    return {"workload": "c4_64x_icosphere4_64", "meshes": B, "faces_per_mesh": n_faces,
            "grid": [R] * 3, "mode": "soft", "precision": "f32",
            "parallelism": f"mesh DP x{world}",
            "step": "MLP fwd + fused soft fwd/loss/bwd per mesh + MLP bwd + Adam",
            "l2": "inputs re-read every step; 67 MB targets + 16.8 MB W per step"}


def c5_config(w, world: int):
    return {"workload": w.name, "faces": w.n_faces, "grid": list(w.res), "mode": "exact",
            "precision": "f32", "step": "pack + exact forward (voxelize, flagged -> 0.5)",
            "l2": "outputs 537 MB per step (> L2)", "parallelism": f"i-slabs x{world}"}


def line_base(args, world, value, ms_step, dtype, config):
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": dtype, "data": "synthetic", "config": config}


# ---------------------------------------------------------------------------
# reference arm

def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as orc
    from paper_2407_11272_b200 import configs
    threads = orc.default_threads()
    steps = max(1, args.steps)
    # the whole run samples args.cpu_nodes nodes (65,536), split
    # evenly over the timed steps; warm-up steps use a small sample
    per = max(64, -(-args.cpu_nodes // steps))
    if args.config == "c4":
        from paper_2407_11272_b200.configs import c4_batch
        meshes = c4_batch(64)
        g = configs.Workload("c4_mesh", *meshes[0], (-1.0,) * 3, (1.0,) * 3, (64,) * 3)
        per = min(per, g.n_nodes)

        def one(k, n):
            v, f = meshes[k % 64]
            r, rf, dt = cpu_fwd_bwd(v, f, g, n, threads, mode="soft", seed=k,
                                    precision="f32")
            return r, rf, dt
        config = c4_config(world)
        what = "soft f32-rounded nodes: fwd (port of soft_batch) + soft_grad_accum, one mesh"
        pairs_per_step = 64 * 64 ** 3 * len(meshes[0][1])
    elif args.config == "c5":
        w = configs.make("c5")
        per = max(64, -(-min(args.cpu_nodes, 8192) // steps))

        def one(k, n):
            r, dt = cpu_fwd(w.vertices, w.faces, w, n, threads, seed=k)
            return r, r, dt
        config = c5_config(w, world)
        what = "exact f64 fwd (bit-exact C port of _kernels.exact_batch)"
        pairs_per_step = w.pairs
    else:
        w = configs.make(args.config)
        per = min(per, w.n_nodes)

        def one(k, n):
            return cpu_fwd_bwd(w.vertices, w.faces, w, n, threads, seed=k)
        config = exact_config(w, args.precision, world)
        what = ("exact f64 fwd (bit-exact C port of _kernels.exact_batch) + exact f64 grad "
                "(closed-form oracle; the reference has no exact-gradient kernel)")
        pairs_per_step = w.pairs
    for k in range(args.warmup):
        one(1000 + k, 64)
    rates, fwd, tot = [], [], 0.0
    t_all = time.perf_counter()
    for k in range(steps):
        r, rf, dt = one(k, per)
        rates.append(r)
        fwd.append(rf)
        tot += dt
    wall = time.perf_counter() - t_all
    rate = statistics.median(rates)
    line = line_base(args, world, rate, wall * 1e3 / steps, "f64" if args.config != "c4"
                     else "f32", config)
    line["impl"] = "reference"
    line.update({
        "fwd_pairs_per_s": statistics.median(fwd),
        "extrapolated_step_s": pairs_per_step / rate,
        "extrapolated_voxelize_ms": pairs_per_step / statistics.median(fwd) * 1e3,
        "cpu_baseline": dict(cpu_desc(threads, per * steps, what + f"; {per} nodes per step",
                                      tot), value=rate),
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    })
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm: exact fwd+bwd step (C1/C2/C3/C3r and the quarter-size variants)

def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    dev = init_dist(local, world)
    local = dev.index
    from paper_2407_11272_b200 import _lib as L, configs, device
    from paper_2407_11272_b200.distributed import CudaSlabEvaluator, SlabDriver, slab_range

    prec = args.precision
    vdt = torch.float32 if prec == "f32" else torch.float64
    w = configs.make(args.config)
    n0, cnt = slab_range(w.n_nodes, rank, world)
    grid = (w.lo, w.hi, w.res)

    # fixed target: binarized exact occupancy of the soup scaled by 1.03 (untimed)
    tmesh = device.DeviceMesh.from_numpy(w.vertices * 1.03, w.faces, dev)
    tv, _ = device.forward(tmesh, "exact", "f32", grid=grid, n0=n0, count=cnt)
    targets = (tv > 0.5).to(vdt)
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
        vals, flags = device.forward(dmesh, "exact", prec, grid=grid, n0=n0, count=cnt)
        mark("f1")
        coefs, sums = device.loss_terms(vals, flags, targets)
        mark("b0")
        fg = device.face_grad(dmesh, "exact", prec, coefs, grid=grid, n0=n0, count=cnt)
        mark("b1")
        g = device.vertex_grad(dmesh, fg)
        buf = torch.cat([g.reshape(-1), sums[:3]])
        if world > 1:
            dist.all_reduce(buf)
        return buf[:-3].reshape(-1, 3) / buf[-2], buf[-3] / buf[-2]

    F = w.n_faces
    active = int(dmesh.exact_grad_setup()[0].shape[0])
    fwd_strip, _ = device.lattice_paths(dmesh, "exact", prec, grid, n0, cnt)
    bpath = device.backward_path(dmesh, "exact", prec, grid, n0, cnt)
    kf = fwd_kernel(prec, fwd_strip, grid, n0, cnt)
    kb = KERNELS[(prec, "bwd", bpath)]

    meas = measured_peaks() if rank == 0 else {}
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches = count_launches(step)
    use_graph = args.graph == "on" or (args.graph == "auto" and world == 1 and w.n_nodes < 1 << 20)
    graph = None
    if use_graph:
        # the whole step (pack, forward, loss, backward, gather) as one CUDA
        # graph: every kernel still runs on every replay, only the host-side
        # launch overhead goes (C1 is launch-bound); phase times below come
        # from un-graphed steps
        for _ in range(args.steps):
            step(record=True)
        torch.cuda.synchronize()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            step()
        torch.cuda.current_stream().wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        c0 = L.lib().wv_launch_count()
        with torch.cuda.graph(graph):
            g_out = step()
        graph_launches = L.lib().wv_launch_count() - c0
        torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # per-step CUDA events around each step (the L2 flush between steps is
    # outside them)
    ev_s = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev_e = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    lib = L.lib()
    with ClockSampler(local) as clk:
        barrier()
        n_before = lib.wv_launch_count()
        for i in range(args.steps):
            flush.zero_()
            ev_s[i].record(stream)
            if graph is not None:
                graph.replay()
                grads, loss = g_out
            else:
                grads, loss = step(record=True)
            ev_e[i].record(stream)
        barrier()
    # our kernels launched in the timed region: the library's own counter
    # (a replayed graph launches the kernels its capture counted)
    n_timed = (graph_launches * args.steps if graph is not None
               else lib.wv_launch_count() - n_before)
    if world > 1:  # all ranks' launches
        nt = torch.tensor([n_timed], device=dev, dtype=torch.int64)
        dist.all_reduce(nt)
        n_timed = int(nt)
    ms = sum(a.elapsed_time(b) for a, b in zip(ev_s, ev_e))
    fwd_ms = statistics.mean(a.elapsed_time(b) for a, b in zip(ev["f0"], ev["f1"]))
    bwd_ms = statistics.mean(a.elapsed_time(b) for a, b in zip(ev["b0"], ev["b1"]))
    t = torch.tensor([ms, fwd_ms, bwd_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t[0]) / args.steps
    fwd_ms, bwd_ms = float(t[1]), float(t[2])
    value = w.pairs / (ms_step / 1e3)

    # --- e2e: host numpy in (mesh + this rank's target slab), host grads out,
    # through the public device path (DeviceMesh + SlabDriver.loss_grad)
    e2e = None
    if not args.no_e2e:
        tgt_host = targets.cpu().numpy()
        h2d = w.vertices.nbytes + w.faces.nbytes + tgt_host.nbytes
        d2h = w.vertices.nbytes + 8

        def e2e_step():
            m = device.DeviceMesh.from_numpy(w.vertices, w.faces, dev)
            tg = torch.from_numpy(tgt_host).pin_memory().to(dev, non_blocking=True)
            drv = SlabDriver(CudaSlabEvaluator(m, grid, mode="exact", precision=prec),
                             w.n_nodes, rank, world)
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
        e2e = {"value": w.pairs / float(dt), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": e2e_steps,
               "api": "DeviceMesh.from_numpy + SlabDriver(CudaSlabEvaluator).loss_grad "
                      "(grad.exact_loss_grad's device path), numpy in / numpy grads out"}

    if rank == 0:
        clocks = clk.summary()
        clk_mhz = clocks.get("sm_mhz") or 1965.0
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            from oracle import oracle as orc
            thr = orc.default_threads()
            n = min(args.cpu_nodes, w.n_nodes)
            r, rf, dt = cpu_fwd_bwd(w.vertices, w.faces, w, n, thr)
            cpu = dict(cpu_desc(thr, n, "exact f64 fwd (bit-exact C port of "
                                        "_kernels.exact_batch) + exact f64 grad (closed-form "
                                        "oracle; no reference exact-gradient kernel exists)",
                                dt), value=r, fwd_pairs_per_s=rf)
        bound = "fp32 (FMA + XU pipes)" if prec == "f32" else "fp64"
        rf_ = roofline(kf, w.name, cnt * F, fwd_ms, PINNED["exact_fwd"], prec, clk_mhz, bound)
        rb_ = roofline(kb, w.name, cnt * active, bwd_ms, PINNED["exact_bwd"], prec, clk_mhz,
                       bound)
        dom = rb_ if bwd_ms >= fwd_ms else rf_
        dom = dict(dom, traffic=traffic(w.name, dom["kernel"]),
                   traffic_unit="dram read+write bytes per launch (profiles/traffic.json; "
                                "null if not captured for this workload)",
                   peak_measured=meas.get(prec),
                   peak_measured_source="tools/ffma2_probe (FFMA/FFMA2 or DFMA chains, this "
                                        "GPU, before the timed region)")
        line = line_base(args, world, value, ms_step, prec, exact_config(w, prec, world, active))
        line.update({
            "fwd_pairs_per_s": w.pairs / (fwd_ms / 1e3),
            "bwd_pairs_per_s": w.pairs / (bwd_ms / 1e3),
            "voxelize_ms": fwd_ms,
            "loss": float(loss),
            "cuda_graph": use_graph,
            "paths": {"forward": kf, "backward": kb, "backward_records": bpath,
                      "shared_corner_fraction": dmesh.shared_corner_fraction(),
                      "strip_restart_fraction": dmesh.strip_restart_fraction()},
            "roofline": dom,
            "roofline_fwd": rf_,
            "roofline_bwd": rb_,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": n_timed,
            "gpu_launches_source": "the library's launch counter (wv_launch_count) over the "
                                   "timed region, summed over ranks; CUDA-activity cross-check "
                                   "(rank 0): "
                                   + (f"{launches * args.steps} wv:: kernels (torch.profiler, "
                                      "one untimed step x steps)" if launches else "unavailable"),
            "clocks": clocks,
        })
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
# C4: the mesh-morphing training batch

def c4_targets(ids, grid, dev):
    """Exact occupancy of seeded primitives (cube / ellipsoid / torus)."""
    import torch
    from paper_2407_11272_b200 import configs, device
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
    return torch.stack(tg)


def run_c4(args):
    """Config C4: a mesh-morphing training batch -- 64 meshes (icosphere(4),
    5120 faces, seeded radial bumps) deformed by a random-init MLP
    [xyz + 32-d latent -> 3, hidden 128x2], soft occupancy loss against
    seeded primitive targets at 64^3; a step = net forward, fused soft
    fwd+loss+bwd for every mesh, net backward, Adam step.  Multi-GPU: the
    meshes shard over ranks, MLP gradients are all-reduced as ONE flattened
    bucket (DP)."""
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
    tmpl_host = torch.stack([torch.from_numpy(meshes[b][0]) for b in ids]).to(torch.float32)
    tmpl = tmpl_host.to(dev)
    targets = c4_targets(ids, grid, dev)
    torch.manual_seed(0)
    net = DeformationNet(B).to(dev)
    opt = torch.optim.Adam(net.parameters(), lr=1e-4)  # soft-W MSE is spiky: 1e-3 oscillates
    mid = torch.tensor(ids, device=dev)
    csr = device.DeviceMesh(tmpl[0], faces).csr()
    params = [p for p in net.parameters()]
    gbuf = torch.zeros(sum(p.numel() for p in params), device=dev)

    def allreduce_grads():
        # one bucket: flatten every parameter gradient, one NCCL all-reduce,
        # scatter back (the DDP pattern without DDP's hooks)
        off = 0
        for p in params:
            n = p.numel()
            gbuf[off:off + n].copy_(p.grad.reshape(-1))
            off += n
        dist.all_reduce(gbuf)
        gbuf.div_(world)
        off = 0
        for p in params:
            n = p.numel()
            p.grad.copy_(gbuf[off:off + n].view_as(p.grad))
            off += n

    def step(tm=tmpl, tg=targets):
        opt.zero_grad(set_to_none=False)
        verts = net(tm, mid)
        losses = batch_occupancy_loss(verts, faces, grid, tg, csr=csr)
        loss = losses.mean()
        loss.backward()
        if world > 1:
            allreduce_grads()
        opt.step()
        return loss

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches = count_launches(step)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    from paper_2407_11272_b200 import _lib as L
    with ClockSampler(local) as clk:
        barrier()
        n_before = L.lib().wv_launch_count()
        e0.record(stream)
        losses = [step() for _ in range(args.steps)]
        e1.record(stream)
        barrier()
        n_timed = L.lib().wv_launch_count() - n_before
    if world > 1:  # all ranks' launches
        nt = torch.tensor([n_timed], device=dev, dtype=torch.int64)
        dist.all_reduce(nt)
        n_timed = int(nt)
    t = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t) / args.steps
    n_faces = int(faces.shape[0])
    pairs = B * R ** 3 * n_faces

    # e2e: every step copies its inputs (mesh templates + target occupancy)
    # from pinned host memory and reads the loss back
    e2e = None
    if not args.no_e2e:
        tm_pin = tmpl_host.pin_memory()
        tg_pin = targets.to(torch.uint8).cpu().pin_memory()

        def e2e_step():
            tm = tm_pin.to(dev, non_blocking=True)
            tg = tg_pin.to(dev, non_blocking=True).float()
            return float(step(tm, tg))

        e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        barrier()
        dt = torch.tensor([(time.perf_counter() - t0) / args.steps], device=dev,
                          dtype=torch.float64)
        if world > 1:
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e = {"value": pairs / float(dt), "unit": UNIT,
               "h2d_bytes_per_step": tm_pin.numel() * 4 + tg_pin.numel(),
               "d2h_bytes_per_step": 4, "steps": args.steps,
               "api": "batch.batch_occupancy_loss (autograd) + Adam; templates (f32) and "
                      "targets (u8) copied from pinned host each step, loss read back"}
    if rank == 0:
        clocks = clk.summary()
        clk_mhz = clocks.get("sm_mhz") or 1965.0
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            from oracle import oracle as orc
            thr = orc.default_threads()
            g = configs.Workload("c4_mesh", *meshes[0], (-1.0,) * 3, (1.0,) * 3, (R,) * 3)
            n = min(args.cpu_nodes, g.n_nodes)
            r, rf, dt = cpu_fwd_bwd(meshes[0][0], meshes[0][1], g, n, thr, mode="soft",
                                    precision="f32")
            cpu = dict(cpu_desc(thr, n, "mesh 0: soft fwd (port of _kernels.soft_batch) + "
                                        "soft_grad_accum (per-chunk buffers)", dt),
                       value=r, fwd_pairs_per_s=rf)
        peak, peak_src = peaks("f32")
        alg = (PINNED["soft_fwd"] + PINNED["soft_bwd"]) * pairs / (ms_step / 1e3) / 1e12
        line = line_base(args, world, pairs / (ms_step / 1e3), ms_step, "f32", c4_config(world))
        line.update({
            "loss_first": float(losses[0].detach()), "loss_last": float(losses[-1].detach()),
            "roofline": {"bound": "fp32", "unit": "TFLOP/s", "peak": peak,
                         "achieved": None, "frac": None,
                         "algorithmic_achieved": alg, "algorithmic_frac": alg / peak,
                         "algorithmic_flops_per_pair": PINNED["soft_fwd"] + PINNED["soft_bwd"],
                         "traffic": None, "peak_source": peak_src,
                         "note": "whole training step at the pinned soft fwd 15 + bwd 72 "
                                 "FLOP/pair (SURVEY 8d); MLP/Adam time included"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": n_timed,
            "gpu_launches_source": "the library's launch counter (wv_launch_count) over the "
                                   "timed region, summed over ranks; CUDA-activity cross-check "
                                   "(rank 0): "
                                   + (f"{launches * args.steps} wv:: kernels (torch.profiler)"
                                      if launches else "unavailable"),
            "clocks": clocks,
        })
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
# C5: 1M faces at 512^3, forward only

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
    launches = count_launches(step)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local, period=0.5) as clk:
        barrier()
        n_before = L.lib().wv_launch_count()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        barrier()
        n_timed = L.lib().wv_launch_count() - n_before
    if world > 1:  # all ranks' launches
        nt = torch.tensor([n_timed], device=dev, dtype=torch.int64)
        dist.all_reduce(nt)
        n_timed = int(nt)
    t = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t) / args.steps

    # e2e: the public voxelize from a host mesh to a host grid (537 MB D2H)
    e2e = None
    if not args.no_e2e:
        host = torch.empty(cnt, dtype=torch.float32).pin_memory()

        def e2e_step():
            m = device.DeviceMesh.from_numpy(w.vertices, w.faces, dev)
            v, _ = device.forward(m, "exact", "f32", grid=grid, n0=n0, count=cnt,
                                  policy=L.POLICY_HALF)
            host.copy_(v)

        barrier()
        t0 = time.perf_counter()
        e2e_step()
        barrier()
        dt = torch.tensor([time.perf_counter() - t0], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e = {"value": w.pairs / float(dt), "unit": UNIT,
               "h2d_bytes_per_step": w.vertices.nbytes + w.faces.nbytes,
               "d2h_bytes_per_step": cnt * 4, "steps": 1,
               "api": "DeviceMesh.from_numpy + device.forward (voxelize's device path), "
                      "host values out"}
    if rank == 0:
        clocks = clk.summary()
        clk_mhz = clocks.get("sm_mhz") or 1965.0
        fwd_strip, _ = device.lattice_paths(dmesh, "exact", "f32", grid, n0, cnt)
        kf = fwd_kernel("f32", fwd_strip, grid, n0, cnt)
        rf = roofline(kf, w.name, cnt * w.n_faces, ms_step, PINNED["exact_fwd"], "f32", clk_mhz,
                      "fp32 (FMA + XU pipes)")
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            from oracle import oracle as orc
            thr = orc.default_threads()
            n = 8192
            r, dt = cpu_fwd(w.vertices, w.faces, w, n, thr)
            cpu = dict(cpu_desc(thr, n, "exact f64 fwd (bit-exact C port of "
                                        "_kernels.exact_batch)", dt), value=r)
        line = line_base(args, world, w.pairs / (ms_step / 1e3), ms_step, "f32",
                         c5_config(w, world))
        line.update({"voxelize_ms": ms_step, "roofline": dict(rf, traffic=None),
                     "cpu_baseline": cpu, "e2e": e2e,
                     "gpu_launches": n_timed,
                     "gpu_launches_source": "the library's launch counter (wv_launch_count) "
                                            "over the timed region",
                     "clocks": clocks})
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main(argv=None):
    args = parse(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "c4":
        return run_c4(args)
    if args.config == "c5":
        return run_c5(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
