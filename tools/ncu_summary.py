"""Summarise an ncu --set full report for profiles/: the pipe/issue/occupancy
readings, DRAM traffic, executed FP32 instruction counts and the stall mix.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [--pairs N] > profiles/x_summary.txt

``--pairs`` (point-face pairs of the launch) adds per-pair instruction and
FLOP counts.  Reads the report with ``ncu -i ... --page raw --csv``.
"""

from __future__ import annotations

import argparse
import csv
import io
import subprocess

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.per_cycle_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second",
    "smsp__warps_eligible.avg.per_cycle_active",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_ops_fadd_fmul_ffma_pred_on.sum",
]
STALL = "smsp__average_warp_latency_issue_stalled_"
STALL2 = "smsp__pcsamp_warps_issue_stalled_"


def rows(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    head, units, data = r[0], r[1], r[2:]
    return head, units, data


def num(s: str):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return None


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--pairs", type=float, default=None)
    a = ap.parse_args()
    head, units, data = rows(a.report)
    col = {h: i for i, h in enumerate(head)}
    for d in data:
        print("----")
        print("  Kernel Name =", d[col["Kernel Name"]][:100])
        for k in KEYS:
            if k in col:
                print(f"  {k} = {d[col[k]]} {units[col[k]]}".rstrip())
        if a.pairs:
            ie = num(d[col["smsp__inst_executed.sum"]]) if "smsp__inst_executed.sum" in col else None
            if ie:
                print(f"  warp instructions per pair = {ie / a.pairs:.3f}"
                      f"  (thread instructions per pair = {32 * ie / a.pairs:.2f})")
            k = "smsp__sass_thread_inst_executed_ops_fadd_fmul_ffma_pred_on.sum"
            if k in col and num(d[col[k]]):
                print(f"  executed FP32 FLOPs per pair (ncu ops metric) = {num(d[col[k]]) / a.pairs:.2f}")
        stalls = []
        for h, i in col.items():
            for pre in (STALL2,):
                if h.startswith(pre) and not h.endswith("_not_issued"):
                    v = num(d[i])
                    if v:
                        stalls.append((h[len(pre):], v))
        tot = sum(v for _, v in stalls)
        if tot:
            print("  stall mix (pc sampling):")
            for n, v in sorted(stalls, key=lambda x: -x[1])[:10]:
                print(f"   {n:30s} {100 * v / tot:5.1f}%")


if __name__ == "__main__":
    main()
