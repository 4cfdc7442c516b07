"""Instruction mix of a kernel's hot loop from the built library's SASS, and
the executed FP32 work per point-face pair it implies (bench.py's
``*_EXEC_FLOPS`` constants come from here).

    python tools/sass_loop_mix.py KERNEL_SUBSTRING [--pairs-per-iter N] [--lib PATH]

The hot loop is taken as the backward branch whose body has the highest
density of packed FP32 instructions (the innermost pair loop).  Packed ops (FFMA2/FADD2/FMUL2) do two lanes of
work; an FMA counts as 2 FLOPs.  ``--pairs-per-iter``: pairs one loop
iteration processes (8 for the forward face loop: one face x 8 points; 4 for
the backward pair loop: 2 packed pairs, unrolled twice).
"""

from __future__ import annotations

import argparse
import collections
import os
import re
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "..", "paper_2407_11272_b200", "_lib", "libwindvox_b200.so")
FLOPS = {"FFMA2": 4, "FADD2": 2, "FMUL2": 2, "FFMA": 2, "FADD": 1, "FMUL": 1}
LANES = {"FFMA2": 2, "FADD2": 2, "FMUL2": 2, "FFMA": 1, "FADD": 1, "FMUL": 1}


def functions(lib: str) -> dict:
    txt = subprocess.run(["cuobjdump", "-sass", lib], check=True, capture_output=True,
                         text=True).stdout
    out = {}
    for part in re.split(r"\n\s*Function : ", txt)[1:]:
        name, body = part.split("\n", 1)
        ins = []
        for line in body.split("\n"):
            m = re.match(r"\s*/\*([0-9a-f]{4,5})\*/\s+(.*?);", line)
            if m:
                ins.append((int(m.group(1), 16), m.group(2).strip()))
        out[name.strip()] = ins
    return out


def opcode(s: str) -> str:
    return re.sub(r"^@!?U?P\w+\s+", "", s).split()[0]


def hot_loop(ins):
    best = None
    for a, s in ins:
        m = re.search(r"BRA.*?(0x[0-9a-f]+)", s)
        if not m:
            continue
        t = int(m.group(1), 16)
        if t >= a:
            continue
        body = [x for x in ins if t <= x[0] <= a]
        packed = sum(1 for _, s2 in body if opcode(s2) in ("FFMA2", "FADD2", "FMUL2"))
        dens = packed / len(body)
        if packed >= 8 and (best is None or dens > best[0]):
            best = (dens, t, a, body)
    return best


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("kernel")
    ap.add_argument("--pairs-per-iter", type=float, default=8.0)
    ap.add_argument("--lib", default=LIB)
    a = ap.parse_args()
    for name, ins in functions(a.lib).items():
        if a.kernel not in name:
            continue
        best = hot_loop(ins)
        if best is None:
            continue
        _, t, e, body = best
        h = collections.Counter(opcode(s) for _, s in body)
        flops = sum(FLOPS.get(k, 0) * v for k, v in h.items())
        lanes = sum(LANES.get(k, 0) * v for k, v in h.items())
        mufu = sum(v for k, v in h.items() if k.startswith("MUFU"))
        n = a.pairs_per_iter
        print(name)
        print(f"  loop {hex(t)}..{hex(e)}: {len(body)} instructions")
        print("  mix:", ", ".join(f"{k} {v}" for k, v in h.most_common(16)))
        print(f"  per pair: {flops / n:.2f} FP32 FLOPs, {lanes / n:.2f} FP32 lane-ops, "
              f"{mufu / n:.2f} MUFU, {len(body) / n:.2f} warp-instructions (incl. rare-path code)")


if __name__ == "__main__":
    main()
