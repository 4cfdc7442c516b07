"""Executed-instruction mix of a kernel from an ncu report's source page
(``ncu -i REP --page source --csv --print-source sass``): opcodes weighted by
their executed warp-instruction counts, optionally per point-face pair.

    python tools/sass_exec_mix.py REP.ncu-rep [--pairs N] [--top 25]
"""

import argparse
import collections
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--pairs", type=float, default=0.0)
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    txt = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source",
                          "sass"], check=True, capture_output=True, text=True).stdout
    lines = txt.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    head = rows[0]
    isrc, iex, ism = head.index("Source"), head.index("Instructions Executed"), head.index(
        "Warp Stall Sampling (All Samples)")
    mix = collections.Counter()
    smp = collections.Counter()
    for r in rows[1:]:
        if len(r) <= iex or not r[iex]:
            continue
        try:
            float(r[iex])
        except ValueError:
            break  # the next kernel's table: report the first only
        op = r[isrc].strip().split()
        if not op:
            continue
        o = op[0]
        if o.startswith("@"):
            o = op[1] if len(op) > 1 else o
        n = float(r[iex])
        mix[o] += n
        smp[o] += float(r[ism] or 0)
    tot = sum(mix.values())
    print(f"executed warp-instructions: {tot:.4g}" +
          (f"  ({tot * 32 / a.pairs:.2f} thread-instr per pair)" if a.pairs else ""))
    for o, n in mix.most_common(a.top):
        per = f"  {n * 32 / a.pairs:7.3f}/pair" if a.pairs else ""
        print(f"  {o:28s} {n:14.4g} {100 * n / tot:6.2f}%{per}  samples {smp[o]:.0f}")


if __name__ == "__main__":
    main()
