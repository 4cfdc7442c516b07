"""Executed-instruction mix of a kernel from an ncu report's source page
(``ncu -i REP --page source --csv --print-source sass``): opcodes weighted by
their executed warp-instruction counts, optionally per point-face pair.

    python tools/sass_exec_mix.py REP.ncu-rep [--pairs N] [--top 25]
        [--json profiles/exec_mix.json --kernel NAME --workload W --source TEXT]

With ``--json`` the per-pair FLOPs, FP32 FMA-pipe lane-ops, MUFU ops, FP64
FLOPs and thread-instructions are written into that file's ``entries``
(replacing the entry with the same kernel and workload): bench.py reads them
for its executed-work roofline.
"""

import argparse
import collections
import csv
import io
import json
import subprocess

# FLOPs per thread-instruction (FMA = 2) and FP32 FMA-pipe lane-ops
F32 = {"FFMA": (2, 1), "FADD": (1, 1), "FMUL": (1, 1),
       "FFMA2": (4, 2), "FADD2": (2, 2), "FMUL2": (2, 2)}
F64 = {"DFMA": 2, "DADD": 1, "DMUL": 1}


def counts(mix, pairs):
    """Per-pair executed work from an opcode -> warp-instruction Counter."""
    per = lambda n: n * 32 / pairs  # noqa: E731
    fl = lo = mu = df = 0.0
    for op, n in mix.items():
        base = op.split(".")[0]
        if base in F32:
            fl += F32[base][0] * per(n)
            lo += F32[base][1] * per(n)
        elif base in F64:
            df += F64[base] * per(n)
        elif base == "MUFU":
            mu += per(n)
    return {"flops": round(fl, 3), "lane_ops": round(lo, 3), "mufu": round(mu, 3),
            "dflops": round(df, 3), "thread_instr": round(per(sum(mix.values())), 3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--pairs", type=float, default=0.0)
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("--json", default=None)
    ap.add_argument("--kernel", default=None)
    ap.add_argument("--workload", default=None)
    ap.add_argument("--source", default="")
    ap.add_argument("--nth", type=int, default=0, help="which kernel of the report (0 = first)")
    a = ap.parse_args()
    txt = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source",
                          "sass"], check=True, capture_output=True, text=True).stdout
    lines = txt.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    # the report holds one table per profiled kernel, each starting with a
    # header row: keep the nth
    starts = [i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r]
    rows = rows[starts[a.nth]:]
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
    if a.pairs:
        c = counts(mix, a.pairs)
        print("per pair:", json.dumps(c))
        if a.json:
            doc = json.load(open(a.json))
            ent = dict(kernel=a.kernel, workload=a.workload, **c, source=a.source)
            doc["entries"] = [e for e in doc["entries"]
                              if (e["kernel"], e["workload"]) != (a.kernel, a.workload)] + [ent]
            with open(a.json, "w") as fh:
                json.dump(doc, fh, indent=1)
                fh.write("\n")


if __name__ == "__main__":
    main()
