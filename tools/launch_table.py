"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_table.py gpurun_out/launches.csv [--top 12]
"""
import csv
import sys

UNITS = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
         "s": 1e3, "second": 1e3}


def main():
    path = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 12
    h, tot, cnt = None, {}, {}
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            h = r
            continue
        if h and len(r) == len(h):
            d = dict(zip(h, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                k = d["Kernel Name"].split("(")[0]
                v = float(d["Metric Value"].replace(",", "")) * UNITS[d["Metric Unit"]]
                tot[k] = tot.get(k, 0.0) + v
                cnt[k] = cnt.get(k, 0) + 1
    s = sum(tot.values())
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        print("%-78s %10.2f ms x%-4d %5.1f%%" % (k[:78], v, cnt[k], 100 * v / s))


if __name__ == "__main__":
    main()
