"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) per kernel name.

    python tools/ncu_summary.py gpurun_out/launches.csv [--skip N] [--last N]
"""
import csv
import re
import sys
from collections import OrderedDict, defaultdict


def load(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.DictReader(lines)
    cur = {}
    for r in rd:
        key = (r["ID"], r["Kernel Name"])
        if key not in cur:
            cur[key] = {"id": int(r["ID"]), "name": r["Kernel Name"], "grid": r.get("Grid Size", ""),
                        "block": r.get("Block Size", "")}
            rows.append(cur[key])
        val = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        m = r["Metric Name"]
        if m == "gpu__time_duration.sum":
            cur[key]["us"] = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                              "msecond": 1e3}.get(unit, 1e-3) * val
        elif m.startswith("dram__bytes"):
            mult = {"byte": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}.get(unit, 1)
            cur[key][m] = val * mult
    return rows


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = name.replace("void ", "")
    return name[:70]


def main():
    path = sys.argv[1]
    rows = load(path)
    args = sys.argv[2:]
    if "--skip" in args:
        rows = rows[int(args[args.index("--skip") + 1]):]
    if "--last" in args:
        rows = rows[-int(args[args.index("--last") + 1]):]
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    tot = 0.0
    for r in rows:
        k = short(r["name"])
        a = agg[k]
        a[0] += 1
        a[1] += r.get("us", 0.0)
        a[2] += r.get("dram__bytes_read.sum", 0.0) + r.get("dram__bytes_write.sum", 0.0)
        tot += r.get("us", 0.0)
    print(f"{len(rows)} launches, {tot/1e3:.3f} ms total (serialised, cold)")
    print(f"{'kernel':72s} {'n':>6s} {'ms':>9s} {'share':>6s} {'us/launch':>10s} {'GB/s':>8s}")
    for k, (n, us, by) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:72s} {n:6d} {us/1e3:9.3f} {100*us/tot:5.1f}% {us/n:10.2f} {by/(us*1e-6)/1e9 if us else 0:8.0f}")


if __name__ == "__main__":
    main()
