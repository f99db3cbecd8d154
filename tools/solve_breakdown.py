"""Per-kernel breakdown of the SOLVE part of an ncu launch list (tools/prof_step.py under ncu).

    python tools/solve_breakdown.py gpurun_out/launches.csv [--iters K]

The solve starts after the last setup-only kernel (coarse inverse Gauss-Jordan / SELL encode).
Times are ncu's (cold, serialised): compare shares, not absolutes.
"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import load, short  # noqa: E402

path = sys.argv[1]
iters = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else 1
rows = load(path)
idx = max(i for i, r in enumerate(rows) if any(k in r["name"] for k in ("gj_step", "k_sell_encode", "pair_codes")))
sol = rows[idx + 1:]
tot = sum(r["us"] for r in sol)
print(f"{len(sol)} solve launches, {tot / 1e3:.3f} ms serialised ({tot / 1e3 / iters:.3f} ms per outer iteration)")
agg = defaultdict(lambda: [0, 0.0, 0.0])
for r in sol:
    k = short(r["name"]) + " g" + r["grid"].replace(", 1, 1)", ")")
    a = agg[k]
    a[0] += 1
    a[1] += r["us"]
    a[2] += r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    gbs = v[2] / (v[1] * 1e3) if v[1] else 0
    print(f"{k:80s} {v[0]:5d} {v[1] / 1e3:8.3f} ms {100 * v[1] / tot:5.1f}% {v[1] / v[0]:8.2f} us {gbs:7.0f} GB/s")
