"""GPU timeline of one setup + solve through the C ABI, from CUPTI (torch.profiler sees every kernel of
the process, the library's included).  Reports, for the setup and the solve separately: the span,
the summed kernel time, the idle time between kernels (host waits: read-backs, launch gaps), and the
largest gaps with the kernels around them.  Real (not serialised) timestamps, unlike ncu.

    python tools/timeline.py C3 [--reps 2] [--gaps 25] [--max-iter K] [--json out.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="C3")
ap.add_argument("--reps", type=int, default=2, help="untraced warm-up repetitions first")
ap.add_argument("--gaps", type=int, default=25)
ap.add_argument("--max-iter", type=int, default=500)
ap.add_argument("--json", default=None)
ap.add_argument("--head", type=int, default=0, help="print the first K operations of each part")
ap.add_argument("--top", type=int, default=0, help="print the K kernels with the most summed time per part")
ap.add_argument("--host", action="store_true", help="pinned host inputs and x (the e2e path of bench.py)")
a = ap.parse_args()

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402
from inputs import gen  # noqa: E402
from paper_1307_6305_b200 import amg  # noqa: E402

p = gen.problem(a.config)
prm = p.params
dev = torch.device("cuda", 0)
if a.host:
    arrs = [torch.from_numpy(x).pin_memory() if x is not None else None for x in (p.rp, p.ci, p.val, p.d)]
    b = torch.from_numpy(gen.rhs(p.n, prm["seed"])).pin_memory()
    x = torch.zeros(p.n, dtype=torch.float64).pin_memory()
else:
    arrs = [torch.from_numpy(x).to(dev) if x is not None else None for x in (p.rp, p.ci, p.val, p.d)]
    b = torch.from_numpy(gen.rhs(p.n, prm["seed"])).to(dev)
    x = torch.zeros(p.n, dtype=torch.float64, device=dev)
mark = torch.zeros(1, dtype=torch.float64, device=dev)  # its fill kernel splits setup from solve
o = amg.amg_options_default(coarsest_size=prm["coarsest_size"], max_iter=a.max_iter)


def run():
    h = amg.amg_setup(*arrs, prm["passes"], prm["degree"], o)
    torch.cuda.synchronize()
    x.zero_()
    if a.host:
        mark.zero_()
    torch.cuda.synchronize()
    amg.amg_solve(h, b, x, prm["tol"], prm["k_inner"])
    info = amg.amg_get_info(h)
    amg.amg_free(h)
    return info


for _ in range(a.reps):
    run()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    info = run()
    torch.cuda.synchronize()

ev = []
for e in prof.events():
    if e.device_type.name != "CUDA":
        continue
    t0 = e.time_range.start
    t1 = e.time_range.end
    ev.append((t0, t1, e.name))
ev.sort()
# the solve starts at the zero fill of x (torch's fill kernel between setup and solve)
split = next((i for i, e in enumerate(ev) if "FillFunctor" in e[2]), None)
parts = {"setup": ev[:split] if split is not None else ev, "solve": ev[split + 1:] if split is not None else []}
out = {"config": a.config, "setup_ms_info": info["setup_ms"], "solve_ms_info": info["solve_ms"]}
for name, es in parts.items():
    if not es:
        continue
    span = (es[-1][1] - es[0][0]) / 1e3
    busy = 0.0
    gaps = []
    end = es[0][0]
    for (t0, t1, nm), prev in zip(es, [None] + es[:-1]):
        if t0 > end and prev is not None:
            gaps.append(((t0 - end) / 1e3, prev[2][:60], nm[:60]))
        busy += (t1 - max(t0, end)) / 1e3 if t1 > end else 0.0
        end = max(end, t1)
    idle = span - busy
    if a.head:
        for t0, t1, nm in es[: a.head]:
            print(f"   +{(t0 - es[0][0]) / 1e3:9.3f} ms  {(t1 - t0):8.1f} us  {nm[:90]}")
    gaps.sort(reverse=True)
    if a.top:
        from collections import defaultdict
        agg = defaultdict(lambda: [0, 0.0])
        for t0, t1, nm in es:
            k = nm.split("(")[0][:70]
            agg[k][0] += 1
            agg[k][1] += (t1 - t0) / 1e3
        for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[: a.top]:
            print(f"   {t:8.3f} ms {c:6d}x  {k}")
    big = sum(g[0] for g in gaps if g[0] > 0.01)
    print(f"== {name}: span {span:.3f} ms, kernels {len(es)}, busy {busy:.3f} ms, idle {idle:.3f} ms "
          f"(gaps > 10 us: {sum(1 for g in gaps if g[0] > 0.01)}, {big:.3f} ms)")
    for g in gaps[: a.gaps]:
        print(f"   {1e3 * g[0]:8.1f} us  after {g[1]:60s} before {g[2]}")
    out[name] = {"span_ms": span, "kernels": len(es), "busy_ms": busy, "idle_ms": idle,
                 "gaps_over_10us": sum(1 for g in gaps if g[0] > 0.01), "gap_ms_over_10us": big}
if a.json:
    with open(a.json, "w") as f:
        json.dump(out, f, indent=1)
