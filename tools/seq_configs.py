"""Several configs one after the other in ONE process (setup + solve + free, device inputs), to see
whether a config's solve time depends on what ran before it (the state of the stream-ordered pool).

    python tools/seq_configs.py C3 C4 [--reps 3] [--profile]

--profile traces every repetition of the LAST config with CUPTI and prints its solve's busy / idle
split and the kernels whose summed time differs most from the first repetition's.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="+")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--profile", action="store_true")
a = ap.parse_args()

import torch  # noqa: E402
from inputs import gen  # noqa: E402
from paper_1307_6305_b200 import amg  # noqa: E402

dev = torch.device("cuda", 0)
for cfg in a.configs:
    p = gen.problem(cfg)
    prm = p.params
    arrs = [torch.from_numpy(x).to(dev) if x is not None else None for x in (p.rp, p.ci, p.val, p.d)]
    b = torch.from_numpy(gen.rhs(p.n, prm["seed"])).to(dev)
    x = torch.zeros(p.n, dtype=torch.float64, device=dev)
    o = amg.amg_options_default(coarsest_size=prm["coarsest_size"])
    base = None
    for r in range(a.reps):
        prof = None
        if a.profile and cfg == a.configs[-1]:
            from torch.profiler import ProfilerActivity, profile
            prof = profile(activities=[ProfilerActivity.CUDA])
            prof.__enter__()
        h = amg.amg_setup(*arrs, prm["passes"], prm["degree"], o)
        torch.cuda.synchronize()
        x.zero_()
        torch.cuda.synchronize()
        st, it, rr = amg.amg_solve(h, b, x, prm["tol"], prm["k_inner"])
        info = amg.amg_get_info(h)
        amg.amg_free(h)
        print(f"{cfg} rep {r}: setup {info['setup_ms']:.2f} ms solve {info['solve_ms']:.2f} ms iters {it}", flush=True)
        if prof is not None:
            torch.cuda.synchronize()
            prof.__exit__(None, None, None)
            ev = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
                        if e.device_type.name == "CUDA")
            split = next(i for i, e in enumerate(ev) if "FillFunctor" in e[2])
            es = ev[split + 1:]
            busy = sum(t1 - t0 for t0, t1, _ in es) / 1e3
            span = (es[-1][1] - es[0][0]) / 1e3
            agg = {}
            for t0, t1, nm in es:
                k = nm.split("(")[0][:72]
                c = agg.setdefault(k, [0, 0.0])
                c[0] += 1
                c[1] += (t1 - t0) / 1e3
            print(f"   solve span {span:.3f} ms, busy {busy:.3f} ms, idle {span - busy:.3f} ms, {len(es)} kernels")
            if base is None:
                base = agg
            else:
                d = sorted(((agg.get(k, [0, 0.0])[1] - base.get(k, [0, 0.0])[1], k) for k in set(agg) | set(base)),
                           key=lambda t: -abs(t[0]))
                for dt, k in d[:8]:
                    print(f"   {dt:+8.3f} ms vs rep 0  {agg.get(k, [0, 0.0])[0]:5d}x {agg.get(k, [0, 0.0])[1]:8.3f} ms  {k}")
    del arrs, b, x
    torch.cuda.empty_cache()
