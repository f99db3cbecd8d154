"""Sweep one amg_options field (or env knob) over values for several configs; prints device solve/setup ms.

    python tools/sweep.py --configs C1,C3 --field tail_nnz --values 0,8192,32768 [--reps 3] [--set tail_smem=2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="C3")
ap.add_argument("--field", default="tail_nnz")
ap.add_argument("--values", default="8192")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--set", action="append", default=[], help="extra option key=value (repeatable)")
a = ap.parse_args()

import torch  # noqa: E402
from inputs import gen  # noqa: E402
from paper_1307_6305_b200 import amg  # noqa: E402

dev = torch.device("cuda", 0)
for cfg in a.configs.split(","):
    p = gen.problem(cfg)
    prm = p.params
    arrs = [torch.from_numpy(x).to(dev) if x is not None else None for x in (p.rp, p.ci, p.val, p.d)]
    b = torch.from_numpy(gen.rhs(p.n, prm["seed"])).to(dev)
    x = torch.zeros(p.n, dtype=torch.float64, device=dev)
    for v in a.values.split(","):
        o = amg.amg_options_default(coarsest_size=prm["coarsest_size"])
        for kv in a.set:
            k_, v_ = kv.split("=")
            setattr(o, k_, type(getattr(o, k_))(float(v_)))
        setattr(o, a.field, type(getattr(o, a.field))(float(v)) if a.field != "kappa" else float(v))
        best = None
        for r in range(a.reps + 1):
            h = amg.amg_setup(*arrs, prm["passes"], prm["degree"], o)
            x.zero_()
            st, it, rr = amg.amg_solve(h, b, x, prm["tol"], prm["k_inner"])
            info = amg.amg_get_info(h)
            amg.amg_free(h)
            if r == 0:
                continue
            cur = (info["solve_ms"], info["setup_ms"], it, info["launches_per_iter"])
            best = cur if best is None or cur[0] < best[0] else best
        print(f"{cfg} {a.field}={v}: solve {best[0]:.2f} ms setup {best[1]:.2f} ms iters {best[2]} "
              f"ms/iter {best[0]/best[2]:.3f} launches/iter {best[3]} levels {info['n']}", flush=True)
