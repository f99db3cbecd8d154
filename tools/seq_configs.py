"""Several configs one after the other in ONE process (setup + solve + free, device inputs), to see
whether a config's solve time depends on what ran before it (the state of the stream-ordered pool).

    python tools/seq_configs.py C3 C4 [--reps 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="+")
ap.add_argument("--reps", type=int, default=3)
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
    for r in range(a.reps):
        h = amg.amg_setup(*arrs, prm["passes"], prm["degree"], o)
        x.zero_()
        st, it, rr = amg.amg_solve(h, b, x, prm["tol"], prm["k_inner"])
        info = amg.amg_get_info(h)
        amg.amg_free(h)
        print(f"{cfg} rep {r}: setup {info['setup_ms']:.2f} ms solve {info['solve_ms']:.2f} ms iters {it}", flush=True)
    del arrs, b, x
    torch.cuda.empty_cache()
