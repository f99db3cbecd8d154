"""One setup + solve of a config through the C ABI (for ncu launch lists / setup traces).

    python tools/prof_step.py C3 [--max-iter K] [--reps R] [--no-graphs]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("config", default="C3", nargs="?")
ap.add_argument("--max-iter", type=int, default=500)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--no-graphs", action="store_true")
ap.add_argument("--size", type=int, default=None)
ap.add_argument("--user-stream", action="store_true")
ap.add_argument("--mis-k", type=int, default=0)
a = ap.parse_args()

import torch  # noqa: E402
from inputs import gen  # noqa: E402
from paper_1307_6305_b200 import amg  # noqa: E402

p = gen.problem(a.config, size=a.size)
prm = p.params
dev = torch.device("cuda", 0)
arrs = [torch.from_numpy(x).to(dev) if x is not None else None for x in (p.rp, p.ci, p.val, p.d)]
b = torch.from_numpy(gen.rhs(p.n, prm["seed"])).to(dev)
x = torch.zeros(p.n, dtype=torch.float64, device=dev)
o = amg.amg_options_default(coarsest_size=prm["coarsest_size"], max_iter=a.max_iter, use_graphs=0 if a.no_graphs else 1)
o.mis_k = a.mis_k
if os.environ.get("AMG_COMPRESS"):
    o.compress = int(os.environ["AMG_COMPRESS"])
if os.environ.get("AMG_TAIL_NNZ"):
    o.tail_nnz = int(os.environ["AMG_TAIL_NNZ"])
if a.user_stream:
    o.stream = torch.cuda.current_stream(dev).cuda_stream
for r in range(a.reps):
    t0 = time.perf_counter()
    h = amg.amg_setup(*arrs, prm["passes"], prm["degree"], o)
    t1 = time.perf_counter()
    x.zero_()
    st, it, rr = amg.amg_solve(h, b, x, prm["tol"], prm["k_inner"])
    t2 = time.perf_counter()
    info = amg.amg_get_info(h)
    amg.amg_free(h)
    print(f"rep {r}: setup {1e3*(t1-t0):.1f} ms (dev {info['setup_ms']:.1f}) solve {1e3*(t2-t1):.1f} ms "
          f"(dev {info['solve_ms']:.1f}) iters {it} relres {rr:.3e} launches/iter {info['launches_per_iter']} "
          f"smoother {info['prof_smoother_ms']/max(1,info['prof_smoother_launches'])*1e3:.1f} us/launch", flush=True)
