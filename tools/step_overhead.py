"""Host-side overheads of one step (setup / solve / free) on a config: wall time of each ABI call and
the graph capture inside the first solve.   python tools/step_overhead.py C3"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from inputs import gen  # noqa: E402
from paper_1307_6305_b200 import amg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
p = gen.problem(cfg)
prm = p.params
dev = torch.device("cuda", 0)
arrs = [torch.from_numpy(x).to(dev) if x is not None else None for x in (p.rp, p.ci, p.val, p.d)]
b = torch.from_numpy(gen.rhs(p.n, prm["seed"])).to(dev)
x = torch.zeros(p.n, dtype=torch.float64, device=dev)
o = amg.amg_options_default(coarsest_size=prm["coarsest_size"])
for r in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = amg.amg_setup(*arrs, prm["passes"], prm["degree"], o)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    x.zero_()
    st, it, rr = amg.amg_solve(h, b, x, prm["tol"], prm["k_inner"])
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    info = amg.amg_get_info(h)
    amg.amg_free(h)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"rep {r}: setup {1e3*(t1-t0):.2f} ms (dev {info['setup_ms']:.2f}) solve {1e3*(t2-t1):.2f} ms "
          f"(dev {info['solve_ms']:.2f}) free {1e3*(t3-t2):.2f} ms", flush=True)
