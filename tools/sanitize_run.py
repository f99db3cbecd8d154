"""Small end-to-end runs of the library for compute-sanitizer: C1, C2 and the C3 recipe
at 1024^2 (compressed level 0, TMA-staged smoother with its mbarrier ring, > 9,472 slices), each a
setup + a short solve + one B_0(r) through the C ABI, plus a two-rank row-partitioned C1 (thread
communicators: halo exchange, split views, dot allreduce).  Exits non-zero on any library error.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [--quick]
"""
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from inputs import gen  # noqa: E402
from paper_1307_6305_b200 import amg, dist  # noqa: E402

quick = "--quick" in sys.argv
cases = [("C1", None, 500), ("C2", None, 500), ("C3", 1024, 3 if quick else 40)]
for name, size, max_iter in cases:
    p = gen.problem(name, size=size)
    prm = p.params
    o = amg.amg_options_default(coarsest_size=prm["coarsest_size"], max_iter=max_iter)
    h = amg.amg_setup(p.rp, p.ci, p.val, p.d, prm["passes"], prm["degree"], o)
    b = gen.rhs(p.n, 0)
    x = np.zeros(p.n)
    st, it, rr = amg.amg_solve(h, b, x, prm["tol"], prm["k_inner"])
    z = np.empty(p.n)
    amg.amg_level_precond(h, 0, prm["k_inner"], b, z)
    info = amg.amg_get_info(h)
    amg.amg_free(h)
    print(f"{name} n={p.n} status={st} iters={it} relres={rr:.3e} level0_format={info['level0_format']} "
          f"level0_path={info['level0_path']}", flush=True)
    assert np.all(np.isfinite(x)) and np.all(np.isfinite(z))

# row-partitioned, two thread ranks
p = gen.problem("C1")
prm = p.params
P = 2
offs = dist.row_blocks(p.n, P)
comms = amg.amg_comm_init_threads(P)
errs = []
b = gen.rhs(p.n, 0)


def rank(k):
    try:
        import torch

        torch.cuda.set_device(0)
        lrp, lci, lv, ld = dist.local_block(p.rp, p.ci, p.val, p.d, offs[k], offs[k + 1])
        o = amg.amg_options_default(coarsest_size=prm["coarsest_size"], gather_rows=300)
        h = amg.amg_setup_dist(comms[k], p.n, offs[k], lrp, lci, lv, ld, prm["passes"], prm["degree"], o)
        x = np.zeros(offs[k + 1] - offs[k])
        st, it, rr = amg.amg_solve(h, np.ascontiguousarray(b[offs[k]:offs[k + 1]]), x, prm["tol"], prm["k_inner"])
        amg.amg_free(h)
        print(f"dist rank {k}: status={st} iters={it} relres={rr:.3e}", flush=True)
    except Exception as e:  # noqa: BLE001
        errs.append(e)


ts = [threading.Thread(target=rank, args=(k,)) for k in range(P)]
for t in ts:
    t.start()
for t in ts:
    t.join()
for c in comms:
    amg.amg_comm_free(c)
if errs:
    raise errs[0]
print("sanitize_run ok", flush=True)
