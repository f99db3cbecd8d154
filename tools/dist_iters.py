"""Outer FCG iterations of the row-partitioned path at full BASELINE size with P thread-emulated ranks
on one GPU (amg_comm_init_threads): decoupled aggregation (reading A20) against global aggregation
(amg_options.global_agg, the single-GPU hierarchy) and the single-GPU solve.
Iteration counts and level sizes only -- thread-emulated timings say nothing about 8 GPUs.

    python tools/dist_iters.py [--P 8] [C3 C4 C5]
"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from inputs import gen  # noqa: E402
from paper_1307_6305_b200 import amg, dist  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--P", type=int, default=8)
ap.add_argument("--gather-rows", type=int, default=50000)
ap.add_argument("configs", nargs="*", default=["C3", "C4", "C5"])
a = ap.parse_args()


def run(p, P, global_agg):
    import torch

    prm = p.params
    offs = dist.row_blocks(p.n, P)
    comms = amg.amg_comm_init_threads(P)
    b = gen.rhs(p.n, prm["seed"])
    out, errs = [None] * P, []

    def fn(r):
        try:
            torch.cuda.set_device(0)
            lrp, lci, lv, ld = dist.local_block(p.rp, p.ci, p.val, p.d, offs[r], offs[r + 1])
            o = amg.amg_options_default(coarsest_size=prm["coarsest_size"], gather_rows=a.gather_rows,
                                        global_agg=int(global_agg))
            t0 = time.perf_counter()
            h = amg.amg_setup_dist(comms[r], p.n, offs[r], lrp, lci, lv, ld, prm["passes"], prm["degree"], o)
            t1 = time.perf_counter()
            x = np.zeros(offs[r + 1] - offs[r])
            st, it, rr = amg.amg_solve(h, np.ascontiguousarray(b[offs[r]:offs[r + 1]]), x, prm["tol"], prm["k_inner"])
            info = amg.amg_get_info(h)
            amg.amg_free(h)
            out[r] = dict(status=st, iters=it, relres=rr, true_relres=info["last_true_relres"],
                          levels=info["levels"], dist_levels=info["dist_levels"], setup_wall_s=t1 - t0)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=fn, args=(r,)) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for c in comms:
        amg.amg_comm_free(c)
    if errs:
        raise errs[0]
    assert len({o["iters"] for o in out}) == 1
    return out[0]


res = {}
gold = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_iters.json")))
for cfg in a.configs:
    p = gen.problem(cfg)
    row = {"single_gpu_oracle_iters": gold.get(cfg, {}).get("iters")}
    for mode in ("decoupled", "global"):
        row[mode] = run(p, a.P, mode == "global")
        print(cfg, mode, row[mode], flush=True)
    res[cfg] = row
print(json.dumps({"P": a.P, "gather_rows": a.gather_rows, "results": res}))
