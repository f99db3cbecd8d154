"""Offline gather-locality of a coarse level under candidate row orders (CPU only; the oracle builds
the hierarchy).  For every 32-row SELL slice it counts the distinct 32-byte sectors and 128-byte
lines its x gathers touch, and the column-offset range (int16 fits or not).

    python tools/level_order.py C4 --level 1 [--rcm]

Orders: the Galerkin numbering (aggregate leader order), BFS levels from vertex 0, and (BFS distance
from vertex 0, BFS distance from the farthest vertex of that search, old index) -- the solve-order
renumbering tried in round 2 session 3 and not kept.  --rcm adds scipy's
reverse Cuthill-McKee.
"""
import argparse
import os
import sys

import numpy as np
import scipy.sparse as sp
import scipy.sparse.csgraph as csg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from inputs import gen  # noqa: E402
from oracle import oracle as O  # noqa: E402


def stats(rp, ci, label):
    n = len(rp) - 1
    rl = np.diff(rp)
    ns = (n + 31) // 32
    row = np.repeat(np.arange(n), rl)
    sl = row // 32
    sec = np.unique(sl.astype(np.int64) * (n // 4 + 2) + ci // 4).size
    lines = np.unique(sl.astype(np.int64) * (n // 16 + 2) + ci // 16).size
    off = ci.astype(np.int64) - row
    print(f"{label:28s} sectors/slice {sec / ns:7.1f}  lines/slice {lines / ns:6.1f}  gathers/slice "
          f"{len(ci) / ns:6.1f}  offsets [{off.min()}, {off.max()}]  beyond int16 {100 * (np.abs(off) > 32767).mean():.3f}%")


def permuted(A, order):
    B = A[order][:, order].tocsr()
    return B.indptr, B.indices


ap = argparse.ArgumentParser()
ap.add_argument("config", default="C4", nargs="?")
ap.add_argument("--level", type=int, default=1)
ap.add_argument("--rcm", action="store_true")
a = ap.parse_args()

p = gen.problem(a.config)
prm = p.params
H = O.Hierarchy(p.rp, p.ci, p.val, p.d, prm["passes"], prm["degree"], coarsest_size=prm["coarsest_size"])
rp, ci, _ = H.level_csr(a.level)
n = len(rp) - 1
A = sp.csr_matrix((np.ones(len(ci)), ci, rp), shape=(n, n))
stats(rp, ci, "Galerkin (leader) order")
d0 = csg.shortest_path(A, method="D", unweighted=True, indices=0)
stats(*permuted(A, np.lexsort((np.arange(n), d0))), "BFS levels from 0")
far = int(np.argmax(np.where(np.isinf(d0), -1, d0)))
d1 = csg.shortest_path(A, method="D", unweighted=True, indices=far)
key0 = np.where(np.isinf(d0), np.inf, d0)
stats(*permuted(A, np.lexsort((np.arange(n), d1, key0))), "(d0, d_far, old)")
if a.rcm:
    stats(*permuted(A, csg.reverse_cuthill_mckee(A, symmetric_mode=True)), "reverse Cuthill-McKee")
