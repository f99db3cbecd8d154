"""Seeded synthetic workloads (BASELINE.json configs C1-C5) and small test graphs.

Shared by the oracle tests, the GPU parity tests and bench.py.  Holds none of the
method's arithmetic (see inputs/gen.c header): it builds the problem of PAPER.md
Eq. (prob) (lines 26-30) -- the weighted graph Laplacian L (CSR with diagonal,
sorted columns, int64 row_ptr / int32 col / fp64 val) and the lower-order terms
d (None for the pure, singular graph Laplacian) -- and the
seeded right-hand side.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libgen.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-D_DEFAULT_SOURCE", "-fPIC", "-shared",
                               "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        i64, u64, vp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p
        lib.gen_rhs.argtypes = [i64, u64, i64, vp]
        lib.gen_grid2d_nnz.argtypes = [i64]
        lib.gen_grid2d_nnz.restype = i64
        lib.gen_grid3d_nnz.argtypes = [i64]
        lib.gen_grid3d_nnz.restype = i64
        lib.gen_grid2d.argtypes = [i64, vp, vp, vp, vp]
        lib.gen_grid3d.argtypes = [i64, vp, vp, vp, vp]
        lib.gen_rgg_build.argtypes = [i64, u64]
        lib.gen_rgg_build.restype = vp
        lib.gen_rgg_sizes.argtypes = [vp, vp, vp]
        lib.gen_rgg_fetch.argtypes = [vp, vp, vp, vp]
        lib.gen_rgg_free.argtypes = [vp]
        _lib = lib
    return _lib


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


@dataclass
class Problem:
    """L (graph-Laplacian part, with diagonal) + optional d; A = L + diag(d)."""
    name: str
    rp: np.ndarray            # int64[n+1]
    ci: np.ndarray            # int32[nnz]
    val: np.ndarray           # float64[nnz]
    d: np.ndarray | None      # float64[n] or None (pure graph Laplacian, singular)
    params: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.rp.shape[0] - 1)

    @property
    def nnz(self) -> int:
        return int(self.ci.shape[0])


def rhs(n: int, seed: int = 0, offset: int = 0) -> np.ndarray:
    """b_i = 2*u(seed ^ (offset+i)) - 1, counter-based."""
    b = np.empty(n, dtype=np.float64)
    _L().gen_rhs(n, seed, offset, _p(b))
    return b


def grid2d(n: int) -> Problem:
    nnz = _L().gen_grid2d_nnz(n)
    rp = np.empty(n * n + 1, np.int64)
    ci = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float64)
    d = np.empty(n * n, np.float64)
    _L().gen_grid2d(n, _p(rp), _p(ci), _p(val), _p(d))
    return Problem(f"grid2d_{n}", rp, ci, val, d)


def grid3d(n: int) -> Problem:
    nnz = _L().gen_grid3d_nnz(n)
    rp = np.empty(n ** 3 + 1, np.int64)
    ci = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float64)
    d = np.empty(n ** 3, np.float64)
    _L().gen_grid3d(n, _p(rp), _p(ci), _p(val), _p(d))
    return Problem(f"grid3d_{n}", rp, ci, val, d)


def rgg(N: int, seed: int = 0) -> Problem:
    lib = _L()
    h = lib.gen_rgg_build(N, seed)
    if not h:
        raise MemoryError("gen_rgg_build failed")
    n = ctypes.c_int64()
    nnz = ctypes.c_int64()
    lib.gen_rgg_sizes(h, ctypes.byref(n), ctypes.byref(nnz))
    rp = np.empty(n.value + 1, np.int64)
    ci = np.empty(nnz.value, np.int32)
    val = np.empty(nnz.value, np.float64)
    lib.gen_rgg_fetch(h, _p(rp), _p(ci), _p(val))
    lib.gen_rgg_free(h)
    return Problem(f"rgg_{N}", rp, ci, val, None)


def from_edges(n: int, edges, weights=None, d=None, name="graph") -> Problem:
    """Weighted graph Laplacian from an undirected edge list (test helper)."""
    edges = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    w = np.ones(len(edges)) if weights is None else np.asarray(weights, dtype=np.float64)
    rows = np.concatenate([edges[:, 0], edges[:, 1], np.arange(n)])
    cols = np.concatenate([edges[:, 1], edges[:, 0], np.arange(n)])
    deg = np.zeros(n)
    np.add.at(deg, edges[:, 0], w)
    np.add.at(deg, edges[:, 1], w)
    vals = np.concatenate([-w, -w, deg])
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    rp = np.cumsum(rp)
    return Problem(name, rp, cols.astype(np.int32), vals.astype(np.float64),
                   None if d is None else np.asarray(d, dtype=np.float64))


def random_graph(n: int, avg_deg: float, seed: int, weighted: bool = False, dirichlet: bool = True,
                 connected: bool = True) -> Problem:
    """Seeded random graph (a spanning path plus random chords) for small parity cases."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n)
    e = [(int(perm[k]), int(perm[k + 1])) for k in range(n - 1)] if connected else []
    m_extra = max(0, int(n * avg_deg / 2) - len(e))
    a = rng.integers(0, n, m_extra)
    b = rng.integers(0, n, m_extra)
    e += [(int(x), int(y)) for x, y in zip(a, b) if x != y]
    e = sorted({(min(x, y), max(x, y)) for x, y in e})
    w = rng.uniform(0.5, 2.0, len(e)) if weighted else None
    d = None
    if dirichlet:
        d = np.zeros(n)
        idx = rng.choice(n, max(1, n // 10), replace=False)
        d[idx] = rng.uniform(0.5, 1.5, len(idx)) if weighted else 1.0
    return from_edges(n, e, w, d, name=f"rand_{n}_{seed}")


# BASELINE.json configs.  coarsest_size follows the paper's
# "< 100" except C2, which BASELINE.json caps at 1000.
CONFIGS = {
    "C1": dict(kind="grid2d", size=64, passes=2, degree=2, k_inner=2, coarsest_size=100, tol=1e-8, seed=0),
    "C2": dict(kind="grid2d", size=512, passes=3, degree=3, k_inner=2, coarsest_size=1000, tol=1e-8, seed=0),
    "C3": dict(kind="grid2d", size=4096, passes=4, degree=4, k_inner=2, coarsest_size=100, tol=1e-8, seed=0),
    "C4": dict(kind="grid3d", size=256, passes=3, degree=3, k_inner=2, coarsest_size=100, tol=1e-8, seed=0),
    "C5": dict(kind="rgg", size=8_000_000, passes=4, degree=4, k_inner=2, coarsest_size=100, tol=1e-8, seed=0),
}


def problem(cfg, size: int | None = None) -> Problem:
    """Build the matrix of a config (name or dict); `size` overrides the grid/point size."""
    c = dict(CONFIGS[cfg]) if isinstance(cfg, str) else dict(cfg)
    s = c["size"] if size is None else size
    if c["kind"] == "grid2d":
        p = grid2d(s)
    elif c["kind"] == "grid3d":
        p = grid3d(s)
    elif c["kind"] == "rgg":
        p = rgg(s, c.get("seed", 0))
    else:
        raise ValueError(c["kind"])
    c["size"] = s
    p.params = c
    return p
