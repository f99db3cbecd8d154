"""ctypes binding of the plain-C CPU oracle (oracle/amg_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product package
(paper_1307_6305_b200) never imports this module.  Every routine is documented,
with its PAPER.md / SURVEY.md citation, in amg_oracle.c.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

i64, i32, u64, dbl, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p

ORC_OK, ORC_NOT_CONVERGED = 0, 1


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "amg_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-D_DEFAULT_SOURCE", "-ffp-contract=off", "-fPIC",
                               "-shared", "-o", LIB_PATH, src, "-lm"])
    return LIB_PATH


def _L():
    global _lib
    if _lib is not None:
        return _lib
    build()
    L = ctypes.CDLL(LIB_PATH)
    sig = {
        "orc_Em": (dbl, [i32, dbl]),
        "orc_kappa_rule": (dbl, [i32]),
        "orc_poly_coeffs": (None, [dbl, dbl, i32, vp, vp]),
        "orc_setup": (i32, [i64, vp, vp, vp, vp, i32, i32, i64, dbl, i32, i32, u64, i32, i64, i32, i32, vp]),
        "orc_free": (None, [vp]),
        "orc_solve": (i32, [vp, vp, vp, dbl, i32, vp, vp, vp]),
        "orc_num_levels": (i32, [vp]),
        "orc_set_amli_kappa": (None, [vp, dbl]),
        "orc_set_lanczos": (None, [i32]),
        "orc_set_mis_k": (None, [i32]),
        "orc_set_xstar": (None, [vp]),
        "orc_mis_aggregate_csr": (i64, [i64, vp, vp, i32, u64, i32, vp, vp]),
        "orc_lanczos_max": (dbl, [i64, vp, vp, vp, i32, u64, i32]),
        "orc_is_singular": (i32, [vp]),
        "orc_level_info": (None, [vp, i32, vp, vp, vp, vp, vp, vp]),
        "orc_level_csr": (None, [vp, i32, vp, vp, vp]),
        "orc_level_agg": (None, [vp, i32, vp]),
        "orc_level_coeffs": (None, [vp, i32, vp, vp]),
        "orc_level_rounds": (None, [vp, i32, vp, i32]),
        "orc_level_smooth": (None, [vp, i32, vp, vp, vp]),
        "orc_level_precond": (None, [vp, i32, i32, vp, vp]),
        "orc_coarse_solve": (None, [vp, vp, vp]),
        "orc_inf_norm": (dbl, [i64, vp, vp, vp]),
        "orc_spmv": (None, [i64, vp, vp, vp, vp, vp]),
        "orc_smooth": (None, [i64, vp, vp, vp, i32, vp, vp, vp, vp, vp]),
        "orc_match": (i32, [i64, vp, vp, vp, u64, i32, i32, i32, vp]),
        "orc_aggregate_pass": (i64, [i64, vp, vp, vp, u64, i32, i32, i32, vp]),
        "orc_edge_hash": (u64, [u64, i32, i32, i64, i64]),
        "orc_quotient": (vp, [i64, vp, vp, vp, vp, vp, i64, i32]),
        "orc_csr_sizes": (None, [vp, vp, vp]),
        "orc_csr_fetch": (None, [vp, vp, vp, vp, vp]),
        "orc_csr_free": (None, [vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _p(a):
    return None if a is None else a.ctypes.data


def _c(a, dt):
    return None if a is None else np.ascontiguousarray(a, dtype=dt)


# ------------------------------------------------------------------ scalars
def Em(m: int, kappa: float) -> float:
    return _L().orc_Em(m, kappa)


def kappa_rule(m: int) -> float:
    return _L().orc_kappa_rule(m)


def poly_coeffs(lambda1: float, kappa: float, m: int):
    a = np.empty(m + 1)
    b = np.empty(m + 1)
    _L().orc_poly_coeffs(lambda1, kappa, m, _p(a), _p(b))
    return a, b


# ------------------------------------------------------------------ CSR pieces
def inf_norm(rp, ci, v) -> float:
    rp, ci, v = _c(rp, np.int64), _c(ci, np.int32), _c(v, np.float64)
    return _L().orc_inf_norm(len(rp) - 1, _p(rp), _p(ci), _p(v))


def spmv(rp, ci, v, x):
    rp, ci, v, x = _c(rp, np.int64), _c(ci, np.int32), _c(v, np.float64), _c(x, np.float64)
    y = np.empty(len(rp) - 1)
    _L().orc_spmv(len(rp) - 1, _p(rp), _p(ci), _p(v), _p(x), _p(y))
    return y


def smooth(rp, ci, v, m, alpha, beta, f, x0):
    rp, ci, v = _c(rp, np.int64), _c(ci, np.int32), _c(v, np.float64)
    alpha, beta, f, x0 = (_c(a, np.float64) for a in (alpha, beta, f, x0))
    x = np.empty(len(rp) - 1)
    _L().orc_smooth(len(rp) - 1, _p(rp), _p(ci), _p(v), m, _p(alpha), _p(beta), _p(f), _p(x0), _p(x))
    return x


def match(rp, ci, w, seed=0, level=0, pass_=0, rule=0):
    rp, ci, w = _c(rp, np.int64), _c(ci, np.int32), _c(w, np.int64)
    mate = np.empty(len(rp) - 1, np.int32)
    rounds = _L().orc_match(len(rp) - 1, _p(rp), _p(ci), _p(w), seed, level, pass_, rule, _p(mate))
    return mate, rounds


def aggregate_pass(rp, ci, w, seed=0, level=0, pass_=0, rule=0):
    rp, ci, w = _c(rp, np.int64), _c(ci, np.int32), _c(w, np.int64)
    agg = np.empty(len(rp) - 1, np.int32)
    nc = _L().orc_aggregate_pass(len(rp) - 1, _p(rp), _p(ci), _p(w), seed, level, pass_, rule, _p(agg))
    return agg, int(nc)


def mis_aggregate(rp, ci, k, seed=0, level=0):
    """MIS-k aggregation of a CSR pattern (reading A25); returns (agg, nc, roots)."""
    rp, ci = _c(rp, np.int64), _c(ci, np.int32)
    agg = np.empty(len(rp) - 1, np.int32)
    roots = np.zeros(len(rp) - 1, np.int8)
    nc = _L().orc_mis_aggregate_csr(len(rp) - 1, _p(rp), _p(ci), k, seed, level, _p(agg), _p(roots))
    return agg, int(nc), roots.astype(bool)


def lanczos_max(rp, ci, v, k, seed=0, level=0) -> float:
    """Largest Ritz value of k Lanczos steps from the counter-based start vector (reading A24)."""
    rp, ci, v = _c(rp, np.int64), _c(ci, np.int32), _c(v, np.float64)
    return _L().orc_lanczos_max(len(rp) - 1, _p(rp), _p(ci), _p(v), k, seed, level)


def edge_hash(seed, level, pass_, a, b) -> int:
    return int(_L().orc_edge_hash(seed, level, pass_, a, b))


def quotient(rp, ci, v, w, agg, nc, drop_diag):
    rp, ci = _c(rp, np.int64), _c(ci, np.int32)
    v, w, agg = _c(v, np.float64), _c(w, np.int64), _c(agg, np.int32)
    L = _L()
    H = L.orc_quotient(len(rp) - 1, _p(rp), _p(ci), _p(v), _p(w), _p(agg), nc, int(drop_diag))
    n, nnz = i64(), i64()
    L.orc_csr_sizes(H, ctypes.byref(n), ctypes.byref(nnz))
    orp = np.empty(n.value + 1, np.int64)
    oci = np.empty(nnz.value, np.int32)
    ov = np.empty(nnz.value) if v is not None else None
    ow = np.empty(nnz.value, np.int64) if w is not None else None
    L.orc_csr_fetch(H, _p(orp), _p(oci), _p(ov), _p(ow))
    L.orc_csr_free(H)
    return orp, oci, (ov if v is not None else ow)


# ------------------------------------------------------------------ hierarchy
class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle status {code}")
        self.code = code


class Hierarchy:
    """Oracle setup + solve (O5-O8)."""

    def __init__(self, rp, ci, val, d, passes, degree, coarsest_size=100, kappa=0.0, restart=5,
                 max_iter=500, seed=0, nparts=1, gather_rows=0, rule=0, cycle=0, amli_kappa=0.0, lanczos=0,
                 mis_k=0):
        self._keep = [_c(rp, np.int64), _c(ci, np.int32), _c(val, np.float64), _c(d, np.float64)]
        rp, ci, val, d = self._keep
        self.m = degree
        self.passes = passes
        h = vp()
        _L().orc_set_lanczos(int(lanczos))
        _L().orc_set_mis_k(int(mis_k))
        st = _L().orc_setup(len(rp) - 1, _p(rp), _p(ci), _p(val), _p(d), passes, degree, coarsest_size, kappa,
                            restart, max_iter, seed, nparts, gather_rows, rule, cycle, ctypes.byref(h))
        self._keep = None
        _L().orc_set_lanczos(0)
        _L().orc_set_mis_k(0)
        if st != 0:
            raise OracleError(st)
        self.h = h
        if amli_kappa:
            _L().orc_set_amli_kappa(h, amli_kappa)

    def __del__(self):
        if getattr(self, "h", None):
            _L().orc_free(self.h)
            self.h = None

    @property
    def nlev(self) -> int:
        return _L().orc_num_levels(self.h)

    @property
    def singular(self) -> bool:
        return bool(_L().orc_is_singular(self.h))

    def level_info(self, l: int) -> dict:
        n, nnz, l1, k, nc, npart = i64(), i64(), dbl(), dbl(), i64(), i32()
        _L().orc_level_info(self.h, l, *(ctypes.byref(x) for x in (n, nnz, l1, k, nc, npart)))
        return dict(n=n.value, nnz=nnz.value, lambda1=l1.value, kappa=k.value, nc=nc.value, nparts=npart.value)

    def level_csr(self, l: int):
        info = self.level_info(l)
        rp = np.empty(info["n"] + 1, np.int64)
        ci = np.empty(info["nnz"], np.int32)
        v = np.empty(info["nnz"])
        _L().orc_level_csr(self.h, l, _p(rp), _p(ci), _p(v))
        return rp, ci, v

    def level_agg(self, l: int) -> np.ndarray:
        a = np.empty(self.level_info(l)["n"], np.int32)
        _L().orc_level_agg(self.h, l, _p(a))
        return a

    def level_coeffs(self, l: int):
        a = np.empty(self.m + 1)
        b = np.empty(self.m + 1)
        _L().orc_level_coeffs(self.h, l, _p(a), _p(b))
        return a, b

    def level_rounds(self, l: int):
        r = np.zeros(self.passes, np.int32)
        _L().orc_level_rounds(self.h, l, _p(r), self.passes)
        return r

    def smooth(self, l: int, f, x0):
        f, x0 = _c(f, np.float64), _c(x0, np.float64)
        x = np.empty_like(f)
        _L().orc_level_smooth(self.h, l, _p(f), _p(x0), _p(x))
        return x

    def precond(self, r, nu: int = 2, level: int = 0):
        r = _c(r, np.float64)
        z = np.empty_like(r)
        _L().orc_level_precond(self.h, level, nu, _p(r), _p(z))
        return z

    def coarse_solve(self, r):
        r = _c(r, np.float64)
        e = np.empty_like(r)
        _L().orc_coarse_solve(self.h, _p(r), _p(e))
        return e

    def solve(self, b, x0=None, tol=1e-8, nu=2, xstar=None):
        """xstar given: stop on the paper's relative A-norm error reduction."""
        b = _c(b, np.float64)
        x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64)
        it, rr, trr = i32(), dbl(), dbl()
        xs = _c(xstar, np.float64)
        _L().orc_set_xstar(_p(xs))
        try:
            st = _L().orc_solve(self.h, _p(b), _p(x), tol, nu, ctypes.byref(it), ctypes.byref(rr), ctypes.byref(trr))
        finally:
            _L().orc_set_xstar(None)
        return dict(status=st, x=x, iters=it.value, relres=rr.value, true_relres=trr.value)

    def complexities(self):
        infos = [self.level_info(l) for l in range(self.nlev)]
        return (sum(i["n"] for i in infos) / infos[0]["n"], sum(i["nnz"] for i in infos) / infos[0]["nnz"])


def setup_problem(prob, **over) -> Hierarchy:
    """Oracle hierarchy for an inputs.gen.Problem with its config's parameters."""
    p = dict(prob.params)
    p.update(over)
    kw = {k: p[k] for k in ("coarsest_size", "kappa", "restart", "max_iter", "seed", "nparts", "gather_rows",
                            "rule", "cycle", "amli_kappa", "lanczos", "mis_k") if k in p}
    return Hierarchy(prob.rp, prob.ci, prob.val, prob.d, p["passes"], p["degree"], **kw)
