"""Thin ctypes binding of libamg_b200.so (C ABI: include/amg.h).  Argument marshalling only.

Every array may be a torch tensor (CUDA or CPU) or a numpy array; the library itself detects host
vs device pointers and does all copies and all computation in its sm_100a kernels.  There is no
CPU or PyTorch fallback: if the shared library is missing this module raises on first use.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# AMG_B200_LIB overrides the in-tree library (A/B timing of another build of the same ABI)
LIB_PATH = os.environ.get("AMG_B200_LIB") or os.path.join(_HERE, "lib", "libamg_b200.so")

AMG_OK, AMG_NOT_CONVERGED = 0, 1
AMG_E_ARG, AMG_E_INPUT, AMG_E_CUDA, AMG_E_NCCL, AMG_E_OOM, AMG_E_BREAKDOWN, AMG_E_SETUP = -1, -2, -3, -4, -5, -6, -7
EXPORTS = ("amg_options_default", "amg_setup", "amg_solve", "amg_free", "amg_get_info", "amg_last_error",
           "amg_level_sizes", "amg_level_export", "amg_level_smooth", "amg_level_precond", "amg_coarse_solve",
           "amg_comm_unique_id", "amg_comm_init_nccl", "amg_comm_init_threads", "amg_comm_rank", "amg_comm_free",
           "amg_setup_dist", "amg_level_dist", "amg_halo_plan")
AMG_COMM_ID_BYTES = 128


class amg_options(ctypes.Structure):
    _fields_ = [("coarsest_size", ctypes.c_int64), ("kappa", ctypes.c_double), ("restart", ctypes.c_int32),
                ("max_iter", ctypes.c_int32), ("seed", ctypes.c_uint64), ("stream", ctypes.c_void_p),
                ("use_graphs", ctypes.c_int32), ("compress", ctypes.c_int32), ("tail_nnz", ctypes.c_int64),
                ("gather_rows", ctypes.c_int64), ("tail_smem", ctypes.c_int32), ("cycle", ctypes.c_int32),
                ("amli_kappa", ctypes.c_double), ("lanczos_steps", ctypes.c_int32), ("mis_k", ctypes.c_int32),
                ("dense_b_rows", ctypes.c_int32), ("global_agg", ctypes.c_int32)]


class amg_info(ctypes.Structure):
    _fields_ = [("levels", ctypes.c_int32), ("poly_degree", ctypes.c_int32), ("n_match_passes", ctypes.c_int32),
                ("singular", ctypes.c_int32), ("n", ctypes.c_int64 * 32), ("nnz", ctypes.c_int64 * 32),
                ("lambda1", ctypes.c_double * 32), ("kappa", ctypes.c_double * 32),
                ("grid_complexity", ctypes.c_double), ("operator_complexity", ctypes.c_double),
                ("setup_ms", ctypes.c_double), ("solve_ms", ctypes.c_double), ("last_iters", ctypes.c_int32),
                ("reserved0", ctypes.c_int32), ("last_relres", ctypes.c_double),
                ("last_true_relres", ctypes.c_double), ("launches_last_solve", ctypes.c_int64),
                ("launches_per_iter", ctypes.c_int64), ("launches_last_setup", ctypes.c_int64),
                ("device_bytes", ctypes.c_int64), ("prof_smoother_ms", ctypes.c_double),
                ("prof_smoother_launches", ctypes.c_int64), ("prof_smoother_bytes", ctypes.c_int64),
                ("level0_format", ctypes.c_int32), ("nranks", ctypes.c_int32), ("dist_levels", ctypes.c_int32),
                ("level0_path", ctypes.c_int32)]


class AmgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_lib = None


def load():
    """Load the in-tree shared library (fails loudly if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    L.amg_options_default.argtypes = [ctypes.POINTER(amg_options)]
    L.amg_setup.argtypes = [ctypes.POINTER(vp), i64, vp, vp, vp, vp, i32, i32, ctypes.POINTER(amg_options)]
    L.amg_solve.argtypes = [vp, vp, vp, dbl, i32, ctypes.POINTER(i32), ctypes.POINTER(dbl)]
    L.amg_free.argtypes = [vp]
    L.amg_get_info.argtypes = [vp, ctypes.POINTER(amg_info)]
    L.amg_last_error.restype = ctypes.c_char_p
    L.amg_level_sizes.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, vp]
    L.amg_level_export.argtypes = [vp, i32, vp, vp, vp, vp]
    L.amg_level_smooth.argtypes = [vp, i32, vp, vp, vp]
    L.amg_level_precond.argtypes = [vp, i32, i32, vp, vp]
    L.amg_coarse_solve.argtypes = [vp, vp, vp]
    L.amg_comm_unique_id.argtypes = [vp]
    L.amg_comm_init_nccl.argtypes = [ctypes.POINTER(vp), vp, i32, i32]
    L.amg_comm_init_threads.argtypes = [vp, i32]
    L.amg_comm_rank.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(i32)]
    L.amg_comm_free.argtypes = [vp]
    L.amg_setup_dist.argtypes = [ctypes.POINTER(vp), vp, i64, i64, i64, vp, vp, vp, vp, i32, i32,
                                 ctypes.POINTER(amg_options)]
    L.amg_level_dist.argtypes = [vp, i32, vp, vp, vp]
    L.amg_halo_plan.argtypes = [i64, i32, vp, i32, i32, vp, i32, vp, vp, vp, vp, vp]
    for name in EXPORTS:
        if name not in ("amg_last_error",):
            getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def _ptr(a, dtype):
    """Raw pointer of a contiguous torch tensor / numpy array with the expected element type."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):  # torch.Tensor
        import torch

        want = {np.int64: torch.int64, np.int32: torch.int32, np.float64: torch.float64}[dtype]
        if a.dtype != want or not a.is_contiguous():
            raise TypeError(f"expected contiguous {want}, got {a.dtype}")
        return a.data_ptr()
    if not isinstance(a, np.ndarray) or a.dtype != dtype or not a.flags["C_CONTIGUOUS"]:
        raise TypeError(f"expected a C-contiguous numpy array of {np.dtype(dtype)}")
    return a.ctypes.data


def _len(a):
    if a is None:
        return None
    return int(a.numel()) if hasattr(a, "numel") else int(a.shape[0])


def _last(a) -> int:
    v = a[-1]
    return int(v.item() if hasattr(v, "item") else v)


def _check_csr(row_ptr, col, val, d, n):
    """Lengths only (the library validates the contents): col and val hold row_ptr[n] entries, d has
    n; a shorter buffer would otherwise be read past its end by the staging copies."""
    if n < 1:
        raise ValueError("row_ptr must have at least 2 entries")
    nnz = _last(row_ptr)
    if _len(col) != nnz or _len(val) != nnz:
        raise ValueError(f"col/val must have row_ptr[-1] = {nnz} entries, got {_len(col)}/{_len(val)}")
    if d is not None and _len(d) != n:
        raise ValueError(f"d must have n = {n} entries, got {_len(d)}")


def _check_vec(h, **vecs):
    n = getattr(h, "n_local", None)
    for k, v in vecs.items():
        if n is not None and v is not None and _len(v) != n:
            raise ValueError(f"{k} must have n = {n} entries (this handle's rows), got {_len(v)}")


def _check(st: int, what: str):
    if st not in (AMG_OK, AMG_NOT_CONVERGED):
        raise AmgError(st, f"{what}: {amg_last_error()}")
    return st


def amg_last_error() -> str:
    return load().amg_last_error().decode()


def amg_options_default(**over) -> amg_options:
    o = amg_options()
    load().amg_options_default(ctypes.byref(o))
    for k, v in over.items():
        setattr(o, k, v)
    return o


def amg_setup(row_ptr, col, val, d, n_match_passes: int, poly_degree: int, opts: amg_options | None = None):
    """Build the hierarchy; returns an opaque handle (ctypes.c_void_p)."""
    h = ctypes.c_void_p()
    n = (row_ptr.shape[0] if hasattr(row_ptr, "shape") else len(row_ptr)) - 1
    _check_csr(row_ptr, col, val, d, n)
    st = load().amg_setup(ctypes.byref(h), n, _ptr(row_ptr, np.int64), _ptr(col, np.int32), _ptr(val, np.float64),
                          _ptr(d, np.float64), n_match_passes, poly_degree,
                          ctypes.byref(opts) if opts is not None else None)
    _check(st, "amg_setup")
    h.n_local = n
    return h


def amg_solve(h, b, x, tol: float, k_inner: int):
    """Solve A x = b in place of x; returns (status, iters, relres)."""
    _check_vec(h, b=b, x=x)
    it = ctypes.c_int32()
    rr = ctypes.c_double()
    st = load().amg_solve(h, _ptr(b, np.float64), _ptr(x, np.float64), tol, k_inner, ctypes.byref(it),
                          ctypes.byref(rr))
    _check(st, "amg_solve")
    return st, it.value, rr.value


def amg_free(h):
    if h is not None and h.value:
        load().amg_free(h)
        h.value = None


def amg_get_info(h) -> dict:
    inf = amg_info()
    _check(load().amg_get_info(h, ctypes.byref(inf)), "amg_get_info")
    L = inf.levels
    return dict(levels=L, poly_degree=inf.poly_degree, n_match_passes=inf.n_match_passes, singular=bool(inf.singular),
                n=list(inf.n[:L]), nnz=list(inf.nnz[:L]), lambda1=list(inf.lambda1[:L]), kappa=list(inf.kappa[:L]),
                grid_complexity=inf.grid_complexity, operator_complexity=inf.operator_complexity,
                setup_ms=inf.setup_ms, solve_ms=inf.solve_ms, last_iters=inf.last_iters,
                last_relres=inf.last_relres, last_true_relres=inf.last_true_relres,
                launches_last_solve=inf.launches_last_solve, launches_per_iter=inf.launches_per_iter,
                launches_last_setup=inf.launches_last_setup, device_bytes=inf.device_bytes,
                prof_smoother_ms=inf.prof_smoother_ms, prof_smoother_launches=inf.prof_smoother_launches,
                prof_smoother_bytes=inf.prof_smoother_bytes, level0_format=inf.level0_format, nranks=inf.nranks,
                dist_levels=inf.dist_levels, level0_path=inf.level0_path)


# ---------------------------------------------------------------- parity hooks (test-only)
def amg_level_sizes(h, level: int, m: int):
    n, nnz, nc = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    l1, k = ctypes.c_double(), ctypes.c_double()
    a = np.empty(m + 1)
    b = np.empty(m + 1)
    _check(load().amg_level_sizes(h, level, ctypes.byref(n), ctypes.byref(nnz), ctypes.byref(nc), ctypes.byref(l1),
                                  ctypes.byref(k), a.ctypes.data, b.ctypes.data), "amg_level_sizes")
    return dict(n=n.value, nnz=nnz.value, nc=nc.value, lambda1=l1.value, kappa=k.value, alpha=a, beta=b)


def amg_level_export(h, level: int, m: int, with_agg: bool = True):
    s = amg_level_sizes(h, level, m)
    rp = np.empty(s["n"] + 1, np.int64)
    ci = np.empty(s["nnz"], np.int32)
    v = np.empty(s["nnz"], np.float64)
    last = level == amg_get_info(h)["levels"] - 1
    agg = np.empty(s["n"], np.int32) if (with_agg and not last) else None
    _check(load().amg_level_export(h, level, rp.ctypes.data, ci.ctypes.data, v.ctypes.data,
                                   agg.ctypes.data if agg is not None else None), "amg_level_export")
    return rp, ci, v, agg


def amg_level_smooth(h, level: int, f, x0, x):
    _check(load().amg_level_smooth(h, level, _ptr(f, np.float64), _ptr(x0, np.float64), _ptr(x, np.float64)),
           "amg_level_smooth")


def amg_level_precond(h, level: int, k_inner: int, r, z):
    _check(load().amg_level_precond(h, level, k_inner, _ptr(r, np.float64), _ptr(z, np.float64)), "amg_level_precond")


def amg_coarse_solve(h, r, e):
    _check(load().amg_coarse_solve(h, _ptr(r, np.float64), _ptr(e, np.float64)), "amg_coarse_solve")


# ---------------------------------------------------------------- row-partitioned path (multi-GPU)
def amg_comm_unique_id() -> bytes:
    """NCCL unique id (rank 0), to be sent to the other ranks (e.g. torch.distributed.broadcast)."""
    buf = (ctypes.c_uint8 * AMG_COMM_ID_BYTES)()
    _check(load().amg_comm_unique_id(ctypes.addressof(buf)), "amg_comm_unique_id")
    return bytes(buf)


def amg_comm_init_nccl(uid: bytes, nranks: int, rank: int):
    """NCCL communicator of this process over the current CUDA device (collective)."""
    if len(uid) != AMG_COMM_ID_BYTES:
        raise ValueError("unique id must be AMG_COMM_ID_BYTES bytes")
    c = ctypes.c_void_p()
    buf = (ctypes.c_uint8 * AMG_COMM_ID_BYTES).from_buffer_copy(uid)
    _check(load().amg_comm_init_nccl(ctypes.byref(c), ctypes.addressof(buf), nranks, rank), "amg_comm_init_nccl")
    return c


def amg_comm_init_threads(nranks: int):
    """nranks communicators for nranks host threads of this process on the current device (tests)."""
    arr = (ctypes.c_void_p * nranks)()
    _check(load().amg_comm_init_threads(ctypes.addressof(arr), nranks), "amg_comm_init_threads")
    return [ctypes.c_void_p(arr[r]) for r in range(nranks)]


def amg_comm_rank(c):
    r, n = ctypes.c_int32(), ctypes.c_int32()
    _check(load().amg_comm_rank(c, ctypes.byref(r), ctypes.byref(n)), "amg_comm_rank")
    return r.value, n.value


def amg_comm_free(c):
    if c is not None and c.value:
        load().amg_comm_free(c)
        c.value = None


def amg_setup_dist(comm, n_global: int, row_begin: int, row_ptr, col_global, val, d, n_match_passes: int,
                   poly_degree: int, opts: amg_options | None = None):
    """Collective setup of this rank's row block [row_begin, row_begin + n_local) (global column ids)."""
    h = ctypes.c_void_p()
    n_local = (row_ptr.shape[0] if hasattr(row_ptr, "shape") else len(row_ptr)) - 1
    _check_csr(row_ptr, col_global, val, d, n_local)
    st = load().amg_setup_dist(ctypes.byref(h), comm, n_global, row_begin, n_local, _ptr(row_ptr, np.int64),
                               _ptr(col_global, np.int32), _ptr(val, np.float64), _ptr(d, np.float64),
                               n_match_passes, poly_degree, ctypes.byref(opts) if opts is not None else None)
    _check(st, "amg_setup_dist")
    h.n_local = n_local
    return h


def amg_level_dist(h, level: int):
    dist, rb, ng = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
    _check(load().amg_level_dist(h, level, ctypes.byref(dist), ctypes.byref(rb), ctypes.byref(ng)),
           "amg_level_dist")
    return dict(dist=bool(dist.value), row_begin=rb.value, n_global=ng.value)


def amg_halo_plan(row_begin: int, n_local: int, offs, rank: int, halo_ids):
    """Host-only halo receive plan (no CUDA): list of (peer, relative offset, count) runs and n_lo."""
    offs = np.ascontiguousarray(offs, dtype=np.int64)
    ids = np.ascontiguousarray(halo_ids, dtype=np.int32)
    m = max(1, ids.shape[0])
    peer, off, cnt = (np.zeros(m, np.int32) for _ in range(3))
    nseg, nlo = ctypes.c_int32(), ctypes.c_int32()
    _check(load().amg_halo_plan(row_begin, n_local, offs.ctypes.data, offs.shape[0] - 1, rank, ids.ctypes.data,
                                ids.shape[0], peer.ctypes.data, off.ctypes.data, cnt.ctypes.data, ctypes.byref(nseg),
                                ctypes.byref(nlo)), "amg_halo_plan")
    k = nseg.value
    return [(int(peer[i]), int(off[i]), int(cnt[i])) for i in range(k)], nlo.value


class Solver:
    """Convenience owner of a handle: Solver(problem arrays...).solve(b, x)."""

    def __init__(self, row_ptr, col, val, d, n_match_passes, poly_degree, **opts):
        self.h = amg_setup(row_ptr, col, val, d, n_match_passes, poly_degree, amg_options_default(**opts))

    def solve(self, b, x, tol=1e-8, k_inner=2):
        return amg_solve(self.h, b, x, tol, k_inner)

    def info(self):
        return amg_get_info(self.h)

    def close(self):
        amg_free(self.h)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
