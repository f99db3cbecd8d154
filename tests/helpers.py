"""Independent dense references for the oracle pins (numpy/scipy only; no oracle code).

Everything here is written from the mathematics, not from oracle/amg_oracle.c:
dense matrices, an independent Remez exchange for the best uniform polynomial
approximation to 1/x (Eq. (1x-1-min), l.149-151), the Chebyshev closed
form of its error polynomial, dense two-level/multilevel
operators and a dense PCG.
"""
from __future__ import annotations

import numpy as np
import numpy.polynomial.chebyshev as C


def dense(rp, ci, v, n=None):
    n = len(rp) - 1 if n is None else n
    A = np.zeros((n, n))
    for i in range(n):
        for p in range(rp[i], rp[i + 1]):
            A[i, ci[p]] += v[p]
    return A


def A0_dense(prob):
    A = dense(prob.rp, prob.ci, prob.val)
    if prob.d is not None:
        A = A + np.diag(prob.d)
    return A


def P_dense(agg, nc):
    P = np.zeros((len(agg), nc))
    P[np.arange(len(agg)), agg] = 1.0
    return P


# ---------------------------------------------------------------- Remez
def remez_inv(a: float, b: float, m: int, iters: int = 60):
    """Best uniform approximation p (degree m) to 1/x on [a, b] by Remez exchange.

    Returns a numpy Polynomial-like callable in the mapped Chebyshev basis and the
    levelled error E (max |1/x - p|)."""
    # work in t in [-1, 1], x = (a+b)/2 + (b-a)/2 t
    xt = lambda t: 0.5 * (a + b) + 0.5 * (b - a) * t
    k = np.arange(m + 2)
    ref = -np.cos(np.pi * k / (m + 1))
    coef = None
    E = 0.0
    grid = np.cos(np.linspace(0, np.pi, 20001))[::-1]
    for _ in range(iters):
        M = np.zeros((m + 2, m + 2))
        for j in range(m + 1):
            M[:, j] = C.chebval(ref, np.eye(m + 1)[j])
        M[:, m + 1] = (-1.0) ** k
        sol = np.linalg.solve(M, 1.0 / xt(ref))
        coef, E = sol[: m + 1], sol[m + 1]
        err = 1.0 / xt(grid) - C.chebval(grid, coef)
        # new reference: extrema of err on each sign-constant run
        s = np.sign(err)
        idx = []
        start = 0
        for i in range(1, len(grid) + 1):
            if i == len(grid) or s[i] != s[start]:
                seg = np.arange(start, i)
                idx.append(seg[np.argmax(np.abs(err[seg]))])
                start = i
        if len(idx) < m + 2:
            break
        idx = np.array(idx)
        # keep m+2 consecutive alternants containing the global max
        if len(idx) > m + 2:
            g = np.argmax(np.abs(err[idx]))
            lo = min(max(0, g - (m + 1)), len(idx) - (m + 2))
            best = max(range(lo, min(g, len(idx) - (m + 2)) + 1), key=lambda s0: np.min(np.abs(err[idx[s0:s0 + m + 2]])))
            idx = idx[best:best + m + 2]
        newref = grid[idx]
        if np.allclose(newref, ref, atol=1e-15, rtol=0):
            break
        ref = newref

    def q(x):
        x = np.asarray(x, dtype=np.float64)
        return C.chebval((2.0 * x - (a + b)) / (b - a), coef)

    return q, abs(E)


def cheb_closed_form_r(x, l0, l1, m):
    """r_{m+1}(x) = P_{m+1}(s(x)) / P_{m+1}(a), P_j = T_j - 2 d T_{j-1} + d^2 T_{j-2}."""
    kappa = l1 / l0
    d = (np.sqrt(kappa) - 1) / (np.sqrt(kappa) + 1)
    a = (kappa + 1) / (kappa - 1)
    s = (l1 + l0 - 2 * np.asarray(x)) / (l1 - l0)

    def T(j, t):
        return C.chebval(t, np.eye(abs(j) + 1)[abs(j)])

    def P(j, t):
        return T(j, t) - 2 * d * T(j - 1, t) + d * d * T(j - 2, t)

    return P(m + 1, s) / P(m + 1, a)


def q_closed_form(l0, l1, m):
    """q_m(x) = (1 - r_{m+1}(x))/x as an explicit degree-m polynomial (fitted exactly on
    Chebyshev nodes of [l0, l1]) so it can be evaluated at x ~ 0 without cancellation."""
    t = np.cos(np.pi * (np.arange(4 * m + 8) + 0.5) / (4 * m + 8))
    x = 0.5 * (l0 + l1) + 0.5 * (l1 - l0) * t
    coef = C.chebfit(t, (1 - cheb_closed_form_r(x, l0, l1, m)) / x, m)
    return lambda w: C.chebval((2.0 * np.asarray(w) - (l0 + l1)) / (l1 - l0), coef)


def matfun_sym(A, f):
    w, V = np.linalg.eigh(A)
    return (V * f(w)) @ V.T


def pinv_sym(A, tol=1e-10):
    w, V = np.linalg.eigh(A)
    inv = np.where(np.abs(w) > tol * max(1.0, np.abs(w).max()), 1.0 / np.where(w == 0, 1, w), 0.0)
    return (V * inv) @ V.T


def two_level_B(A, P, R, AH_inv):
    """B = Rbar + (I - R A) P A_H^+ P^T (I - A R), Rbar = 2R - R A R."""
    n = A.shape[0]
    I = np.eye(n)
    Rbar = 2 * R - R @ A @ R
    return Rbar + (I - R @ A) @ P @ AH_inv @ P.T @ (I - A @ R)


def pcg(A, b, Bop, tol, maxit):
    x = np.zeros_like(b)
    r = b.copy()
    z = Bop(r)
    d = z.copy()
    rz = r @ z
    bn = np.linalg.norm(b)
    xs = [x.copy()]
    for k in range(maxit):
        if np.linalg.norm(r) <= tol * bn:
            return x, k, xs
        q = A @ d
        alpha = rz / (d @ q)
        x = x + alpha * d
        r = r - alpha * q
        xs.append(x.copy())
        z = Bop(r)
        rz_new = r @ z
        d = z + (rz_new / rz) * d
        rz = rz_new
    return x, maxit, xs


def splitmix64(z: int) -> int:
    """SplitMix64 output for state z (docs/keys.md), written independently for the tests."""
    M = (1 << 64) - 1
    z = (int(z) + 0x9E3779B97F4A7C15) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def edge_key(w, a, b, seed, level, pas):
    seed, level, pas, a, b = int(seed), int(level), int(pas), int(a), int(b)
    salt = splitmix64(seed ^ ((level << 8) ^ pas))
    lo, hi = min(a, b), max(a, b)
    h = splitmix64(((lo << 32) | hi) ^ salt)
    return (int(w), h, lo, hi)


def fcg_restarted(A, b, Bop, tol, maxit, restart, x0=None, anorm_stop=None):
    """Flexible CG with a window of at most `restart` stored directions (PAPER.md l.322-323:
    "restart ... every five iterations"), written from the method's definition:
    every new direction is B(r) made A-orthogonal to the directions of the current window; after
    `restart` directions the window is emptied (x and r kept).  Returns the list of iterates
    x_0, x_1, ... and the iteration count at the stop.  anorm_stop = (x*, ) switches to the paper's
    relative A-norm error test ||x_k - x*||_A <= tol ||x_0 - x*||_A, evaluated densely."""
    x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=float)
    r = b - A @ x
    bn = np.linalg.norm(b)
    win = []  # (d, Ad, d.Ad)
    xs = [x.copy()]

    def aerr(v):
        e = v - anorm_stop
        return np.sqrt(max(e @ (A @ e), 0.0))

    e0 = aerr(x) if anorm_stop is not None else None
    for k in range(maxit + 1):
        done = aerr(x) <= tol * e0 if anorm_stop is not None else np.linalg.norm(r) <= tol * bn
        if done or k == maxit:
            return xs, k
        z = Bop(r)
        d = z - sum(((z @ Ad) / dAd) * dj for dj, Ad, dAd in win) if win else z.copy()
        q = A @ d
        dq = d @ q
        a = (d @ r) / dq
        x = x + a * d
        r = r - a * q
        xs.append(x.copy())
        win.append((d, q, dq))
        if len(win) == restart:
            win = []
    return xs, maxit


def assert_close(got, ref, tol, what=""):
    """Parity bar, element by element and in norm: max_i |got_i - ref_i| <= tol * max_i |ref_i| and
    ||got - ref||_2 <= tol ||ref||_2 (a handful of wrong rows cannot hide inside the 2-norm)."""
    got = np.asarray(got)
    ref = np.asarray(ref)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    assert np.all(np.isfinite(got)), f"{what}: non-finite entries"
    d = np.abs(got - ref)
    scale = np.max(np.abs(ref)) if ref.size else 0.0
    imax = int(np.argmax(d)) if d.size else 0
    assert (d.max() if d.size else 0.0) <= tol * scale, \
        f"{what}: max elementwise error {d.max():.3e} at {imax} > {tol:g} * max|ref| = {tol * scale:.3e}"
    assert np.linalg.norm(got - ref) <= tol * np.linalg.norm(ref), f"{what}: 2-norm error"
