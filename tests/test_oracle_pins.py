"""-m "not gpu" pins of the CPU oracle against what the paper and the mathematics fix.

Each test names the passage it pins.  Nothing here reuses oracle code for the
expected value: closed forms are evaluated independently, dense references come
from tests/helpers.py (numpy), brute force enumerates small cases, and golden
values come from tests/golden/ (each file cites its source).
"""
import itertools
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import helpers as H

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def path_graph(gen, n, d=None):
    return gen.from_edges(n, [(i, i + 1) for i in range(n - 1)], d=d)


# ----------------------------------------------------------------- core sparse
def test_spmv_inf_norm_spec_examples(oracle_mod, gen_mod):
    g = gold("spec_examples.json")
    p = path_graph(gen_mod, 4)
    assert np.array_equal(oracle_mod.spmv(p.rp, p.ci, p.val, np.ones(4)), g["spmv_path4_ones"])
    assert np.array_equal(oracle_mod.spmv(p.rp, p.ci, p.val, np.arange(4.0)), g["spmv_path4_ramp"])
    assert oracle_mod.inf_norm(p.rp, p.ci, p.val) == g["inf_norm_path4"]
    q = gen_mod.grid2d(3)
    A = H.dense(q.rp, q.ci, q.val)
    assert oracle_mod.inf_norm(q.rp, q.ci, q.val) == np.abs(A).sum(1).max()
    # 5-pt Dirichlet operator (with d): still 8; 7-pt scaled by h: 12 h
    h0 = oracle_mod.Hierarchy(q.rp, q.ci, q.val, q.d, 1, 2, coarsest_size=100)
    assert h0.level_info(0)["lambda1"] == 8.0
    r = gen_mod.grid3d(3)
    h1 = oracle_mod.Hierarchy(r.rp, r.ci, r.val, r.d, 1, 2, coarsest_size=100)
    assert h1.level_info(0)["lambda1"] == pytest.approx(12.0 / 4.0, rel=1e-15)
    rng = np.random.default_rng(0)
    rg = gen_mod.random_graph(50, 4, seed=1, weighted=True)
    x = rng.standard_normal(50)
    assert np.allclose(oracle_mod.spmv(rg.rp, rg.ci, rg.val, x), H.dense(rg.rp, rg.ci, rg.val) @ x, rtol=1e-14)


# ----------------------------------------------------------------- E_m, kappa
def test_Em_closed_forms(oracle_mod):
    """P:167 (2 kappa delta^m / ((kappa-1)(a^2-1))) and P:177 (delta^m (kappa-1)/2) agree with the oracle."""
    for kappa in (2.0, 9.0, 10.0, 100.0):
        delta = (np.sqrt(kappa) - 1) / (np.sqrt(kappa) + 1)
        a = (kappa + 1) / (kappa - 1)
        for m in range(0, 8):
            e167 = 2 * kappa * delta ** m / ((kappa - 1) * (a * a - 1))
            e177 = delta ** m * (kappa - 1) / 2
            assert oracle_mod.Em(m, kappa) == pytest.approx(e167, rel=1e-13)
            assert oracle_mod.Em(m, kappa) == pytest.approx(e177, rel=1e-13)
    assert oracle_mod.Em(3, 9.0) == 0.5  # delta(9) = 1/2 exactly
    assert oracle_mod.Em(0, 10.0) == pytest.approx(4.5)


def test_golden_coefficients_and_kappa_rule(oracle_mod):
    g = gold("poly_coeffs.json")
    for row in g["rows"]:
        k = row["kappa"]
        a, b = oracle_mod.poly_coeffs(1.0, k, 4)
        assert b[0] == pytest.approx(row["beta0"], rel=1e-14)
        assert a[1] == pytest.approx(row["alpha1"], rel=1e-14)
        assert b[1] == pytest.approx(row["beta1"], rel=1e-14)
        assert a[2] == pytest.approx(row["alpha2"], rel=1e-14) and a[3] == a[2] and a[4] == a[2]
        assert b[2] == pytest.approx(row["beta2"], rel=1e-14) and b[4] == b[2]
        for m in (2, 3, 4):
            assert oracle_mod.Em(m, k) == pytest.approx(row[f"E{m}"], rel=1e-12)
        # beta scales as 1/lambda1
        a8, b8 = oracle_mod.poly_coeffs(8.0, k, 4)
        assert np.allclose(b8 * 8.0, b, rtol=1e-15) and np.array_equal(a8, a)
    assert oracle_mod.kappa_rule(1) == pytest.approx(g["kappa_star"]["1"], rel=1e-15)
    assert oracle_mod.kappa_rule(2) == pytest.approx(g["kappa_star"]["2"], rel=1e-15)
    for m in (3, 4, 5):
        assert oracle_mod.kappa_rule(m) == 10.0  # P:327 lambda0 = lambda1/10 whenever E_m(10) < 1
    # R1: E_m(kappa*) = 1/2 exactly for the rule's m
    assert oracle_mod.Em(2, oracle_mod.kappa_rule(2)) == pytest.approx(0.5, abs=1e-15)
    t = np.sqrt(oracle_mod.kappa_rule(2))
    assert t ** 3 - 3 * t ** 2 + 2 * t - 2 == pytest.approx(0.0, abs=1e-13)


# ----------------------------------------------------------------- smoother
def _diag_q(oracle_mod, xs, l1, kappa, m):
    n = len(xs)
    rp = np.arange(n + 1)
    ci = np.arange(n)
    a, b = oracle_mod.poly_coeffs(l1, kappa, m)
    return oracle_mod.smooth(rp, ci, xs, m, a, b, np.ones(n), np.zeros(n))


@pytest.mark.parametrize("kappa", [9.0, 10.0, 6.3573556258858871, 30.0])
@pytest.mark.parametrize("m", [1, 2, 3, 4, 5])
def test_smoother_is_best_uniform_approximation(oracle_mod, kappa, m):
    """S(1, 0) on diag(x) = q_m(x): equals an independent Remez best approximation to 1/x on
    [lambda1/kappa, lambda1], max|1 - x q_m| = E_m, lambda1 an
    alternation point, and the Chebyshev closed form."""
    l1 = 8.0
    l0 = l1 / kappa
    xs = np.linspace(l0, l1, 4001)
    q = _diag_q(oracle_mod, xs, l1, kappa, m)
    qr, Estar = H.remez_inv(l0, l1, m)
    assert np.max(np.abs(q - qr(xs))) <= 1e-7 * np.max(np.abs(q))
    r = 1 - xs * q
    Em = (np.sqrt(kappa) - 1) ** m / (np.sqrt(kappa) + 1) ** m * (kappa - 1) / 2
    assert np.max(np.abs(r)) == pytest.approx(Em, rel=1e-12)
    assert r[-1] == pytest.approx((-1) ** (m + 1) * Em, rel=1e-12)  # value at lambda1
    assert Estar * l1 == pytest.approx(Em, rel=1e-7)
    assert np.max(np.abs(r - H.cheb_closed_form_r(xs, l0, l1, m))) < 1e-13 * max(1, Em)
    # (1 - r)/x is a polynomial of degree m: interpolate on m+1 nodes, predict elsewhere
    nodes = np.linspace(l0, l1, m + 1)
    qn = _diag_q(oracle_mod, nodes, l1, kappa, m)
    coef = np.polyfit(nodes, qn, m)
    assert np.max(np.abs(np.polyval(coef, xs) - q)) < 1e-9 * np.max(np.abs(q))
    # r(0) = 1: q finite at 0 (x=0 row gives S(1,0)=q(0), and 1 - 0*q = 1 trivially); check continuity
    q0 = _diag_q(oracle_mod, np.array([1e-300]), l1, kappa, m)
    assert np.isfinite(q0).all()


def test_smoother_matrix_function(oracle_mod, gen_mod):
    """S(f, x0) = x0 + q_m(A)(f - A x0) with q_m(A) from a dense eigendecomposition."""
    rng = np.random.default_rng(5)
    p = gen_mod.random_graph(40, 5, seed=7, weighted=True)
    A = H.A0_dense(p)
    hier = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 1, 3, coarsest_size=1000)
    l1 = np.abs(A).sum(1).max()
    assert hier.level_info(0)["lambda1"] == pytest.approx(l1, rel=1e-15)
    kappa = hier.level_info(0)["kappa"]
    qf = H.q_closed_form(l1 / kappa, l1, 3)
    R = H.matfun_sym(A, qf)
    f = rng.standard_normal(40)
    x0 = rng.standard_normal(40)
    x = hier.smooth(0, f, x0)
    ref = x0 + R @ (f - A @ x0)
    assert np.linalg.norm(x - ref) <= 1e-12 * np.linalg.norm(ref)
    # exact solution is a fixed point
    xs = np.linalg.solve(A, f)
    assert np.allclose(hier.smooth(0, f, xs), xs, rtol=1e-12, atol=1e-12)


# ----------------------------------------------------------------- matching
def _random_pass_graph(rng, n, deg, maxw):
    e = {(min(a, b), max(a, b)) for a, b in rng.integers(0, n, (int(n * deg / 2), 2)) if a != b}
    e = sorted(e)
    w = rng.integers(1, maxw + 1, len(e))
    rows = [a for a, b in e] + [b for a, b in e]
    cols = [b for a, b in e] + [a for a, b in e]
    ww = list(w) + list(w)
    M = sp.csr_matrix((np.array(ww, dtype=np.int64), (rows, cols)), shape=(n, n))
    M.sort_indices()
    return M.indptr.astype(np.int64), M.indices.astype(np.int32), M.data.astype(np.int64), e, w


def test_handshake_equals_edge_greedy(oracle_mod):
    """A1: the parallel handshake and the sequential edge-greedy rule give the same matching."""
    rng = np.random.default_rng(11)
    for trial in range(120):
        n = int(rng.integers(2, 300))
        rp, ci, w, _, _ = _random_pass_graph(rng, n, rng.uniform(0.5, 8), int(rng.integers(1, 4)))
        m0, _ = oracle_mod.match(rp, ci, w, seed=trial, level=trial % 3, pass_=trial % 4, rule=0)
        m1, rounds = oracle_mod.match(rp, ci, w, seed=trial, level=trial % 3, pass_=trial % 4, rule=1)
        assert np.array_equal(m0, m1)
        # matching invariants: symmetric, along edges, maximal
        for v in range(n):
            u = m0[v]
            if u >= 0:
                assert m0[u] == v and u in ci[rp[v]:rp[v + 1]]
            else:
                assert all(m0[x] >= 0 for x in ci[rp[v]:rp[v + 1]])


def test_matching_brute_force_unique(oracle_mod):
    """Brute force on <= 10-vertex graphs with the test's own key function (docs/keys.md): the
    unique matching M in which every non-M edge touches a larger-key M edge is the oracle's."""
    rng = np.random.default_rng(3)
    for trial in range(40):
        n = int(rng.integers(3, 11))
        rp, ci, w, e, ew = _random_pass_graph(rng, n, 3.0, 2)
        if len(e) == 0 or len(e) > 14:
            continue
        keys = [H.edge_key(ew[k], a, b, 7, 1, 2) for k, (a, b) in enumerate(e)]
        keys = [(int(w_), h_, lo_, hi_) for (w_, h_, lo_, hi_) in keys]
        # the oracle's hash equals the test's independent SplitMix64 implementation
        assert all(oracle_mod.edge_hash(7, 1, 2, int(a), int(b)) == keys[k][1] for k, (a, b) in enumerate(e))
        sols = []
        for mask in range(1 << len(e)):
            M = [k for k in range(len(e)) if mask >> k & 1]
            verts = [v for k in M for v in e[k]]
            if len(verts) != len(set(verts)):
                continue
            ok = True
            for k in range(len(e)):
                if k in M:
                    continue
                if not any(set(e[k]) & set(e[j]) and keys[j] > keys[k] for j in M):
                    ok = False
                    break
            if ok:
                sols.append(M)
        assert len(sols) == 1
        mate, _ = oracle_mod.match(rp, ci, w, seed=7, level=1, pass_=2, rule=0)
        got = sorted((v, int(mate[v])) for v in range(n) if mate[v] > v)
        assert got == sorted((int(e[k][0]), int(e[k][1])) for k in sols[0])


def _check_partition(rp, ci, agg, nc):
    n = len(agg)
    assert agg.min() >= 0 and agg.max() == nc - 1 and len(np.unique(agg)) == nc
    G = sp.csr_matrix((np.ones(len(ci)), ci, rp), shape=(n, n))
    import scipy.sparse.csgraph as csg
    for I in range(nc):
        mem = np.flatnonzero(agg == I)
        ncomp, _ = csg.connected_components(G[mem][:, mem], directed=False)
        assert ncomp == 1  # P:70 "all subgraphs ... non empty and connected"
    # numbering: ids increase with the aggregate's leader (min vertex of its pair <= min member ... monotone)
    first = np.array([np.flatnonzero(agg == I).min() for I in range(nc)])
    return first


def test_aggregate_pass_invariants(oracle_mod):
    rng = np.random.default_rng(21)
    for trial in range(40):
        n = int(rng.integers(2, 200))
        rp, ci, w, _, _ = _random_pass_graph(rng, n, rng.uniform(1, 6), 2)
        agg0, nc0 = oracle_mod.aggregate_pass(rp, ci, w, seed=trial, rule=0)
        agg1, nc1 = oracle_mod.aggregate_pass(rp, ci, w, seed=trial, rule=1)
        assert nc0 == nc1 and np.array_equal(agg0, agg1)
        _check_partition(rp, ci, agg0, nc0)
        mate, _ = oracle_mod.match(rp, ci, w, seed=trial)
        # every matched pair shares an aggregate; every aggregate has exactly one leader pair or is an isolated singleton
        for v in range(n):
            if mate[v] >= 0:
                assert agg0[v] == agg0[mate[v]]
        for I in range(nc0):
            mem = np.flatnonzero(agg0 == I)
            pairs = [v for v in mem if mate[v] > v]
            iso = [v for v in mem if rp[v + 1] == rp[v]]
            assert (len(pairs) == 1 and not iso) or (len(mem) == 1 and len(iso) == 1)
        # A4: ids are the rank of the leader (pair min) in increasing vertex order
        leaders = [min(np.flatnonzero(agg0 == I)[[mate[v] >= 0 or rp[v + 1] == rp[v] for v in np.flatnonzero(agg0 == I)]]) for I in range(nc0)]
        assert leaders == sorted(leaders)


# ----------------------------------------------------------------- Galerkin
def test_galerkin_dense_and_invariants(oracle_mod, gen_mod):
    """A_H = P^T A P as entry sums; for d = 0 a weighted graph Laplacian with
    zero row sums and negative off-diagonals; 1^T A_H 1 = 1^T A 1; nnz(A_H) <= nnz(A)."""
    rng = np.random.default_rng(2)
    for trial in range(20):
        n = int(rng.integers(5, 200))
        p = gen_mod.random_graph(n, 5, seed=trial, weighted=True, dirichlet=bool(trial % 2))
        A = H.A0_dense(p)
        agg = rng.integers(0, max(1, n // 4), n).astype(np.int32)
        _, agg = np.unique(agg, return_inverse=True)
        agg = agg.astype(np.int32)
        nc = int(agg.max()) + 1
        Asp = sp.csr_matrix(A)
        Asp.sort_indices()
        rp, ci, v = oracle_mod.quotient(Asp.indptr, Asp.indices, Asp.data, None, agg, nc, drop_diag=False)
        AH = H.dense(rp, ci, v, nc)
        P = H.P_dense(agg, nc)
        assert np.allclose(AH, P.T @ A @ P, rtol=1e-13, atol=1e-13)
        assert np.allclose(AH, AH.T, rtol=1e-14, atol=1e-14)
        assert len(ci) <= Asp.nnz
        assert AH.sum() == pytest.approx(A.sum(), rel=1e-12)
        off = AH - np.diag(np.diag(AH))
        assert (off[np.abs(off) > 0] < 0).all()
        if p.d is None:
            assert np.allclose(AH.sum(1), 0.0, atol=1e-12)
        # pass-graph quotient: multiplicities = number of fine edges joining I, J; no self loops
        W = (np.abs(A - np.diag(np.diag(A))) > 0).astype(np.int64)
        Wsp = sp.csr_matrix(W)
        Wsp.sort_indices()
        qrp, qci, qw = oracle_mod.quotient(Wsp.indptr, Wsp.indices, None, Wsp.data, agg, nc, drop_diag=True)
        WH = H.dense(qrp, qci, qw.astype(float), nc)
        ref = P.T @ W @ P
        np.fill_diagonal(ref, 0)
        assert np.array_equal(WH, ref)
    g = gold("spec_examples.json")
    p4 = path_graph(gen_mod, 4)
    rp, ci, v = oracle_mod.quotient(p4.rp, p4.ci, p4.val, None, np.array([0, 0, 1, 1], np.int32), 2, False)
    assert np.array_equal(H.dense(rp, ci, v, 2), g["galerkin_path4_pairs"])


def _hier_check(oracle_mod, p, hier, exact):
    A = sp.csr_matrix((p.val, p.ci, p.rp), shape=(p.n, p.n))
    if p.d is not None:
        A = A + sp.diags(p.d)
    A = sp.csr_matrix(A)
    for l in range(hier.nlev):
        rp, ci, v = hier.level_csr(l)
        Al = sp.csr_matrix((v, ci, rp), shape=(len(rp) - 1,) * 2)
        diff = abs(Al - A)
        tol = 0.0 if exact else 1e-12 * abs(A).max()
        assert diff.max() <= tol
        info = hier.level_info(l)
        assert info["lambda1"] == pytest.approx(np.abs(A).sum(1).max(), rel=1e-15)
        if l < hier.nlev - 1:
            agg = hier.level_agg(l)
            nc = info["nc"]
            _check_partition(rp, ci, agg, nc)
            P = sp.csr_matrix((np.ones(len(agg)), (np.arange(len(agg)), agg)), shape=(len(agg), nc))
            A = sp.csr_matrix(P.T @ A @ P)
            A.sum_duplicates()


def test_hierarchy_C1_exact(oracle_mod, gen_mod):
    """Every level of the C1 hierarchy is exactly P^T A P of the one above (integer-valued)."""
    p = gen_mod.problem("C1")
    hier = oracle_mod.setup_problem(p)
    assert hier.nlev >= 3  # A6: coarsest 100 keeps the inner FCG recursion exercised
    _hier_check(oracle_mod, p, hier, exact=True)
    hier2 = oracle_mod.setup_problem(p, rule=1)
    for l in range(hier.nlev - 1):
        assert np.array_equal(hier.level_agg(l), hier2.level_agg(l))  # A1 on a real hierarchy
    hier3 = oracle_mod.setup_problem(p)
    for l in range(hier.nlev):  # determinism
        assert all(np.array_equal(a, b) for a, b in zip(hier.level_csr(l), hier3.level_csr(l)))


def test_hierarchy_3d_and_singular(oracle_mod, gen_mod):
    p = gen_mod.grid3d(10)
    hier = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 3, 3, coarsest_size=20)
    _hier_check(oracle_mod, p, hier, exact=False)
    q = gen_mod.rgg(3000, seed=1)
    hs = oracle_mod.Hierarchy(q.rp, q.ci, q.val, None, 2, 2, coarsest_size=30)
    assert hs.singular
    _hier_check(oracle_mod, q, hs, exact=True)
    for l in range(hs.nlev):
        rp, ci, v = hs.level_csr(l)
        rs = np.add.reduceat(v, rp[:-1]) if len(rp) > 1 else []
        assert np.allclose(rs, 0.0, atol=1e-12)  # A_H 1 = 0


# ----------------------------------------------------------------- coarsest
def test_coarse_solve(oracle_mod, gen_mod):
    rng = np.random.default_rng(4)
    p = gen_mod.random_graph(60, 4, seed=3, weighted=True)
    hier = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 1, 2, coarsest_size=100)
    assert hier.nlev == 1
    A = H.A0_dense(p)
    b = rng.standard_normal(60)
    x = hier.coarse_solve(b)
    assert np.linalg.norm(A @ x - b) <= 1e-12 * np.linalg.norm(b)
    q = gen_mod.random_graph(60, 4, seed=4, weighted=True, dirichlet=False)
    hs = oracle_mod.Hierarchy(q.rp, q.ci, q.val, None, 1, 2, coarsest_size=100)
    As = H.A0_dense(q)
    x = hs.coarse_solve(b)
    assert abs(x.mean()) < 1e-13
    assert np.allclose(x, H.pinv_sym(As) @ b, rtol=1e-10, atol=1e-12)
    # S:64 example: path-2, b = (1,-1) -> (0.5,-0.5)
    p2 = path_graph(gen_mod, 2)
    h2 = oracle_mod.Hierarchy(p2.rp, p2.ci, p2.val, None, 1, 2, coarsest_size=10)
    assert np.allclose(h2.coarse_solve(np.array([1.0, -1.0])), [0.5, -0.5], atol=1e-15)


# ----------------------------------------------------------------- two-level / k-cycle
def _seed_for_pairs(gen_mod):
    """A seed whose level-0/pass-0 keys make {0,1},{2,3} the matching of path-4."""
    for s in range(100):
        k = [H.edge_key(1, a, a + 1, s, 0, 0) for a in range(3)]
        if k[1] < max(k[0], k[2]):
            return s
    raise AssertionError


def test_golden_W1(oracle_mod, gen_mod):
    g = gold("w1_path4.json")
    p = path_graph(gen_mod, 4, d=[1, 0, 0, 0])
    seed = _seed_for_pairs(gen_mod)
    hier = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 1, g["m"], coarsest_size=2, seed=seed)
    assert hier.nlev == 2
    assert list(hier.level_agg(0)) == g["aggregates"]
    info = hier.level_info(0)
    assert info["lambda1"] == g["lambda1"] and info["kappa"] == g["kappa"]
    a, b = hier.level_coeffs(0)
    assert np.allclose(a, g["alpha"], rtol=1e-15) and np.allclose(b, g["beta"], rtol=1e-15)
    rp, ci, v = hier.level_csr(1)
    assert np.array_equal(H.dense(rp, ci, v, 2), g["A_H"])
    e0 = np.array([1.0, 0, 0, 0])
    assert np.allclose(hier.smooth(0, e0, np.zeros(4)), g["q3_A_e0"], rtol=1e-14, atol=1e-15)
    Be0 = hier.precond(e0, nu=2)
    assert np.allclose(Be0, g["B_e0"], rtol=1e-14, atol=1e-15)
    A = np.array(g["A"], float)
    B = np.column_stack([hier.precond(np.eye(4)[j]) for j in range(4)])
    assert np.allclose(np.sort(np.linalg.eigvals(B @ A).real), g["eig_BA"], atol=1e-12)


@pytest.mark.parametrize("singular", [False, True])
@pytest.mark.parametrize("m", [2, 3, 4])
def test_two_level_dense_formula(oracle_mod, gen_mod, singular, m):
    """B(r) equals Rbar + (I-RA) P A_H^+ P^T (I-AR) with R = q_m(A) from the closed form;
    B symmetric; eig(BA) in (0, 1] when E_m < 1."""
    rng = np.random.default_rng(m + 10 * singular)
    p = gen_mod.random_graph(120, 5, seed=m, weighted=True, dirichlet=not singular)
    hier = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 2, m, coarsest_size=60)
    assert hier.nlev == 2
    A = H.A0_dense(p)
    l1 = hier.level_info(0)["lambda1"]
    kappa = hier.level_info(0)["kappa"]
    R = H.matfun_sym(A, H.q_closed_form(l1 / kappa, l1, m))
    agg = hier.level_agg(0)
    P = H.P_dense(agg, hier.level_info(0)["nc"])
    AH = P.T @ A @ P
    AHi = H.pinv_sym(AH) if singular else np.linalg.inv(AH)
    B = H.two_level_B(A, P, R, AHi)
    Bo = np.column_stack([hier.precond(np.eye(120)[j]) for j in range(120)])
    assert np.linalg.norm(Bo - B) <= 1e-10 * np.linalg.norm(B)
    r = rng.standard_normal(120)
    assert np.linalg.norm(hier.precond(r) - B @ r) <= 1e-10 * np.linalg.norm(B @ r)
    assert np.allclose(Bo, Bo.T, atol=1e-10 * np.abs(Bo).max())
    ev = np.linalg.eigvals(Bo @ A).real
    if singular:
        ev = np.sort(ev)[1:]  # drop the kernel
    assert ev.min() > 0 and ev.max() <= 1 + 1e-10


def test_kcycle_partial_pins(oracle_mod, gen_mod):
    """Multilevel k-cycle: positive homogeneity B(cr) = cB(r); the linear V-cycle switch is
    symmetric and equals the dense recursion B_l = Rbar + (I-RA)P B_{l+1} P^T (I-AR)."""
    p = gen_mod.grid2d(18)
    hk = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 2, 3, coarsest_size=10)
    assert hk.nlev >= 3
    rng = np.random.default_rng(9)
    r = rng.standard_normal(p.n)
    z = hk.precond(r)
    assert np.allclose(hk.precond(3.5 * r), 3.5 * z, rtol=1e-13, atol=1e-13)
    hv = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 2, 3, coarsest_size=10, cycle=1)
    s = rng.standard_normal(p.n)
    assert (hv.precond(r) @ s) == pytest.approx(r @ hv.precond(s), rel=1e-10)
    # dense recursion
    mats = []
    for l in range(hv.nlev):
        rp, ci, v = hv.level_csr(l)
        mats.append(H.dense(rp, ci, v))
    Bl = np.linalg.inv(mats[-1])
    for l in range(hv.nlev - 2, -1, -1):
        A = mats[l]
        l1 = hv.level_info(l)["lambda1"]
        kap = hv.level_info(l)["kappa"]
        R = H.matfun_sym(A, H.q_closed_form(l1 / kap, l1, 3))
        P = H.P_dense(hv.level_agg(l), hv.level_info(l)["nc"])
        Bl = H.two_level_B(A, P, R, Bl)
    assert np.linalg.norm(hv.precond(r) - Bl @ r) <= 1e-10 * np.linalg.norm(Bl @ r)
    # two levels: k-cycle == two-level B (no inner FCG runs)
    h2 = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 2, 3, coarsest_size=200)
    h2v = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 2, 3, coarsest_size=200, cycle=1)
    assert h2.nlev == 2 and np.allclose(h2.precond(r), h2v.precond(r), rtol=0, atol=0)


def test_fcg_equals_pcg_and_exact_precond(oracle_mod, gen_mod):
    """FCG == PCG when B is linear SPD and restart >= max_iter; FCG with B = A^{-1}
    converges in one iteration."""
    p = gen_mod.grid2d(20)
    hv = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 2, 3, coarsest_size=10, cycle=1, restart=1000)
    A = H.A0_dense(p)
    b = gen_mod.rhs(p.n, 1)
    res = hv.solve(b, tol=1e-10)
    x, k, _ = H.pcg(A, b, lambda r: hv.precond(r), 1e-10, 500)
    assert res["status"] == 0 and res["iters"] == k
    assert np.linalg.norm(res["x"] - x) <= 1e-8 * np.linalg.norm(x)
    h1 = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 2, 3, coarsest_size=1000)
    assert h1.nlev == 1
    r1 = h1.solve(b, tol=1e-10)
    assert r1["iters"] == 1 and r1["relres"] < 1e-12


def test_full_solve_C1(oracle_mod, gen_mod):
    """relres <= tol on the recursive and the true residual; error vs a sparse direct solve within
    tol * sqrt(cond(A)) in the A-norm (SURVEY 8(c) pins, 'Full solve')."""
    p = gen_mod.problem("C1")
    hier = oracle_mod.setup_problem(p)
    b = gen_mod.rhs(p.n, 0)
    res = hier.solve(b, tol=1e-8, nu=2)
    assert res["status"] == 0 and res["relres"] <= 1e-8 and res["true_relres"] <= 1.5e-8
    assert 8 <= res["iters"] <= 30
    A = sp.csr_matrix((p.val, p.ci, p.rp), shape=(p.n, p.n)) + sp.diags(p.d)
    xs = spla.spsolve(sp.csc_matrix(A), b)
    e = res["x"] - xs
    cond = 8.0 / (2 * (1 - np.cos(np.pi / 65)))  # 5-pt Dirichlet spectrum
    assert np.sqrt(e @ (A @ e)) <= 1e-8 * np.sqrt(cond) * np.sqrt(xs @ (A @ xs))


def test_singular_solve(oracle_mod, gen_mod):
    q = gen_mod.rgg(4000, seed=2)
    hier = oracle_mod.Hierarchy(q.rp, q.ci, q.val, None, 3, 3, coarsest_size=50)
    b = gen_mod.rhs(q.n, 0)
    res = hier.solve(b, tol=1e-8)
    assert res["status"] == 0 and res["true_relres"] <= 2e-8


def test_error_codes(oracle_mod, gen_mod):
    p = path_graph(gen_mod, 5)
    with pytest.raises(oracle_mod.OracleError) as e:
        oracle_mod.Hierarchy(p.rp, p.ci, p.val, None, 0, 2)
    assert e.value.code == -1
    with pytest.raises(oracle_mod.OracleError) as e:
        oracle_mod.Hierarchy(p.rp, p.ci, p.val, None, 1, 2, kappa=10.0)  # A9: E_2(10) >= 1
    assert e.value.code == -1
    bad = p.val.copy()
    bad[1] = 0.5  # positive off-diagonal
    with pytest.raises(oracle_mod.OracleError) as e:
        oracle_mod.Hierarchy(p.rp, p.ci, bad, None, 1, 2)
    assert e.value.code == -2
    asym = p.val.copy()
    asym[1] = -2.0
    with pytest.raises(oracle_mod.OracleError) as e:
        oracle_mod.Hierarchy(p.rp, p.ci, asym, None, 1, 2)
    assert e.value.code == -2
    # diagonal-only matrix above coarsest size: coarsening stagnates
    n = 200
    with pytest.raises(oracle_mod.OracleError) as e:
        oracle_mod.Hierarchy(np.zeros(n + 1, np.int64), np.zeros(0, np.int32), np.zeros(0), np.ones(n), 1, 2, coarsest_size=10)
    assert e.value.code == -7


def test_missing_diagonal_inserted(oracle_mod, gen_mod):
    p = gen_mod.random_graph(30, 4, seed=5, weighted=True)
    keep = p.ci != np.repeat(np.arange(p.n), np.diff(p.rp))
    rp = np.concatenate([[0], np.cumsum(np.add.reduceat(keep.astype(np.int64), p.rp[:-1]))])
    h_full = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 1, 2, coarsest_size=10)
    h_nod = oracle_mod.Hierarchy(rp, p.ci[keep], p.val[keep], p.d, 1, 2, coarsest_size=10)
    for l in range(h_full.nlev):
        a, b = h_full.level_csr(l), h_nod.level_csr(l)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and np.allclose(a[2], b[2], rtol=1e-15)


def test_decoupled_aggregation(oracle_mod, gen_mod):
    """A20: with nparts = P no aggregate crosses a row block; coarse blocks stay contiguous."""
    p = gen_mod.grid2d(40)
    for P in (2, 3, 4):
        hier = oracle_mod.setup_problem(gen_mod.problem("C1", size=40), nparts=P, gather_rows=100)
        n = p.n
        blk = np.zeros(n, np.int64)
        for b in range(P):
            blk[b * n // P:(b + 1) * n // P] = b
        for l in range(hier.nlev - 1):
            info = hier.level_info(l)
            agg = hier.level_agg(l)
            if info["nparts"] > 1:
                for I in range(info["nc"]):
                    assert len(np.unique(blk[agg == I])) == 1
                cblk = np.zeros(info["nc"], np.int64)
                cblk[agg] = blk
                assert np.all(np.diff(cblk) >= 0)
                blk = cblk
            else:
                blk = np.zeros(info["nc"], np.int64)
        res = hier.solve(gen_mod.rhs(n, 0), tol=1e-8)
        assert res["status"] == 0
    h1 = oracle_mod.setup_problem(gen_mod.problem("C1", size=40), nparts=1)
    h1b = oracle_mod.setup_problem(gen_mod.problem("C1", size=40))
    assert np.array_equal(h1.level_agg(0), h1b.level_agg(0))


def _poly_of_matrix(M, q, m, l0, l1):
    """q(M) for the degree-m polynomial q (exact monomial fit on m+1 Chebyshev points of [l0, l1])."""
    t = 0.5 * (l0 + l1) + 0.5 * (l1 - l0) * np.cos(np.pi * (np.arange(m + 1) + 0.5) / (m + 1))
    c = np.linalg.solve(np.vander(t, m + 1, increasing=True), q(t))
    out = c[m] * np.eye(M.shape[0])
    for k in range(m - 1, -1, -1):  # Horner
        out = out @ M + c[k] * np.eye(M.shape[0])
    return out


@pytest.mark.parametrize("nu", [2, 3])
def test_amli_cycle_pins(oracle_mod, gen_mod, nu):
    """Stationary AMLI cycle (cycle=2, reading A23): a fixed LINEAR symmetric operator
    (S:406-408); equals the dense recursion B_l = Rbar + (I-RA) P M_{l+1} P^T (I-AR) with
    M_{l+1} = q(B_{l+1} A_{l+1}) B_{l+1} (q = degree-(nu-1) best approximation to 1/t on [1/kappa_A, 1],
    evaluated here as an explicit matrix polynomial), M = A_L^{-1} on the coarsest; SPD."""
    p = gen_mod.grid2d(18)
    h = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 2, 3, coarsest_size=10, cycle=2)
    assert h.nlev >= 4
    rng = np.random.default_rng(nu)
    r, s = rng.standard_normal(p.n), rng.standard_normal(p.n)
    z = h.precond(r, nu=nu)
    assert np.allclose(h.precond(3.5 * r, nu=nu), 3.5 * z, rtol=1e-13, atol=1e-13)
    assert (z @ s) == pytest.approx(r @ h.precond(s, nu=nu), rel=1e-10)
    mats = []
    for l in range(h.nlev):
        rp, ci, v = h.level_csr(l)
        mats.append(H.dense(rp, ci, v))
    kapA = oracle_mod.kappa_rule(nu - 1)
    q = H.q_closed_form(1.0 / kapA, 1.0, nu - 1)
    M = np.linalg.inv(mats[-1])  # coarse operator seen by level L-2: exact solve (A12)
    for l in range(h.nlev - 2, -1, -1):
        A = mats[l]
        l1 = h.level_info(l)["lambda1"]
        kap = h.level_info(l)["kappa"]
        R = H.matfun_sym(A, H.q_closed_form(l1 / kap, l1, 3))
        P = H.P_dense(h.level_agg(l), h.level_info(l)["nc"])
        B = H.two_level_B(A, P, R, M)
        if l >= 1:
            M = _poly_of_matrix(B @ A, q, nu - 1, 1.0 / kapA, 1.0) @ B
    assert np.linalg.norm(z - B @ r) <= 1e-10 * np.linalg.norm(B @ r)
    ev = np.linalg.eigvals(B @ mats[0]).real
    assert ev.min() > 0
    # nu = 1: the AMLI cycle is the V-cycle (one B application per coarse level)
    hv = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 2, 3, coarsest_size=10, cycle=1)
    assert np.array_equal(h.precond(r, nu=1), hv.precond(r, nu=1))


def test_amli_solve_converges(oracle_mod, gen_mod):
    """CG (the outer FCG with a linear preconditioner) with the AMLI cycle solves C1."""
    p = gen_mod.problem("C1")
    h = oracle_mod.setup_problem(p, cycle=2)
    b = gen_mod.rhs(p.n, 0)
    res = h.solve(b, tol=1e-8, nu=2)
    assert res["status"] == 0 and res["true_relres"] <= 2e-8
    assert res["iters"] <= 40


def test_lanczos_lambda_max_pins(oracle_mod, gen_mod):
    """Reading A24 (opt-in): the Ritz value is a lower bound of lambda_max that
    reaches it with k = n steps; 1.1 x the 10-step value bounds lambda_max from above on the test
    graphs; the setup uses min(||A||_inf, 1.1 theta_10)."""
    for seed, (n, weighted) in enumerate([(40, False), (60, True)]):
        p = gen_mod.random_graph(n, 5, seed=seed + 3, weighted=weighted, dirichlet=True)
        A = H.A0_dense(p)
        lmax = np.linalg.eigvalsh(A).max()
        rp, ci, v = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 1, 2, coarsest_size=n).level_csr(0)
        for k in (2, 5, 10):
            t = oracle_mod.lanczos_max(rp, ci, v, k)
            assert t <= lmax * (1 + 1e-12)
        assert oracle_mod.lanczos_max(rp, ci, v, n) == pytest.approx(lmax, rel=1e-8)
    for p in (gen_mod.problem("C1"), gen_mod.rgg(3000, seed=2), gen_mod.random_graph(800, 7, seed=4, weighted=True)):
        import scipy.sparse as sp
        import scipy.sparse.linalg as sla

        h0 = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 2, 3, coarsest_size=50)
        rp, ci, v = h0.level_csr(0)
        A = sp.csr_matrix((v, ci, rp))
        lmax = sla.eigsh(A, k=1, which="LA", return_eigenvectors=False)[0]
        t = oracle_mod.lanczos_max(rp, ci, v, 10)
        assert t <= lmax * (1 + 1e-12) and 1.1 * t >= lmax
        h = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 2, 3, coarsest_size=50, lanczos=10)
        assert h.level_info(0)["lambda1"] == pytest.approx(min(h0.level_info(0)["lambda1"], 1.1 * t), rel=1e-15)
        assert h.level_info(0)["lambda1"] >= lmax


def _bfs_dist(rp, ci, src, n):
    d = np.full(n, -1)
    d[src] = 0
    q = [src]
    for u in q:
        for p in range(rp[u], rp[u + 1]):
            x = ci[p]
            if x != u and d[x] < 0:
                d[x] = d[u] + 1
                q.append(x)
    return d


@pytest.mark.parametrize("k", [2, 4])
def test_mis_aggregation_pins(oracle_mod, gen_mod, k):
    """Reading A25 (the paper's partitioner; NEXT row f2, oracle only): the roots are an
    independent set of the graph of A^k (pairwise distance > k) that is maximal (every vertex within
    distance k of a root) and greedy by key; every vertex is assigned to a root at its distance to the
    root set (the BFS layer), aggregates are connected and numbered by root order."""
    for p in (gen_mod.problem("C1", size=20), gen_mod.random_graph(300, 5, seed=8)):
        n = p.n
        agg, nc, roots = oracle_mod.mis_aggregate(p.rp, p.ci, k, seed=3, level=1)
        assert nc > 0 and agg.min() == 0 and agg.max() == nc - 1
        dist = np.array([_bfs_dist(p.rp, p.ci, v, n) for v in range(n)])  # all-pairs hop distances
        dist = np.where(dist < 0, 10 ** 9, dist)
        S = np.flatnonzero(roots)
        assert len(S) == nc and np.array_equal(agg[S], np.arange(nc))  # numbered by root order
        DS = dist[:, S]
        for a in range(len(S)):
            for b in range(a + 1, len(S)):
                assert DS[S[a], b] > k, "roots within distance k"
        assert np.all(DS.min(axis=1) <= k), "not maximal"
        # greedy by key (reading A25): v is a root iff no root with a larger key lies within distance k
        misalt = H.splitmix64((3 ^ 0x4D49530000000000 ^ 1) & (2 ** 64 - 1))
        key = np.array([((H.splitmix64(v ^ misalt) >> 32) << 32) | v for v in range(n)], dtype=object)
        for v in range(n):
            near = [u for u in S if dist[v, u] <= k and u != v]
            assert roots[v] == all(key[u] < key[v] for u in near)
        for v in range(n):  # assigned to a root at the vertex's distance to the root set (its layer)
            assert DS[v, agg[v]] == DS[v].min()
        for I in range(nc):  # connected
            mem = np.flatnonzero(agg == I)
            sub = set(mem.tolist())
            seen, stack = {mem[0]}, [mem[0]]
            while stack:
                u = stack.pop()
                for pp in range(p.rp[u], p.rp[u + 1]):
                    x = p.ci[pp]
                    if x in sub and x not in seen:
                        seen.add(x)
                        stack.append(x)
            assert len(seen) == len(mem)


def test_mis_hierarchy_paper_protocol(oracle_mod):
    """The paper's protocol on the P1-FE pattern of a 128^2 Neumann problem (structural zeros on the
    hypotenuse couplings kept, A17): MIS on A^4 coarsens by ~30 with complexities near the
    paper's, and both cycles converge under the A-norm error stop."""
    N = 128
    n = N * N
    rows = []
    for y in range(N):
        for x in range(N):
            i = y * N + x
            nb = [(i - 1, -1.0)] * (x > 0) + [(i + 1, -1.0)] * (x < N - 1) + [(i - N, -1.0)] * (y > 0) + \
                [(i + N, -1.0)] * (y < N - 1) + [(i - N - 1, 0.0)] * (x > 0 and y > 0) + \
                [(i + N + 1, 0.0)] * (x < N - 1 and y < N - 1)
            rows.append(sorted(nb + [(i, -sum(v for _, v in nb))]))
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    ci = np.array([c for r in rows for c, _ in r], np.int32)
    v = np.array([w for r in rows for _, w in r])
    h = oracle_mod.Hierarchy(rp, ci, v, None, 1, 4, coarsest_size=99, mis_k=4)
    cf = h.level_info(0)["n"] / h.level_info(1)["n"]
    gc, oc = h.complexities()
    assert 25 < cf < 35 and gc < 1.05 and oc < 1.05
    import scipy.sparse as sp

    xs = np.random.default_rng(0).standard_normal(n)
    xs -= xs.mean()
    b = sp.csr_matrix((v, ci, rp)) @ xs
    for cyc in (0, 2):
        hc = oracle_mod.Hierarchy(rp, ci, v, None, 1, 4, coarsest_size=99, mis_k=4, cycle=cyc)
        r = hc.solve(b, tol=1e-8, nu=2, xstar=xs)
        assert r["status"] == 0 and r["iters"] <= 40


def test_kcycle_three_and_four_levels_pinned(oracle_mod, gen_mod):
    """The nonlinear k-cycle at L > 2 against mathematics:
    (1) with nu large the inner FCG on level 1 is preconditioned by a linear SPD B_1, so it is PCG and
        solves A_1 e = rho exactly (Krylov termination): B_0 equals the two-level formula of P:136
        with the exact A_1^{-1} (L = 3 and L = 4);
    (2) with nu = 1 the inner FCG takes one step from e = 0 along d = B_1 rho with the optimal
        (A_1-norm minimising) step d.rho / d.A_1 d: B_0(r) is the smoothed two-level cycle with that
        coarse correction, B_1 itself the exact two-level operator of level 1 (L = 3)."""
    p = gen_mod.grid2d(18)
    rng = np.random.default_rng(2)
    r = rng.standard_normal(p.n)
    for cs, L in [(30, 3), (10, 4)]:
        hk = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 2, 3, coarsest_size=cs)
        assert hk.nlev == L
        mats = []
        for l in range(hk.nlev):
            rp, ci, v = hk.level_csr(l)
            mats.append(H.dense(rp, ci, v))

        def smoother_R(l):
            l1 = hk.level_info(l)["lambda1"]
            kap = hk.level_info(l)["kappa"]
            return H.matfun_sym(mats[l], H.q_closed_form(l1 / kap, l1, 3))

        A, A1 = mats[0], mats[1]
        R = smoother_R(0)
        P = H.P_dense(hk.level_agg(0), hk.level_info(0)["nc"])
        B = H.two_level_B(A, P, R, np.linalg.inv(A1))
        z = hk.precond(r, nu=2 * A1.shape[0])
        assert np.linalg.norm(z - B @ r) <= 1e-12 * np.linalg.norm(B @ r), L
        if L == 3:
            R1 = smoother_R(1)
            P1 = H.P_dense(hk.level_agg(1), hk.level_info(1)["nc"])
            B1 = H.two_level_B(A1, P1, R1, np.linalg.inv(mats[2]))
            x0 = R @ r
            rho = P.T @ (r - A @ x0)
            d = B1 @ rho
            e = (d @ rho) / (d @ (A1 @ d)) * d
            x1 = x0 + P @ e
            x2 = x1 + R @ (r - A @ x1)
            z1 = hk.precond(r, nu=1)
            assert np.linalg.norm(z1 - x2) <= 1e-12 * np.linalg.norm(x2)


# ----------------------------------------------------------------- sub-rules pinned independently
def test_attach_rule_recomputed(oracle_mod):
    """Reading A3 (SURVEY 8(c) O3c 'Attach'; matching named at P:71-73): every vertex left unmatched
    by the maximal matching joins the pair of its MAX-key neighbour (all its neighbours are matched);
    isolated vertices stay singletons; ids are leader ranks (A4).  Recomputed here with the test's own
    key function (tests/helpers.py edge_key, docs/keys.md) from the matching alone (itself pinned by
    brute force above), and checked to discriminate: on these graphs a first-neighbour or min-key
    attach gives different aggregates."""
    rng = np.random.default_rng(77)
    discriminating = 0
    for trial in range(60):
        n = int(rng.integers(6, 250))
        rp, ci, w, _, _ = _random_pass_graph(rng, n, rng.uniform(1.5, 6), int(rng.integers(1, 4)))
        seed, level, pas = trial * 7 + 1, trial % 4, trial % 3
        mate, _ = oracle_mod.match(rp, ci, w, seed=seed, level=level, pass_=pas, rule=1)
        got, nc = oracle_mod.aggregate_pass(rp, ci, w, seed=seed, level=level, pass_=pas, rule=1)

        def expected(choose):
            leader = np.empty(n, np.int64)
            for v in range(n):
                nb = list(range(rp[v], rp[v + 1]))
                if mate[v] >= 0:
                    leader[v] = min(v, mate[v])
                elif not nb:
                    leader[v] = v
                else:
                    u = choose(v, nb)
                    assert mate[u] >= 0  # maximality
                    leader[v] = min(u, mate[u])
            leaders = sorted(set(leader.tolist()))
            rank = {L: k for k, L in enumerate(leaders)}
            return np.array([rank[L] for L in leader], np.int32), len(leaders)

        def by_key(sign):
            def choose(v, nb):
                keys = [H.edge_key(w[p], v, ci[p], seed, level, pas) for p in nb]
                best = max(range(len(nb)), key=lambda k: keys[k]) if sign > 0 else \
                    min(range(len(nb)), key=lambda k: keys[k])
                return int(ci[nb[best]])
            return choose

        ref, ncr = expected(by_key(+1))
        assert nc == ncr and np.array_equal(got, ref), f"trial {trial}"
        for alt in (by_key(-1), lambda v, nb: int(ci[nb[0]])):
            a, _ = expected(alt)
            discriminating += int(not np.array_equal(a, ref))
    assert discriminating >= 40  # the pin would catch a min-key or first-neighbour attach


def test_restart_window_iterates(oracle_mod, gen_mod):
    """Restart every five iterations: the oracle's outer FCG equals an
    independent numpy FCG (tests/helpers.py fcg_restarted) with the oracle's preconditioner used as
    a black box, iterate by iterate (orc_solve stopped after k iterations by max_iter = k), for
    restart 5 and 3 and for the linear V-cycle (cycle 1) and the nonlinear k-cycle (cycle 0).  The
    same reference with the window cleared one step late, or never, differs by far more than the
    tolerance, so an off-by-one or a missing clear fails."""
    p = gen_mod.grid2d(24)
    A = H.A0_dense(p)
    b = gen_mod.rhs(p.n, 3)
    K = 13
    for cycle in (1, 0):
        for W in (5, 3):
            hb = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 2, 3, coarsest_size=30, cycle=cycle, restart=W)
            Bop = lambda r: hb.precond(r, nu=2)  # noqa: E731
            xs, _ = H.fcg_restarted(A, b, Bop, 1e-30, K, W)
            late, _ = H.fcg_restarted(A, b, Bop, 1e-30, K, W + 1)
            never, _ = H.fcg_restarted(A, b, Bop, 1e-30, K, 10 ** 6)
            sep = 0.0
            for k in range(1, K + 1):
                hk = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 2, 3, coarsest_size=30, cycle=cycle, restart=W,
                                          max_iter=k)
                res = hk.solve(b, tol=1e-30, nu=2)
                assert res["status"] == oracle_mod.ORC_NOT_CONVERGED and res["iters"] == k
                scale = max(np.linalg.norm(xs[k]), 1e-300)
                assert np.linalg.norm(res["x"] - xs[k]) <= 1e-9 * scale, (cycle, W, k)
                sep = max(sep, np.linalg.norm(late[k] - xs[k]) / scale, np.linalg.norm(never[k] - xs[k]) / scale)
            assert sep > 1e-6, (cycle, W, sep)


def test_anorm_stop_rule_dense(oracle_mod, gen_mod):
    """The paper's stopping test, relative A-norm error reduction 1e-8, evaluated with a
    dense A: the oracle stops at the FIRST k with ||x_k - x*||_A <= tol ||x_0 - x*||_A, i.e. at k
    the dense ratio is <= tol and at k - 1 (same hierarchy stopped by max_iter) it is > tol; the
    iteration count equals the independent numpy FCG's with the same dense test."""
    for name, p, d in (("grid", gen_mod.grid2d(24), True), ("rgg", gen_mod.rgg(1500, seed=4), False)):
        A = H.A0_dense(p)
        rng = np.random.default_rng(5)
        xstar = rng.standard_normal(p.n)
        if not d:
            xstar -= xstar.mean()
        b = A @ xstar
        dd = p.d if d else None
        for tol in (1e-4, 1e-8):
            h = oracle_mod.Hierarchy(p.rp, p.ci, p.val, dd, 2, 3, coarsest_size=30)
            res = h.solve(b, tol=tol, nu=2, xstar=xstar)
            assert res["status"] == 0
            k = res["iters"]

            def ratio(x):
                e = x - xstar
                return np.sqrt(e @ (A @ e)) / np.sqrt(xstar @ (A @ xstar))

            assert ratio(res["x"]) <= tol * (1 + 1e-9), name
            hp = oracle_mod.Hierarchy(p.rp, p.ci, p.val, dd, 2, 3, coarsest_size=30, max_iter=k - 1)
            prev = hp.solve(b, tol=tol, nu=2, xstar=xstar)
            assert prev["status"] == oracle_mod.ORC_NOT_CONVERGED and ratio(prev["x"]) > tol, name
            xs, kref = H.fcg_restarted(A, b, lambda r: h.precond(r, nu=2) - (0 if d else h.precond(r, nu=2).mean()),
                                       tol, 200, 5, anorm_stop=xstar)
            assert kref == k, (name, tol, kref, k)


def test_zero_residual_inner_fcg(oracle_mod, gen_mod):
    """Reading A13 (inner FCG): rho = 0 gives d = 0 and d.q = 0; the step and every later
    orthogonalisation against that direction contribute nothing, so B_l(0) = 0 exactly (no 0/0) for
    nu = 1, 2, 3 on a hierarchy with inner FCG levels (L >= 3); B is positively homogeneous, so the
    zero vector is its only fixed output for r = 0."""
    p = gen_mod.grid2d(24)
    h = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 2, 3, coarsest_size=10)
    assert h.nlev >= 3
    for nu in (1, 2, 3):
        z = h.precond(np.zeros(p.n), nu=nu)
        assert np.all(np.isfinite(z)) and not np.any(z), nu
