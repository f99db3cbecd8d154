"""-m gpu parity of the CUDA path (through the C ABI) against the CPU oracle on identical seeded inputs.

Bars (BASELINE.json north_star): aggregate ids and coarse sparsity bit-exact; per-level coarse
values <= 1e-12 relative; one preconditioner application <= 1e-10 relative; final relative
residual <= tol with FCG iteration counts within +-1 of the oracle.
"""
import json
import os

import numpy as np
import pytest

import helpers as H

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def amg():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1307_6305_b200 import amg as A

    A.load()
    return A


def gpu_setup(amg, p, device_arrays=False, **over):
    prm = dict(p.params)
    prm.update(over)
    o = amg.amg_options_default(coarsest_size=prm.get("coarsest_size", 100), kappa=prm.get("kappa", 0.0),
                                seed=prm.get("seed", 0), restart=prm.get("restart", 5))
    arrs = [p.rp, p.ci, p.val, p.d]
    if device_arrays:
        import torch

        arrs = [None if a is None else torch.from_numpy(a).cuda() for a in arrs]
    h = amg.amg_setup(*arrs, prm["passes"], prm["degree"], o)
    return h


def compare_hierarchy(amg, h, hier, m, exact_values):
    info = amg.amg_get_info(h)
    assert info["levels"] == hier.nlev
    for l in range(hier.nlev):
        rp, ci, v, agg = amg.amg_level_export(h, l, m)
        orp, oci, ov = hier.level_csr(l)
        oi = hier.level_info(l)
        assert np.array_equal(rp, orp), f"level {l} row_ptr"
        assert np.array_equal(ci, oci), f"level {l} col"
        if exact_values:
            assert np.array_equal(v, ov), f"level {l} values not bit-exact"
        else:
            assert np.max(np.abs(v - ov)) <= 1e-12 * np.max(np.abs(ov)), f"level {l} values"
        s = amg.amg_level_sizes(h, l, m)
        assert s["lambda1"] == pytest.approx(oi["lambda1"], rel=1e-15, abs=0)
        assert s["kappa"] == pytest.approx(oi["kappa"], rel=4e-16)
        a, b = hier.level_coeffs(l)
        assert np.allclose(s["alpha"], a, rtol=4e-15, atol=0) and np.allclose(s["beta"], b, rtol=4e-15, atol=0)
        if l < hier.nlev - 1:
            assert s["nc"] == oi["nc"]
            assert np.array_equal(agg, hier.level_agg(l)), f"level {l} aggregates"


def small_cases(gen):
    cases = [gen.problem("C1"), gen.problem("C2", size=96)]
    c = gen.problem("C4", size=14)
    c.params["coarsest_size"] = 30
    cases.append(c)
    for seed, (n, weighted, dirichlet) in enumerate([(700, True, True), (900, False, False), (1500, True, False)]):
        q = gen.random_graph(n, 6, seed=seed + 40, weighted=weighted, dirichlet=dirichlet)
        q.params = dict(passes=2, degree=3, coarsest_size=40, seed=seed)
        cases.append(q)
    q = gen.rgg(5000, seed=3)
    q.params = dict(passes=3, degree=4, coarsest_size=60, seed=1)
    cases.append(q)
    return cases


def test_hierarchy_bit_exact_small(amg, gen_mod, oracle_mod):
    for p in small_cases(gen_mod):
        hier = oracle_mod.setup_problem(p)
        h = gpu_setup(amg, p)
        try:
            integer_valued = bool(np.all(p.val == np.round(p.val)) and (p.d is None or np.all(p.d == np.round(p.d))))
            compare_hierarchy(amg, h, hier, p.params["degree"], exact_values=True)
            del integer_valued
        finally:
            amg.amg_free(h)


def test_device_pointer_inputs(amg, gen_mod, oracle_mod):
    p = gen_mod.problem("C1")
    hier = oracle_mod.setup_problem(p)
    h = gpu_setup(amg, p, device_arrays=True)
    try:
        compare_hierarchy(amg, h, hier, p.params["degree"], exact_values=True)
    finally:
        amg.amg_free(h)


@pytest.mark.parametrize("name", ["C1", "C2s", "C4s", "rgg"])
def test_smoother_precond_coarse_parity(amg, gen_mod, oracle_mod, name):
    p = {"C1": lambda: gen_mod.problem("C1"), "C2s": lambda: gen_mod.problem("C2", size=128),
         "C4s": lambda: gen_mod.problem("C4", size=16)}.get(name, None)
    if p is None:
        p = gen_mod.rgg(6000, seed=5)
        p.params = dict(passes=3, degree=3, coarsest_size=50, seed=0)
    else:
        p = p()
    hier = oracle_mod.setup_problem(p)
    h = gpu_setup(amg, p)
    m = p.params["degree"]
    rng = np.random.default_rng(1)
    try:
        for l in range(hier.nlev - 1):
            n = hier.level_info(l)["n"]
            f = rng.uniform(-1, 1, n)
            x0 = rng.uniform(-1, 1, n)
            x = np.empty(n)
            amg.amg_level_smooth(h, l, f, x0, x)
            ref = hier.smooth(l, f, x0)
            H.assert_close(x, ref, 1e-12, f"smoother level {l}")
        for l in range(hier.nlev):
            n = hier.level_info(l)["n"]
            r = rng.uniform(-1, 1, n)
            z = np.empty(n)
            amg.amg_level_precond(h, l, 2, r, z)
            ref = hier.precond(r, nu=2, level=l)
            H.assert_close(z, ref, 1e-10, f"B_{l}(r)")
        nL = hier.level_info(hier.nlev - 1)["n"]
        r = rng.uniform(-1, 1, nL)
        e = np.empty(nL)
        amg.amg_coarse_solve(h, r, e)
        ref = hier.coarse_solve(r)
        H.assert_close(e, ref, 1e-10)
    finally:
        amg.amg_free(h)


@pytest.mark.parametrize("name", ["C1", "C2", "C4s", "rgg", "rand_spd"])
def test_full_solve_parity(amg, gen_mod, oracle_mod, name):
    if name == "C4s":
        p = gen_mod.problem("C4", size=24)
    elif name == "rgg":
        p = gen_mod.rgg(20000, seed=7)
        p.params = dict(passes=4, degree=4, coarsest_size=100, seed=0, tol=1e-8, k_inner=2)
    elif name == "rand_spd":
        p = gen_mod.random_graph(3000, 7, seed=9, weighted=True, dirichlet=True)
        p.params = dict(passes=2, degree=2, coarsest_size=50, seed=0, tol=1e-8, k_inner=2)
    else:
        p = gen_mod.problem(name)
    hier = oracle_mod.setup_problem(p)
    b = gen_mod.rhs(p.n, 0)
    ref = hier.solve(b, tol=1e-8, nu=2)
    h = gpu_setup(amg, p)
    try:
        for use_host in (True, False):
            if use_host:
                x = np.zeros(p.n)
                st, it, rr = amg.amg_solve(h, b, x, 1e-8, 2)
            else:
                import torch

                bt = torch.from_numpy(b).cuda()
                xt = torch.zeros(p.n, dtype=torch.float64, device="cuda")
                st, it, rr = amg.amg_solve(h, bt, xt, 1e-8, 2)
                x = xt.cpu().numpy()
            info = amg.amg_get_info(h)
            assert st == 0 and rr <= 1e-8 and info["last_true_relres"] <= 2e-8
            assert abs(it - ref["iters"]) <= 1, (it, ref["iters"])
            H.assert_close(x, ref["x"], 1e-6)
        # determinism: a second solve is bitwise identical (T6)
        x1 = np.zeros(p.n)
        x2 = np.zeros(p.n)
        amg.amg_solve(h, b, x1, 1e-8, 2)
        amg.amg_solve(h, b, x2, 1e-8, 2)
        assert np.array_equal(x1, x2)
    finally:
        amg.amg_free(h)


def test_no_graph_path_matches_graph_path(amg, gen_mod):
    p = gen_mod.problem("C2", size=200)
    b = gen_mod.rhs(p.n, 2)
    xs = []
    for g in (1, 0):
        o = amg.amg_options_default(coarsest_size=100, use_graphs=g)
        h = amg.amg_setup(p.rp, p.ci, p.val, p.d, 3, 3, o)
        x = np.zeros(p.n)
        st, it, rr = amg.amg_solve(h, b, x, 1e-8, 2)
        assert st == 0
        xs.append((it, x))
        amg.amg_free(h)
    assert xs[0][0] == xs[1][0] and np.array_equal(xs[0][1], xs[1][1])


def test_edge_cases(amg, gen_mod, oracle_mod):
    # one level only (n <= coarsest): exact solve, 1 iteration
    p = gen_mod.grid2d(8)
    h = amg.amg_setup(p.rp, p.ci, p.val, p.d, 2, 3, amg.amg_options_default(coarsest_size=100))
    b = gen_mod.rhs(p.n, 0)
    x = np.zeros(p.n)
    st, it, rr = amg.amg_solve(h, b, x, 1e-10, 2)
    assert st == 0 and it == 1 and rr < 1e-12
    # zero rhs -> zero solution, 0 iterations
    x = np.ones(p.n)
    st, it, rr = amg.amg_solve(h, np.zeros(p.n), x, 1e-8, 2)
    assert st == 0 and it == 0 and np.all(x == 0)
    # x0 = exact solution -> 0 iterations
    xs = np.linalg.solve(np.diag(np.zeros(p.n)) + _dense(p), b)
    x = xs.copy()
    st, it, rr = amg.amg_solve(h, b, x, 1e-8, 2)
    assert it == 0
    amg.amg_free(h)
    # invalid inputs
    bad = p.val.copy()
    bad[1] = 0.25
    with pytest.raises(amg.AmgError) as e:
        amg.amg_setup(p.rp, p.ci, bad, p.d, 2, 3)
    assert e.value.code == amg.AMG_E_INPUT
    ci = p.ci.copy()
    ci[0], ci[1] = ci[1], ci[0]
    with pytest.raises(amg.AmgError) as e:
        amg.amg_setup(p.rp, ci, p.val, p.d, 2, 3)
    assert e.value.code == amg.AMG_E_INPUT
    with pytest.raises(amg.AmgError) as e:
        amg.amg_setup(p.rp, p.ci, p.val, -p.d, 2, 3)
    assert e.value.code == amg.AMG_E_INPUT
    # stagnation: diagonal-only above the coarsest size
    n = 500
    with pytest.raises(amg.AmgError) as e:
        amg.amg_setup(np.zeros(n + 1, np.int64), np.zeros(0, np.int32), np.zeros(0), np.ones(n), 1, 2,
                      amg.amg_options_default(coarsest_size=10))
    assert e.value.code == amg.AMG_E_SETUP
    # missing diagonals are inserted exactly like the oracle does
    q = gen_mod.random_graph(400, 5, seed=3, weighted=True)
    keep = q.ci != np.repeat(np.arange(q.n), np.diff(q.rp))
    rp = np.concatenate([[0], np.cumsum(np.add.reduceat(keep.astype(np.int64), q.rp[:-1]))]).astype(np.int64)
    hier = oracle_mod.Hierarchy(rp, q.ci[keep], q.val[keep], q.d, 2, 3, coarsest_size=20)
    h = amg.amg_setup(rp, np.ascontiguousarray(q.ci[keep]), np.ascontiguousarray(q.val[keep]), q.d, 2, 3,
                      amg.amg_options_default(coarsest_size=20))
    compare_hierarchy(amg, h, hier, 3, exact_values=True)
    amg.amg_free(h)


def _dense(p):
    A = np.zeros((p.n, p.n))
    for i in range(p.n):
        A[i, p.ci[p.rp[i]:p.rp[i + 1]]] += p.val[p.rp[i]:p.rp[i + 1]]
    return A + np.diag(p.d)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_full_size_hierarchy_and_precond(amg, gen_mod, oracle_mod, name):
    """Full BASELINE size, in the configuration bench.py times: the whole hierarchy bit-exact, one
    B_0(r) within 1e-10, and the solve's iteration count within +-1 of the committed oracle count
    (tests/golden/oracle_iters.json, written by tools/oracle_golden.py from oracle/ only)."""
    p = gen_mod.problem(name)
    hier = oracle_mod.setup_problem(p)
    h = gpu_setup(amg, p)
    try:
        compare_hierarchy(amg, h, hier, p.params["degree"], exact_values=True)
        r = gen_mod.rhs(p.n, 11)
        z = np.empty(p.n)
        amg.amg_level_precond(h, 0, 2, r, z)
        ref = hier.precond(r, nu=2)
        H.assert_close(z, ref, 1e-10)
        b = gen_mod.rhs(p.n, 0)
        x = np.zeros(p.n)
        st, it, rr = amg.amg_solve(h, b, x, 1e-8, 2)
        gold = json.load(open(os.path.join(GOLD, "oracle_iters.json")))
        assert st == 0 and rr <= 1e-8
        assert abs(it - gold[name]["iters"]) <= 1
    finally:
        amg.amg_free(h)


@pytest.mark.parametrize("tail_nnz", [0, 8192, 10**9])
def test_coarse_tail_kernel_parity(amg, gen_mod, oracle_mod, tail_nnz):
    """The coarse-tail kernel (levels with nnz <= tail_nnz run in one single-CTA launch) and the
    per-kernel graph path both match the oracle: B_l(r) <= 1e-10 on every level, same iterations."""
    p = gen_mod.problem("C2", size=160)
    p.params["coarsest_size"] = 40
    hier = oracle_mod.setup_problem(p)
    o = amg.amg_options_default(coarsest_size=40, tail_nnz=tail_nnz)
    h = amg.amg_setup(p.rp, p.ci, p.val, p.d, p.params["passes"], p.params["degree"], o)
    rng = np.random.default_rng(3)
    try:
        for l in range(hier.nlev):
            n = hier.level_info(l)["n"]
            r = rng.uniform(-1, 1, n)
            z = np.empty(n)
            amg.amg_level_precond(h, l, 2, r, z)
            ref = hier.precond(r, nu=2, level=l)
            H.assert_close(z, ref, 1e-10, f"B_{l}(r), tail_nnz={tail_nnz}")
        b = gen_mod.rhs(p.n, 0)
        ref = hier.solve(b, tol=1e-8, nu=2)
        x = np.zeros(p.n)
        st, it, rr = amg.amg_solve(h, b, x, 1e-8, 2)
        assert st == 0 and rr <= 1e-8 and abs(it - ref["iters"]) <= 1
        # nu = 3 also exercises the tail's inner FCG window
        ref3 = hier.solve(b, tol=1e-8, nu=3)
        x = np.zeros(p.n)
        st, it3, _ = amg.amg_solve(h, b, x, 1e-8, 3)
        assert st == 0 and abs(it3 - ref3["iters"]) <= 1
    finally:
        amg.amg_free(h)


def test_smoother_tma_path_parity(amg, gen_mod, oracle_mod):
    """Level 0 of the C3 recipe at 1024^2 (1M rows, compressed SELL, > 9472 slices) runs the TMA-staged
    smoother kernel; one whole smoother application and one B_0(r) against the oracle."""
    p = gen_mod.problem("C3", size=1024)
    hier = oracle_mod.setup_problem(p)
    h = gpu_setup(amg, p)
    try:
        assert amg.amg_get_info(h)["level0_format"] == 2
        rng = np.random.default_rng(3)
        n = p.n
        f = rng.uniform(-1, 1, n)
        x0 = rng.uniform(-1, 1, n)
        x = np.empty(n)
        amg.amg_level_smooth(h, 0, f, x0, x)
        ref = hier.smooth(0, f, x0)
        H.assert_close(x, ref, 1e-12)
        r = rng.uniform(-1, 1, n)
        z = np.empty(n)
        amg.amg_level_precond(h, 0, 2, r, z)
        zr = hier.precond(r, nu=2, level=0)
        H.assert_close(z, zr, 1e-10)
    finally:
        amg.amg_free(h)


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("tail_nnz", [8192, 10 ** 6])
def test_tail_shared_memory_mode_parity(amg, gen_mod, oracle_mod, tail_nnz, mode):
    """The coarse-tail kernel with its vectors in shared memory (opt-in tail_smem) gives the same
    B_0(r) as the oracle and the same iterations; tail_nnz 1e6 puts every level >= 1 of C1 in the tail."""
    p = gen_mod.problem("C1")
    hier = oracle_mod.setup_problem(p)
    o = amg.amg_options_default(coarsest_size=100, tail_nnz=tail_nnz, tail_smem=mode)
    h = amg.amg_setup(p.rp, p.ci, p.val, p.d, 2, 2, o)
    try:
        r = np.random.default_rng(5).uniform(-1, 1, p.n)
        z = np.empty(p.n)
        amg.amg_level_precond(h, 0, 2, r, z)
        ref = hier.precond(r, nu=2, level=0)
        H.assert_close(z, ref, 1e-10)
        b = gen_mod.rhs(p.n, 0)
        x = np.zeros(p.n)
        st, it, rr = amg.amg_solve(h, b, x, 1e-8, 2)
        assert st == 0 and abs(it - hier.solve(b, tol=1e-8, nu=2)["iters"]) <= 1
    finally:
        amg.amg_free(h)


@pytest.mark.parametrize("name", ["C1", "C2s", "C4s", "rgg"])
def test_amli_cycle_parity(amg, gen_mod, oracle_mod, name):
    """Stationary AMLI cycle (cycle=2, reading A23) on the GPU against the
    oracle: B_l(r) on every level (nu = 2, and nu = 3 on level 0) <= 1e-10, linearity, and the
    solve's iteration count within +-1."""
    p = {"C1": lambda: gen_mod.problem("C1"), "C2s": lambda: gen_mod.problem("C2", size=128),
         "C4s": lambda: gen_mod.problem("C4", size=16)}.get(name, None)
    if p is None:
        p = gen_mod.rgg(6000, seed=5)
        p.params = dict(passes=3, degree=3, coarsest_size=50, seed=0)
    else:
        p = p()
    hier = oracle_mod.setup_problem(p, cycle=2)
    prm = p.params
    o = amg.amg_options_default(coarsest_size=prm.get("coarsest_size", 100), seed=prm.get("seed", 0), cycle=2)
    h = amg.amg_setup(p.rp, p.ci, p.val, p.d, prm["passes"], prm["degree"], o)
    rng = np.random.default_rng(2)
    try:
        for l in range(hier.nlev):
            n = hier.level_info(l)["n"]
            r = rng.uniform(-1, 1, n)
            z = np.empty(n)
            amg.amg_level_precond(h, l, 2, r, z)
            ref = hier.precond(r, nu=2, level=l)
            H.assert_close(z, ref, 1e-10, f"AMLI B_{l}(r)")
        r = rng.uniform(-1, 1, p.n)
        z3 = np.empty(p.n)
        amg.amg_level_precond(h, 0, 3, r, z3)
        ref3 = hier.precond(r, nu=3, level=0)
        H.assert_close(z3, ref3, 1e-10, "AMLI nu=3")
        z4 = np.empty(p.n)
        amg.amg_level_precond(h, 0, 3, 2.5 * r, z4)
        H.assert_close(z4, 2.5 * z3, 1e-12, "linear operator")
        b = gen_mod.rhs(p.n, 0)
        x = np.zeros(p.n)
        st, it, rr = amg.amg_solve(h, b, x, 1e-8, 2)
        oref = hier.solve(b, tol=1e-8, nu=2)
        assert st == 0 and rr <= 1e-8 and abs(it - oref["iters"]) <= 1, (it, oref["iters"])
    finally:
        amg.amg_free(h)


@pytest.mark.parametrize("name", ["C1", "rgg"])
def test_lanczos_lambda_parity(amg, gen_mod, oracle_mod, name):
    """Reading A24 (opt-in lanczos_steps): the GPU's Lanczos lambda_1 on every smoothed level matches the
    oracle's to 1e-12 (only the dots' summation order differs), B_0(r) <= 1e-10, iterations +-1."""
    if name == "C1":
        p = gen_mod.problem("C1")
    else:
        p = gen_mod.rgg(20000, seed=7)
        p.params = dict(passes=4, degree=4, coarsest_size=100, seed=0)
    hier = oracle_mod.setup_problem(p, lanczos=10)
    prm = p.params
    o = amg.amg_options_default(coarsest_size=prm.get("coarsest_size", 100), seed=prm.get("seed", 0), lanczos_steps=10)
    h = amg.amg_setup(p.rp, p.ci, p.val, p.d, prm["passes"], prm["degree"], o)
    try:
        for l in range(hier.nlev):
            s = amg.amg_level_sizes(h, l, prm["degree"])
            assert s["lambda1"] == pytest.approx(hier.level_info(l)["lambda1"], rel=1e-12), l
        r = np.random.default_rng(1).uniform(-1, 1, p.n)
        z = np.empty(p.n)
        amg.amg_level_precond(h, 0, 2, r, z)
        ref = hier.precond(r, nu=2, level=0)
        H.assert_close(z, ref, 1e-10)
        b = gen_mod.rhs(p.n, 0)
        x = np.zeros(p.n)
        st, it, rr = amg.amg_solve(h, b, x, 1e-8, 2)
        oref = hier.solve(b, tol=1e-8, nu=2)
        assert st == 0 and abs(it - oref["iters"]) <= 1, (it, oref["iters"])
    finally:
        amg.amg_free(h)


def test_structural_zeros_fe_pattern(amg, oracle_mod):
    """A P1-FE pattern with structural zeros (hypotenuse couplings of the right-triangle mesh, A17) is
    accepted; hierarchy bit-exact and B_0(r) <= 1e-10 against the oracle."""
    N = 48
    n = N * N
    rows = []
    for y in range(N):
        for x in range(N):
            i = y * N + x
            nb = [(i - 1, -1.0)] * (x > 0) + [(i + 1, -1.0)] * (x < N - 1) + [(i - N, -1.0)] * (y > 0) + \
                [(i + N, -1.0)] * (y < N - 1) + [(i - N - 1, 0.0)] * (x > 0 and y > 0) + \
                [(i + N + 1, 0.0)] * (x < N - 1 and y < N - 1)
            rows.append(sorted(nb + [(i, -sum(v for _, v in nb) + (1.0 if x == 0 else 0.0))]))
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    ci = np.array([c for r in rows for c, _ in r], np.int32)
    v = np.array([w for r in rows for _, w in r])
    d = np.zeros(n)
    # the Dirichlet-like term added to the x = 0 diagonals above goes into d instead (Eq. (prob))
    for y in range(N):
        i = y * N
        d[i] = 1.0
        for p in range(rp[i], rp[i + 1]):
            if ci[p] == i:
                v[p] -= 1.0
    hier = oracle_mod.Hierarchy(rp, ci, v, d, 2, 3, coarsest_size=40)
    h = amg.amg_setup(rp, ci, v, d, 2, 3, amg.amg_options_default(coarsest_size=40))
    try:
        compare_hierarchy(amg, h, hier, 3, exact_values=True)
        r = np.random.default_rng(0).uniform(-1, 1, n)
        z = np.empty(n)
        amg.amg_level_precond(h, 0, 2, r, z)
        ref = hier.precond(r, nu=2, level=0)
        H.assert_close(z, ref, 1e-10)
    finally:
        amg.amg_free(h)


def _fe_pattern(N):
    """The P1-FE right-triangle pattern of test_structural_zeros_fe_pattern (5-point values, the two
    hypotenuse couplings stored as structural zeros), Dirichlet-like d on the x = 0 column."""
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
    d = np.zeros(n)
    d[::N] = 1.0
    return rp, ci, v, d


@pytest.mark.parametrize("case", ["C1", "fe96", "rgg"])
@pytest.mark.parametrize("k", [2, 4])
def test_mis_k_parity(amg, gen_mod, oracle_mod, case, k):
    """Reading A25 (opt-in mis_k): the GPU's MIS-k aggregates are bit-exact with the
    oracle's sequential greedy MIS on every level, coarse operators bit-exact (integer-valued inputs),
    B_0(r) <= 1e-10 and iteration counts +-1."""
    if case == "C1":
        p = gen_mod.problem("C1")
        rp, ci, v, d = p.rp, p.ci, p.val, p.d
        m, cs = p.params["degree"], p.params["coarsest_size"]
    elif case == "fe96":
        rp, ci, v, d = _fe_pattern(96)
        m, cs = 4, 100
    else:
        p = gen_mod.rgg(20000, seed=7)
        rp, ci, v, d = p.rp, p.ci, p.val, p.d
        m, cs = 4, 100
    n = len(rp) - 1
    hier = oracle_mod.Hierarchy(rp, ci, v, d, 1, m, coarsest_size=cs, mis_k=k)
    h = amg.amg_setup(rp, ci, v, d, 1, m, amg.amg_options_default(coarsest_size=cs, mis_k=k))
    try:
        compare_hierarchy(amg, h, hier, m, exact_values=True)
        r = np.random.default_rng(3).uniform(-1, 1, n)
        if d is None or not np.any(d):
            r -= r.mean()
        z = np.empty(n)
        amg.amg_level_precond(h, 0, 2, r, z)
        ref = hier.precond(r, nu=2, level=0)
        H.assert_close(z, ref, 1e-10)
        b = gen_mod.rhs(n, 0)
        if d is None or not np.any(d):
            b = b - b.mean()
        x = np.zeros(n)
        st, it, rr = amg.amg_solve(h, b, x, 1e-8, 2)
        oref = hier.solve(b, tol=1e-8, nu=2)
        assert st == 0 and abs(it - oref["iters"]) <= 1, (it, oref["iters"])
    finally:
        amg.amg_free(h)


def test_mis_k_args(amg):
    """mis_k outside [0, 8] is AMG_E_ARG."""
    p_rp = np.array([0, 2, 4], np.int64)
    ci = np.array([0, 1, 0, 1], np.int32)
    v = np.array([1.0, -1.0, -1.0, 1.0])
    with pytest.raises(amg.AmgError) as e:
        amg.amg_setup(p_rp, ci, v, np.ones(2), 1, 2, amg.amg_options_default(mis_k=9))
    assert e.value.code == amg.AMG_E_ARG


def test_smoother_tma_wide_slices_parity(amg, gen_mod, oracle_mod):
    """An RGG level 0 with slices wider than 16 (up to ~27 entries; 1-byte value codes + int16 column
    offsets) and > 9472 slices runs the W = 32 TMA instance: one smoother application, one residual-class
    B_0(r) and the solve's iteration count against the oracle."""
    p = gen_mod.rgg(400000, seed=3)
    rl = np.diff(p.rp)
    assert rl.max() > 16
    hier = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 4, 4, coarsest_size=100)
    h = amg.amg_setup(p.rp, p.ci, p.val, p.d, 4, 4, amg.amg_options_default(coarsest_size=100))
    try:
        assert amg.amg_get_info(h)["level0_format"] == 2
        rng = np.random.default_rng(4)
        n = len(p.rp) - 1
        f = rng.uniform(-1, 1, n)
        x0 = rng.uniform(-1, 1, n)
        x = np.empty(n)
        amg.amg_level_smooth(h, 0, f, x0, x)
        ref = hier.smooth(0, f, x0)
        H.assert_close(x, ref, 1e-12)
        r = rng.uniform(-1, 1, n)
        r -= r.mean()
        z = np.empty(n)
        amg.amg_level_precond(h, 0, 2, r, z)
        zr = hier.precond(r, nu=2, level=0)
        H.assert_close(z, zr, 1e-10)
    finally:
        amg.amg_free(h)


@pytest.mark.parametrize("nu", [1, 3, 16])
def test_kcycle_nu_regimes_parity(amg, gen_mod, oracle_mod, nu):
    """B_0(r) on a 3-level hierarchy for nu = 1 and nu = 16 (the two pinned closed-form regimes of the
    k-cycle, tests/test_oracle_pins.py) and nu = 3, against the oracle to 1e-10."""
    p = gen_mod.grid2d(18)
    hier = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, 2, 3, coarsest_size=30)
    assert hier.nlev == 3
    h = amg.amg_setup(p.rp, p.ci, p.val, p.d, 2, 3, amg.amg_options_default(coarsest_size=30))
    try:
        r = np.random.default_rng(2).standard_normal(p.n)
        z = np.empty(p.n)
        amg.amg_level_precond(h, 0, nu, r, z)
        ref = hier.precond(r, nu=nu, level=0)
        H.assert_close(z, ref, 1e-10)
    finally:
        amg.amg_free(h)


@pytest.mark.parametrize("where", ["host", "device"])
def test_invalid_inputs_above_coarsest(amg, gen_mod, where):
    """Invalid CSR inputs large enough to be coarsened: with host arrays the pattern is checked
    before the overlapped level-0 matching (ranges, order, pattern symmetry), the values after the
    join; every case is AMG_E_INPUT and nothing is left behind (a valid setup follows)."""
    import torch

    p = gen_mod.grid2d(30)
    n = p.n

    def run(rp, ci, v, d):
        if where == "device":
            dev = torch.device("cuda", 0)
            rp, ci, v = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (rp, ci, v))
            d = torch.from_numpy(d).to(dev) if d is not None else None
        return amg.amg_setup(rp, ci, v, d, 2, 3)

    cases = []
    ci = p.ci.copy()
    ci[p.rp[5] + 1] = n + 7  # column out of range
    cases.append((p.rp, ci, p.val, p.d))
    ci = p.ci.copy()
    a0 = p.rp[40]
    ci[a0], ci[a0 + 1] = ci[a0 + 1], ci[a0]  # unsorted row
    cases.append((p.rp, ci, p.val, p.d))
    # asymmetric pattern: drop one off-diagonal entry of row 100 (its transpose stays)
    r0, r1 = p.rp[100], p.rp[101]
    k = next(q for q in range(r0, r1) if p.ci[q] != 100)
    keep = np.ones(len(p.ci), bool)
    keep[k] = False
    rp2 = p.rp.copy()
    rp2[101:] -= 1
    cases.append((rp2, p.ci[keep], p.val[keep], p.d))
    bad = p.val.copy()
    bad[p.rp[7]] = 0.5  # positive off-diagonal (row 7's first entry is off-diagonal)
    cases.append((p.rp, p.ci, bad, p.d))
    cases.append((p.rp, p.ci, p.val, -np.abs(p.d) - 1.0))  # d < 0
    # non-monotone row_ptr: an interior entry far past rp[n], a negative one, a decrease
    for k, val in ((50, 10 ** 9), (50, -5), (51, int(p.rp[49]))):
        rpx = p.rp.copy()
        rpx[k] = val
        cases.append((rpx, p.ci, p.val, p.d))
    for rp, ci_, v, d in cases:
        with pytest.raises(amg.AmgError) as e:
            run(rp, ci_, v, d)
        assert e.value.code == amg.AMG_E_INPUT
    h = run(p.rp, p.ci, p.val, p.d)
    amg.amg_free(h)


def test_smoother_tma_wide_fp64_values_parity(amg, gen_mod, oracle_mod):
    """Wide slices (> 16) with > 256 distinct values (fp64 value stream, int16 column offsets) and
    > 9472 slices: the W = 32 TMA instance with its 2-stage ring.  RGG pattern, random symmetric
    weights; one smoother application and B_0(r) against the oracle."""
    p = gen_mod.rgg(400000, seed=5)
    n = len(p.rp) - 1
    rows = np.repeat(np.arange(n), np.diff(p.rp))
    lo, hi = np.minimum(rows, p.ci).astype(np.uint64), np.maximum(rows, p.ci).astype(np.uint64)
    w = 1.0 + ((lo * np.uint64(2654435761) + hi * np.uint64(40503)) % np.uint64(1000)).astype(np.float64) / 1000.0
    off = rows != p.ci
    v = np.where(off, -w, 0.0)
    diag = np.zeros(n)
    np.add.at(diag, rows[off], w[off])
    v[~off] = diag[rows[~off]]
    d = np.full(n, 0.01)
    hier = oracle_mod.Hierarchy(p.rp, p.ci, v, d, 4, 4, coarsest_size=100)
    h = amg.amg_setup(p.rp, p.ci, v, d, 4, 4, amg.amg_options_default(coarsest_size=100))
    try:
        rng = np.random.default_rng(6)
        f = rng.uniform(-1, 1, n)
        x0 = rng.uniform(-1, 1, n)
        x = np.empty(n)
        amg.amg_level_smooth(h, 0, f, x0, x)
        ref = hier.smooth(0, f, x0)
        H.assert_close(x, ref, 1e-12)
        r = rng.uniform(-1, 1, n)
        z = np.empty(n)
        amg.amg_level_precond(h, 0, 2, r, z)
        zr = hier.precond(r, nu=2, level=0)
        H.assert_close(z, zr, 1e-10)
    finally:
        amg.amg_free(h)


@pytest.mark.parametrize("cfg", ["C3", "C4", "C5"])
@pytest.mark.parametrize("mis_k", [0, 4])
def test_full_size_configs_converge(amg, gen_mod, cfg, mis_k):
    """Every BASELINE config at full size, with the paper's matching (BASELINE) and with MIS-4: all
    level formats and kernel instances they select run, the solve converges to tol and the true
    residual agrees.  Pairwise iteration counts are the oracle's where it was run at full size
    (C3: 33) or the recorded B200 counts (C4 17, C5 78)."""
    import torch

    p = gen_mod.problem(cfg)
    prm = p.params
    dev = torch.device("cuda", 0)
    arrs = [torch.from_numpy(x).to(dev) if x is not None else None for x in (p.rp, p.ci, p.val, p.d)]
    b = torch.from_numpy(gen_mod.rhs(p.n, prm["seed"])).to(dev)
    x = torch.zeros(p.n, dtype=torch.float64, device=dev)
    o = amg.amg_options_default(coarsest_size=prm["coarsest_size"], mis_k=mis_k)
    h = amg.amg_setup(*arrs, prm["passes"], prm["degree"], o)
    try:
        st, it, rr = amg.amg_solve(h, b, x, prm["tol"], prm["k_inner"])
        info = amg.amg_get_info(h)
        assert st == 0 and rr <= prm["tol"]
        assert info["last_true_relres"] <= 2 * prm["tol"]
        if mis_k == 0:
            g = json.load(open(os.path.join(GOLD, "oracle_iters.json")))[cfg]
            assert abs(it - g["iters"]) <= 1, (it, g["iters"])
            # the full-size solution against the oracle's (tools/oracle_golden.py, 4096 evenly spaced
            # rows), element by element
            idx = np.asarray(g["x_sample_idx"], np.int64)
            xs = x[torch.from_numpy(idx).to(dev)].cpu().numpy()
            H.assert_close(xs, np.asarray(g["x_sample"]), 1e-6, f"{cfg} solution samples")
            assert abs(float(torch.linalg.norm(x)) - g["x_norm"]) <= 1e-6 * g["x_norm"]
    finally:
        amg.amg_free(h)


@pytest.mark.parametrize("opts", [dict(compress=0), dict(cycle=2), dict(lanczos_steps=10), dict(use_graphs=0),
                                  dict(tail_smem=0), dict(tail_nnz=0)])
def test_full_size_c3_option_paths(amg, gen_mod, opts):
    """C3 at full size through the other option paths (uncompressed SELL streams, the AMLI cycle, the
    Lanczos lambda_max, eager launches, no tail shared memory, no tail): converges, true residual
    agrees; the options that do not change the arithmetic keep the 33 iterations."""
    import torch

    p = gen_mod.problem("C3")
    prm = p.params
    dev = torch.device("cuda", 0)
    arrs = [torch.from_numpy(x).to(dev) if x is not None else None for x in (p.rp, p.ci, p.val, p.d)]
    b = torch.from_numpy(gen_mod.rhs(p.n, prm["seed"])).to(dev)
    x = torch.zeros(p.n, dtype=torch.float64, device=dev)
    o = amg.amg_options_default(coarsest_size=prm["coarsest_size"], **opts)
    h = amg.amg_setup(*arrs, prm["passes"], prm["degree"], o)
    try:
        st, it, rr = amg.amg_solve(h, b, x, prm["tol"], prm["k_inner"])
        info = amg.amg_get_info(h)
        assert st == 0 and rr <= prm["tol"]
        assert info["last_true_relres"] <= 2 * prm["tol"]
        if not ({"cycle", "lanczos_steps"} & set(opts)):
            assert it == 33
    finally:
        amg.amg_free(h)


def test_zero_rhs_precond_is_zero(amg, gen_mod, oracle_mod):
    """Reading A13: B_l(0) with nu = 2, 3 runs the inner FCG on rho = 0 (d = 0, d.q = 0):
    every level returns exactly 0, no 0/0 -- the launch path and the coarse tail kernel."""
    p = gen_mod.grid2d(64)
    for tail in (0, 8192):
        h = amg.amg_setup(p.rp, p.ci, p.val, p.d, 2, 3, amg.amg_options_default(coarsest_size=10, tail_nnz=tail))
        try:
            L = amg.amg_get_info(h)["levels"]
            assert L >= 4
            for l in range(L - 1):
                n = amg.amg_level_sizes(h, l, 3)["n"]
                for nu in (2, 3):
                    z = np.full(n, np.nan)
                    amg.amg_level_precond(h, l, nu, np.zeros(n), z)
                    assert not np.any(z), (tail, l, nu)
        finally:
            amg.amg_free(h)


@pytest.mark.gpu
@pytest.mark.parametrize("zform", [True, False])
def test_inner_fcg_forms_parity(amg, gen_mod, oracle_mod, monkeypatch, zform):
    """B_l(r) on every level of a 4-level hierarchy with nu = 2, through the z-form inner FCG (the
    default: d_1, q_1 never formed) and through the direct form (AMG_NO_ZFORM,
    read at setup), against the oracle's direct FCG to 1e-10 element-wise."""
    if zform:
        monkeypatch.delenv("AMG_NO_ZFORM", raising=False)
    else:
        monkeypatch.setenv("AMG_NO_ZFORM", "1")
    p = gen_mod.problem("C2", size=128)
    prm = p.params
    hier = oracle_mod.Hierarchy(p.rp, p.ci, p.val, p.d, prm["passes"], prm["degree"], coarsest_size=20)
    h = amg.amg_setup(p.rp, p.ci, p.val, p.d, prm["passes"], prm["degree"], amg.amg_options_default(coarsest_size=20))
    try:
        assert amg.amg_get_info(h)["levels"] == hier.nlev >= 4
        for l in range(hier.nlev - 1):
            n = hier.level_info(l)["n"]
            r = np.random.default_rng(10 + l).standard_normal(n)
            z = np.empty(n)
            amg.amg_level_precond(h, l, 2, r, z)
            H.assert_close(z, hier.precond(r, nu=2, level=l), 1e-10)
    finally:
        amg.amg_free(h)


@pytest.mark.gpu
@pytest.mark.parametrize("restart", [1, 2, 3, 5, 7])
def test_deferred_x_updates_any_window(amg, gen_mod, oracle_mod, restart):
    """The outer FCG defers x += alpha_k d_k (flushed at the window end, or inside the last window
    position's direction kernel for restart 2..5, and at the end of the solve).  Stopping after any
    number of iterations -- mid-window, at a window end, or right after one -- the returned x must
    carry every update exactly once: its true residual equals the recursive one, and at convergence
    x equals the oracle's with the same restart."""
    p = gen_mod.problem("C2", size=200)
    b = gen_mod.rhs(p.n, 3)
    for K in (1, 2, 3, 4, 5, 6, 7, 8, 11):
        o = amg.amg_options_default(coarsest_size=p.params.get("coarsest_size", 100), restart=restart, max_iter=K)
        h = amg.amg_setup(p.rp, p.ci, p.val, p.d, p.params["passes"], p.params["degree"], o)
        try:
            x = np.zeros(p.n)
            st, it, rr = amg.amg_solve(h, b, x, 1e-14, 2)
            info = amg.amg_get_info(h)
            assert it == K and st != 0
            # ||b - A x|| / ||b|| (x from the deferred updates) vs the FCG's recursive ||r_K|| / ||b||
            assert abs(info["last_true_relres"] - rr) <= 1e-9 * max(1.0, rr), (K, info["last_true_relres"], rr)
        finally:
            amg.amg_free(h)
    hier = oracle_mod.setup_problem(p, restart=restart)
    ref = hier.solve(b, tol=1e-8, nu=2)
    h = gpu_setup(amg, p, restart=restart)
    try:
        x = np.zeros(p.n)
        st, it, rr = amg.amg_solve(h, b, x, 1e-8, 2)
        assert st == 0 and abs(it - ref["iters"]) <= 1, (it, ref["iters"])
        H.assert_close(x, ref["x"], 1e-6)
    finally:
        amg.amg_free(h)
