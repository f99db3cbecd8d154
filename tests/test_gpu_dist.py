"""-m gpu parity of the row-partitioned (multi-GPU) library path against the oracle's decoupled
aggregation (oracle nparts = P, gather_rows as the library, reading A20).

Only one GPU is available per run, so the P ranks are P host threads of this process on the same
device, each with its own handle and an in-process communicator (amg_comm_init_threads): every
exchange synchronises the rank's stream and meets the others at a host barrier -- no kernel waits on
another rank's kernel.  The halo / dot / gather logic, the decoupled matching with global ids, the
distributed Galerkin product and the gathered levels are the same code the NCCL backend runs.

Bars (BASELINE.json north_star): aggregates and coarse sparsity bit-exact (concatenated over the
ranks), coarse values bit-exact (same summation order), one preconditioner application <= 1e-10
relative, solves to tol with iteration counts within +-1 of the oracle.
"""
import threading

import numpy as np
import pytest

import helpers as H

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def amg():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1307_6305_b200 import amg as A

    A.load()
    return A


def run_ranks(amg, P, fn):
    """fn(rank, comm) on P threads (one handle each); returns the per-rank results."""
    import torch

    comms = amg.amg_comm_init_threads(P)
    out, err = [None] * P, [None] * P

    def work(r):
        try:
            torch.cuda.set_device(0)
            out[r] = fn(r, comms[r])
        except BaseException as e:  # noqa: BLE001 -- re-raised below
            err[r] = e

    ts = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for c in comms:
        amg.amg_comm_free(c)
    for e in err:
        if e is not None:
            raise e
    return out


def dist_case(amg, p, P, gather_rows, oracle_mod, nu=2, check_solve=True, exact_values=True, cycle=0,
              overlap=(True,), expect_path=None, global_agg=False):
    """GPU row-partitioned run(s) vs the oracle's nparts = P hierarchy; `overlap` lists the halo
    overlap settings to run (True: interior/boundary split, False: AMG_NO_OVERLAP=1); expect_path:
    required amg_info level0_path bits on every rank (1 = TMA interior kernel, 2 = split)."""
    import os

    res = None
    # global aggregation: the single-GPU rule, i.e. the oracle's nparts = 1
    hier = oracle_mod.setup_problem(p, nparts=1 if global_agg else P, gather_rows=gather_rows, cycle=cycle)
    oref = None
    for ov in overlap:
        if ov:
            os.environ.pop("AMG_NO_OVERLAP", None)
        else:
            os.environ["AMG_NO_OVERLAP"] = "1"
        try:
            res, oref = _dist_case(amg, p, P, gather_rows, hier, nu, check_solve, exact_values, cycle, oref,
                                   global_agg)
        finally:
            os.environ.pop("AMG_NO_OVERLAP", None)
        if expect_path is not None:
            want = expect_path if ov else (expect_path & ~2)
            assert all(r["info"]["level0_path"] == want for r in res), \
                ([r["info"]["level0_path"] for r in res], want, ov)
    return res


def _dist_case(amg, p, P, gather_rows, hier, nu, check_solve, exact_values, cycle, oref, global_agg=False):
    from paper_1307_6305_b200 import dist

    prm = p.params
    m = prm["degree"]
    offs = dist.row_blocks(p.n, P)
    rng = np.random.default_rng(11)
    r0 = rng.uniform(-1, 1, p.n)
    from inputs import gen

    b = gen.rhs(p.n, 0)

    def fn(rank, comm):
        beg, end = offs[rank], offs[rank + 1]
        lrp, lci, lv, ld = dist.local_block(p.rp, p.ci, p.val, p.d, beg, end)
        o = amg.amg_options_default(coarsest_size=prm.get("coarsest_size", 100), seed=prm.get("seed", 0),
                                    gather_rows=gather_rows, cycle=cycle, global_agg=int(global_agg))
        h = amg.amg_setup_dist(comm, p.n, beg, lrp, lci, lv, ld, prm["passes"], m, o)
        try:
            info = amg.amg_get_info(h)
            levels = []
            for l in range(info["levels"]):
                dl = amg.amg_level_dist(h, l)
                rp, ci, v, agg = amg.amg_level_export(h, l, m)
                s = amg.amg_level_sizes(h, l, m)
                levels.append(dict(dist=dl, rp=rp, ci=ci, v=v, agg=agg, lambda1=s["lambda1"]))
            d0 = levels[0]["dist"]["dist"]
            rr = r0[beg:end] if d0 else r0
            z = np.empty_like(rr)
            amg.amg_level_precond(h, 0, nu, np.ascontiguousarray(rr), z)
            res = dict(info=info, levels=levels, z=z)
            if check_solve:
                x = np.zeros(end - beg)
                st, it, rel = amg.amg_solve(h, np.ascontiguousarray(b[beg:end]), x, 1e-8, nu)
                res.update(status=st, iters=it, relres=rel, x=x, true_relres=amg.amg_get_info(h)["last_true_relres"])
            return res
        finally:
            amg.amg_free(h)

    res = run_ranks(amg, P, fn)
    # hierarchy: concatenation of the row-partitioned levels == oracle level; replicated levels equal
    L = res[0]["info"]["levels"]
    assert L == hier.nlev
    assert all(r["info"]["levels"] == L for r in res)
    ndist = sum(1 for lv in res[0]["levels"] if lv["dist"]["dist"])
    assert res[0]["info"]["dist_levels"] == ndist
    for l in range(L):
        orp, oci, ov = hier.level_csr(l)
        oagg = hier.level_agg(l) if l < L - 1 else None
        if res[0]["levels"][l]["dist"]["dist"]:
            # rebase each block's row pointer
            parts, base = [np.zeros(1, np.int64)], 0
            for r in res:
                lrp = r["levels"][l]["rp"]
                parts.append(lrp[1:] + base)
                base += int(lrp[-1])
            rp = np.concatenate(parts)
            ci = np.concatenate([r["levels"][l]["ci"] for r in res])
            v = np.concatenate([r["levels"][l]["v"] for r in res])
            agg = None if oagg is None else np.concatenate([r["levels"][l]["agg"] for r in res])
            assert [r["levels"][l]["dist"]["row_begin"] for r in res] == sorted(
                r["levels"][l]["dist"]["row_begin"] for r in res)
        else:
            rp, ci, v, agg = (res[0]["levels"][l][k] for k in ("rp", "ci", "v", "agg"))
            for r in res[1:]:
                for k in ("rp", "ci", "v"):
                    assert np.array_equal(r["levels"][l][k], res[0]["levels"][l][k]), f"replicated level {l} {k}"
        assert np.array_equal(rp, orp), f"level {l} row_ptr"
        assert np.array_equal(ci, oci), f"level {l} columns"
        if exact_values:
            assert np.array_equal(v, ov), f"level {l} values not bit-exact"
        else:
            assert np.max(np.abs(v - ov)) <= 1e-12 * np.max(np.abs(ov)), f"level {l} values"
        if oagg is not None:
            assert np.array_equal(agg, oagg), f"level {l} aggregates"
        for r in res:
            assert r["levels"][l]["lambda1"] == pytest.approx(hier.level_info(l)["lambda1"], rel=1e-15, abs=0)
    # one preconditioner application
    d0 = res[0]["levels"][0]["dist"]["dist"]
    z = np.concatenate([r["z"] for r in res]) if d0 else res[0]["z"]
    ref = hier.precond(r0, nu=nu, level=0)
    H.assert_close(z, ref, 1e-10, "B_0(r)")
    if check_solve:
        if oref is None:
            oref = hier.solve(b, tol=1e-8, nu=nu)
        x = np.concatenate([r["x"] for r in res])
        its = {r["iters"] for r in res}
        assert len(its) == 1, its  # every rank takes the same decisions
        it = its.pop()
        assert all(r["status"] == 0 and r["relres"] <= 1e-8 for r in res)
        assert res[0]["true_relres"] <= 2e-8
        assert abs(it - oref["iters"]) <= 1, (it, oref["iters"])
        H.assert_close(x, oref["x"], 1e-6)
    return res, oref


def test_dist_c1_two_ranks(amg, gen_mod, oracle_mod):
    p = gen_mod.problem("C1")
    res = dist_case(amg, p, 2, 300, oracle_mod)
    assert res[0]["info"]["dist_levels"] >= 2  # the gather happens below level 1
    dist_case(amg, p, 2, 300, oracle_mod, overlap=(False,))


def test_dist_c1_three_ranks_deep(amg, gen_mod, oracle_mod):
    p = gen_mod.problem("C1")
    dist_case(amg, p, 3, 0, oracle_mod)  # gather_rows 0: row-partitioned down to the coarsest


def test_dist_3d_four_ranks(amg, gen_mod, oracle_mod):
    p = gen_mod.problem("C4", size=14)
    p.params["coarsest_size"] = 30
    dist_case(amg, p, 4, 200, oracle_mod)


def test_dist_weighted_random_graph(amg, gen_mod, oracle_mod):
    p = gen_mod.random_graph(3000, 7, seed=9, weighted=True, dirichlet=True)
    p.params = dict(passes=2, degree=2, coarsest_size=50, seed=0)
    dist_case(amg, p, 3, 400, oracle_mod, exact_values=True)


def test_dist_singular_rgg(amg, gen_mod, oracle_mod):
    p = gen_mod.rgg(12000, seed=7)
    p.params = dict(passes=3, degree=4, coarsest_size=60, seed=0)
    dist_case(amg, p, 2, 1000, oracle_mod)


def test_dist_amli_cycle(amg, gen_mod, oracle_mod):
    """The stationary AMLI cycle on the row-partitioned path (halo-exchanged residual passes of the
    coarse polynomial)."""
    p = gen_mod.problem("C1")
    dist_case(amg, p, 2, 0, oracle_mod, cycle=2)


def test_dist_fully_replicated(amg, gen_mod, oracle_mod):
    """gather_rows > n: level 0 is gathered at setup and every rank solves the whole problem."""
    p = gen_mod.problem("C1")
    res = dist_case(amg, p, 2, 10 ** 9, oracle_mod)
    assert res[0]["info"]["dist_levels"] == 0


@pytest.mark.parametrize("case", ["c1_p2", "c1_p3_deep", "3d_p4", "rand_p3", "rgg_p2", "c2_p4", "c1_p2_amli"])
def test_dist_global_aggregation(amg, gen_mod, oracle_mod, case):
    """global (non-decoupled) aggregation across the ranks -- matching by halo
    rounds over the inter-block edges, aggregates owned by their leader's rank, coarse rows formed
    from members on several ranks, restriction with the remote members' residuals, prolongation from
    the coarse halo.  Every level concatenated over the ranks equals the oracle's single-GPU (nparts
    = 1) hierarchy bit for bit; B_0(r) element-wise <= 1e-10; iterations +-1."""
    if case.startswith("c1"):
        p = gen_mod.problem("C1")
    elif case == "3d_p4":
        p = gen_mod.problem("C4", size=14)
        p.params["coarsest_size"] = 30
    elif case == "rand_p3":
        p = gen_mod.random_graph(3000, 7, seed=9, weighted=True, dirichlet=True)
        p.params = dict(passes=2, degree=2, coarsest_size=50, seed=0)
    elif case == "rgg_p2":
        p = gen_mod.rgg(12000, seed=7)
        p.params = dict(passes=3, degree=4, coarsest_size=60, seed=0)
    else:
        p = gen_mod.problem("C2", size=128)
    P, G = {"c1_p2": (2, 300), "c1_p3_deep": (3, 0), "3d_p4": (4, 200), "rand_p3": (3, 400), "rgg_p2": (2, 1000),
            "c2_p4": (4, 2000), "c1_p2_amli": (2, 0)}[case]
    res = dist_case(amg, p, P, G, oracle_mod, global_agg=True, cycle=2 if case.endswith("amli") else 0,
                    overlap=(True, False) if case == "c2_p4" else (True,))
    assert res[0]["info"]["dist_levels"] >= 1


@pytest.mark.slow
def test_dist_global_aggregation_production_size(amg, gen_mod, oracle_mod):
    """Global aggregation on the production configuration: C3 recipe 2048^2 over 4 ranks (compressed
    level 0, TMA interior views, aggregates crossing the block boundaries): bit-exact hierarchy vs
    the oracle's single-GPU one, B_0(r) element-wise <= 1e-10, iterations +-1."""
    p = gen_mod.problem("C3", size=2048)
    res = dist_case(amg, p, 4, 50000, oracle_mod, global_agg=True, expect_path=3)
    assert all(r["info"]["level0_format"] == 2 for r in res)


@pytest.mark.slow
@pytest.mark.parametrize("case", ["c3_2048_p2", "c3_2048_p4", "c4_128_p2"])
def test_dist_production_size(amg, gen_mod, oracle_mod, case):
    """The configuration every rank runs at P = 8 on C3: level 0 large enough per rank
    to be stored compressed (>= 4M entries) and to take the TMA-staged kernel on its interior slice
    view (>= 9,472 slices) with halo columns outside [0, n) -- C3 recipe 2048^2 at P = 2 and 4, a C4
    slab 128^3 at P = 2.  Hierarchy bit-exact vs the oracle's nparts = P, B_0(r) element-wise
    <= 1e-10, iterations +-1, with the halo overlap on and off."""
    name, size, P = {"c3_2048_p2": ("C3", 2048, 2), "c3_2048_p4": ("C3", 2048, 4),
                     "c4_128_p2": ("C4", 128, 2)}[case]
    p = gen_mod.problem(name, size=size)
    res = dist_case(amg, p, P, 50000, oracle_mod, overlap=(True, False), expect_path=3)
    for r in res:
        assert r["info"]["level0_format"] == 2  # compressed SELL streams
        assert r["info"]["dist_levels"] >= 2


def test_dist_single_rank_matches_single_gpu(amg, gen_mod):
    """P = 1 through the distributed entry point == amg_setup (same kernels, bitwise)."""
    p = gen_mod.problem("C2", size=128)
    from inputs import gen

    b = gen.rhs(p.n, 0)
    o = amg.amg_options_default(coarsest_size=1000, gather_rows=0)
    h = amg.amg_setup(p.rp, p.ci, p.val, p.d, 3, 3, o)
    x1 = np.zeros(p.n)
    st1, it1, _ = amg.amg_solve(h, b, x1, 1e-8, 2)
    amg.amg_free(h)

    def fn(rank, comm):
        hd = amg.amg_setup_dist(comm, p.n, 0, p.rp, p.ci, p.val, p.d, 3, 3, o)
        x = np.zeros(p.n)
        st, it, _ = amg.amg_solve(hd, b, x, 1e-8, 2)
        amg.amg_free(hd)
        return st, it, x

    st2, it2, x2 = run_ranks(amg, 1, fn)[0]
    assert st1 == st2 == 0 and it1 == it2
    H.assert_close(x2, x1, 1e-12)


def test_dist_bad_blocks_fail_on_every_rank(amg, gen_mod):
    """Blocks that do not tile [0, n) are rejected collectively (no rank hangs)."""
    p = gen_mod.problem("C1")
    from paper_1307_6305_b200 import dist

    def fn(rank, comm):
        beg, end = (0, 2000) if rank == 0 else (2100, p.n)  # gap [2000, 2100)
        lrp, lci, lv, ld = dist.local_block(p.rp, p.ci, p.val, p.d, beg, end)
        try:
            amg.amg_setup_dist(comm, p.n, beg, lrp, lci, lv, ld, 2, 2, amg.amg_options_default())
        except amg.AmgError as e:
            return e.code
        return 0

    assert run_ranks(amg, 2, fn) == [amg.AMG_E_ARG, amg.AMG_E_ARG]


def test_dist_non_monotone_row_ptr_fails_on_every_rank(amg, gen_mod, oracle_mod):
    """A rank's row_ptr with an interior entry past its nnz is AMG_E_INPUT on every rank,
    without an out-of-bounds read (the next setup on the same device works)."""
    p = gen_mod.problem("C1")
    from paper_1307_6305_b200 import dist

    offs = dist.row_blocks(p.n, 2)

    def fn(rank, comm):
        lrp, lci, lv, ld = dist.local_block(p.rp, p.ci, p.val, p.d, offs[rank], offs[rank + 1])
        if rank == 1:
            lrp = lrp.copy()
            lrp[7] = 10 ** 9
        try:
            amg.amg_setup_dist(comm, p.n, offs[rank], lrp, lci, lv, ld, 2, 2, amg.amg_options_default())
        except amg.AmgError as e:
            return e.code
        return 0

    assert run_ranks(amg, 2, fn) == [amg.AMG_E_INPUT, amg.AMG_E_INPUT]
    dist_case(amg, p, 2, 300, oracle_mod, check_solve=False)


def test_nccl_one_rank_matches_single_gpu(amg, gen_mod):
    """The NCCL backend (dlopen'd libnccl, grouped send/recv, allgather, CUDA-graph capture of the
    exchanges) on a one-rank communicator: bitwise the single-GPU result."""
    p = gen_mod.problem("C2", size=160)
    from inputs import gen

    b = gen.rhs(p.n, 0)
    o = amg.amg_options_default(coarsest_size=1000, gather_rows=0)
    h = amg.amg_setup(p.rp, p.ci, p.val, p.d, 3, 3, o)
    x1 = np.zeros(p.n)
    st1, it1, _ = amg.amg_solve(h, b, x1, 1e-8, 2)
    amg.amg_free(h)
    uid = amg.amg_comm_unique_id()
    comm = amg.amg_comm_init_nccl(uid, 1, 0)
    try:
        assert amg.amg_comm_rank(comm) == (0, 1)
        hd = amg.amg_setup_dist(comm, p.n, 0, p.rp, p.ci, p.val, p.d, 3, 3, o)
        info = amg.amg_get_info(hd)
        assert info["nranks"] == 1 and info["dist_levels"] >= 1
        x2 = np.zeros(p.n)
        st2, it2, _ = amg.amg_solve(hd, b, x2, 1e-8, 2)
        x3 = np.zeros(p.n)
        amg.amg_solve(hd, b, x3, 1e-8, 2)  # replay of the captured graphs
        amg.amg_free(hd)
    finally:
        amg.amg_comm_free(comm)
    assert st1 == st2 == 0 and it1 == it2
    H.assert_close(x2, x1, 1e-12)
    assert np.array_equal(x2, x3)
