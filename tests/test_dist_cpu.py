"""CPU (gloo, world_size 2) tests of the host logic of the row-partitioned path.

No GPU: the library's host-only halo planner (amg_halo_plan, the code amg_setup_dist runs) is driven
by two real processes that exchange their requests and halo values over torch.distributed/gloo, and
the resulting block SpMV with relative columns is checked against the global SpMV.  Also covers the
unique-id broadcast the NCCL communicator bootstrap uses and the row-block partition helpers.
"""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _body(rank, world, case)))
    except BaseException as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _problem(case):
    from inputs import gen

    if case == "grid":
        return gen.problem("C1", size=17)
    return gen.random_graph(300, 6, seed=5, weighted=True, dirichlet=True)


def _body(rank, world, case):
    import torch
    import torch.distributed as dist

    from paper_1307_6305_b200 import amg
    from paper_1307_6305_b200 import dist as pdist

    p = _problem(case)
    offs = pdist.row_blocks(p.n, world)
    beg, end = offs[rank], offs[rank + 1]
    lrp, lci, lv, _ = pdist.local_block(p.rp, p.ci, p.val, p.d, beg, end)
    n = end - beg
    halo = np.unique(lci[(lci < beg) | (lci >= end)]).astype(np.int32)
    segs, nlo = amg.amg_halo_plan(beg, n, np.array(offs, np.int64), rank, halo)
    # every segment is one owner's contiguous run; below the block first
    assert nlo == int(np.sum(halo < beg))
    assert sum(c for _, _, c in segs) == len(halo)
    # requests per owner from the plan, exchanged over gloo
    req = {q: [] for q in range(world)}
    k = 0
    for peer, off, cnt in segs:
        run = halo[k:k + cnt]
        assert np.all((run >= offs[peer]) & (run < offs[peer + 1])) and peer != rank
        assert off == (k - nlo if k < nlo else n + (k - nlo))
        req[peer] = run.tolist()
        k += cnt
    allreq = [None] * world
    dist.all_gather_object(allreq, req)
    # the values each owner sends = its x at the requested rows; receive into [halo lo | own | halo hi]
    xg = np.sin(np.arange(p.n) * 0.37)  # global vector (each rank only reads its own block of it)
    x_own = xg[beg:end].copy()
    send = {q: torch.from_numpy(x_own[np.array(allreq[q][rank], dtype=np.int64) - beg].copy())
            for q in range(world) if q != rank and allreq[q][rank]}
    ext = np.zeros(nlo + n + (len(halo) - nlo))
    ext[nlo:nlo + n] = x_own
    ops = []
    for q, t in send.items():
        ops.append(dist.P2POp(dist.isend, t, q))
    bufs = []
    for peer, off, cnt in segs:
        t = torch.empty(cnt, dtype=torch.float64)
        bufs.append((off, t))
        ops.append(dist.P2POp(dist.irecv, t, peer))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    for off, t in bufs:
        ext[nlo + off:nlo + off + t.numel()] = t.numpy()
    # relative columns (the library's k_to_rel) and the block SpMV
    rel = np.where((lci >= beg) & (lci < end), lci - beg, 0)
    pos = np.searchsorted(halo, lci)
    rel = np.where(lci < beg, pos - nlo, rel)
    rel = np.where(lci >= end, n + (pos - nlo), rel)
    y = np.zeros(n)
    for i in range(n):
        s = slice(lrp[i], lrp[i + 1])
        y[i] = np.dot(lv[s], ext[nlo + rel[s]])
    full = np.array([np.dot(p.val[p.rp[i]:p.rp[i + 1]], xg[p.ci[p.rp[i]:p.rp[i + 1]]]) for i in range(beg, end)])
    assert np.allclose(y, full, rtol=0, atol=1e-13)
    # NCCL bootstrap plumbing: rank 0's 128-byte id reaches every rank unchanged
    uid = bytes(range(128)) if rank == 0 else None
    got = pdist.torch_broadcast_bytes(uid)
    assert got == bytes(range(128))
    return "ok"


@pytest.mark.parametrize("case", ["grid", "random"])
def test_halo_plan_two_ranks_gloo(case):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = dict(q.get(timeout=240) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    assert out == {0: "ok", 1: "ok"}, out


def test_row_blocks_and_local_block(gen_mod):
    from paper_1307_6305_b200 import dist as pdist

    assert pdist.row_blocks(10, 3) == [0, 3, 6, 10]
    with pytest.raises(ValueError):
        pdist.row_blocks(2, 3)
    p = gen_mod.problem("C1", size=9)
    offs = pdist.row_blocks(p.n, 4)
    parts = [pdist.local_block(p.rp, p.ci, p.val, p.d, offs[b], offs[b + 1]) for b in range(4)]
    assert np.array_equal(np.concatenate([x[1] for x in parts]), p.ci)
    assert np.array_equal(np.concatenate([x[2] for x in parts]), p.val)
    assert np.array_equal(np.concatenate([x[3] for x in parts]), p.d)
    assert all(x[0][0] == 0 for x in parts)


def test_halo_plan_argument_errors():
    from paper_1307_6305_b200 import amg

    with pytest.raises(amg.AmgError):  # unsorted ids
        amg.amg_halo_plan(0, 4, np.array([0, 4, 8], np.int64), 0, np.array([6, 5], np.int32))
    with pytest.raises(amg.AmgError):  # a "halo" id inside the own block
        amg.amg_halo_plan(0, 4, np.array([0, 4, 8], np.int64), 0, np.array([2], np.int32))
    segs, nlo = amg.amg_halo_plan(4, 4, np.array([0, 4, 8, 12], np.int64), 1, np.array([1, 3, 8, 9], np.int32))
    assert nlo == 2 and segs == [(0, -2, 2), (2, 4, 2)]


def test_bench_launcher_guards():
    """bench.py --gpus N > 1 outside torchrun re-executes itself as N ranks; with fewer visible
    GPUs (none here) it exits 2 with a JSON error instead of silently running one rank, and under a
    launcher whose WORLD_SIZE differs from --gpus it exits 2 as well (the driver calls
    python bench.py --gpus N)."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 2, (r.returncode, r.stdout, r.stderr)
    assert "error" in json.loads(r.stdout.strip().splitlines()[-1])
    env["WORLD_SIZE"] = "4"
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2"], capture_output=True,
                       text=True, env=env, timeout=300)
    assert r.returncode == 2 and "WORLD_SIZE" in r.stdout
