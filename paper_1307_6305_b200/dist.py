"""Row-partition helpers of the multi-GPU path (argument marshalling only).

* ``row_blocks(n, P)``   -- block offsets floor(b n / P), the partition of reading A20 (SURVEY
                            8(c) O1), so parity runs compare like with like.
* ``local_block(...)``   -- this rank's rows of a global CSR, columns kept GLOBAL (the input of
                            amg_setup_dist).
* ``nccl_comm(...)``     -- the library's NCCL communicator for a torch.distributed job: rank 0 asks
                            the library for an NCCL unique id, torch.distributed broadcasts the 128
                            bytes (plumbing), every rank calls amg_comm_init_nccl.
"""
from __future__ import annotations

import numpy as np

from . import amg


def row_blocks(n: int, P: int) -> list[int]:
    """offs[b] = floor(b n / P), b = 0..P (block b = rows [offs[b], offs[b+1]))."""
    if P < 1 or n < P:
        raise ValueError("need 1 <= P <= n")
    return [(b * n) // P for b in range(P + 1)]


def local_block(rp, ci, val, d, beg: int, end: int):
    """Rows [beg, end) of a CSR (int64 row_ptr rebased to 0, int32 GLOBAL columns, fp64 values) and d."""
    rp = np.asarray(rp, dtype=np.int64)
    p0, p1 = int(rp[beg]), int(rp[end])
    lrp = np.ascontiguousarray(rp[beg:end + 1] - p0)
    lci = np.ascontiguousarray(np.asarray(ci, dtype=np.int32)[p0:p1])
    lv = np.ascontiguousarray(np.asarray(val, dtype=np.float64)[p0:p1])
    ld = None if d is None else np.ascontiguousarray(np.asarray(d, dtype=np.float64)[beg:end])
    return lrp, lci, lv, ld


def nccl_comm(rank: int, world: int, broadcast_bytes):
    """NCCL communicator of this rank.  ``broadcast_bytes(buf: bytes | None) -> bytes`` moves rank 0's
    unique id to every rank (e.g. a torch.distributed broadcast of a uint8 tensor)."""
    uid = amg.amg_comm_unique_id() if rank == 0 else None
    uid = broadcast_bytes(uid)
    return amg.amg_comm_init_nccl(uid, world, rank)


def torch_broadcast_bytes(buf: bytes | None, device=None) -> bytes:
    """broadcast_bytes over the default torch.distributed process group (rank 0 is the source)."""
    import torch
    import torch.distributed as dist

    t = torch.zeros(amg.AMG_COMM_ID_BYTES, dtype=torch.uint8, device=device)
    if buf is not None:
        t.copy_(torch.frombuffer(bytearray(buf), dtype=torch.uint8))
    dist.broadcast(t, src=0)
    return bytes(t.cpu().numpy().tobytes())
