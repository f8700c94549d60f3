"""CPU, world_size 2 (gloo): the row-sharded multi-GPU schedule of the range
finder, executed with numpy on each rank's shard and gloo allreduces exactly
where rfgpu issues its NCCL allreduces (paper_1607_01649_b200/csrc/
rfgpu_api.cu: range_core / orth / pass_tn / small_svd_of_bt), must reproduce
the single-process reference rsvd (reorthonormalised) to 1e-10 in the
singular values. This pins the distributed algorithm (which products are
row-local, which are summed, where CholeskyQR2's R2^-1 is folded) without a
GPU; the CUDA kernels themselves are covered by the -m gpu parity tests.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def shard_rows(m, world, rank):
    """Row partition used by bench.py / the rfgpu handles: contiguous blocks."""
    return m * rank // world, m * (rank + 1) // world


def allreduce(x):
    t = torch.from_numpy(np.ascontiguousarray(x))
    dist.all_reduce(t)
    return t.numpy()


def cholqr2_folded(x_loc):
    """orth(): G1 = sum X^T X; Q1 = X R1^-1; G2 = sum Q1^T Q1; basis Q1 R2^-1."""
    g1 = allreduce(x_loc.T @ x_loc)
    r1 = np.linalg.cholesky(g1).T
    q1 = x_loc @ np.linalg.inv(r1)
    g2 = allreduce(q1.T @ q1)
    r2 = np.linalg.cholesky(g2).T
    return q1, np.linalg.inv(r2), r2 @ r1


def cholqr2_replicated(x):
    r1 = np.linalg.cholesky(x.T @ x).T
    q1 = x @ np.linalg.inv(r1)
    r2 = np.linalg.cholesky(q1.T @ q1).T
    return q1 @ np.linalg.inv(r2), r2 @ r1


def sharded_rsvd(a_loc, g, k, q):
    """rsvd(A, k, p, q, reorthonormalize=true) on a row shard."""
    y = a_loc @ g                                   # pass_nn: row-local
    a_fro2 = allreduce(np.array([np.sum(a_loc * a_loc)]))[0]
    q1, r2i, _ = cholqr2_folded(y)
    for _ in range(q):
        z = allreduce(a_loc.T @ q1) @ r2i           # pass_tn + allreduce, R2^-1 folded
        w, _ = cholqr2_replicated(z)                # replicated n x l orth
        y = a_loc @ w                               # pass_nn
        q1, r2i, _ = cholqr2_folded(y)
    bt = allreduce(a_loc.T @ q1) @ r2i              # B^T = A^T Q
    qb, rb = cholqr2_replicated(bt)                 # small SVD of B via R
    ur, s, vrt = np.linalg.svd(rb)
    ub = vrt.T                                      # left singular vectors of B
    resid2 = a_fro2 - np.sum(bt * bt)
    u_loc = q1 @ (r2i @ ub[:, :k])                  # lift: row-local
    v = qb @ ur[:, :k]
    return u_loc, s[:k], v, resid2


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    from oracle.oracle import get
    port_o = get("port")
    m, n, k, p, q = 600, 240, 20, 10, 1
    a = port_o.planted(m, n, np.arange(1, 241, dtype=np.float64) ** -1.5, 1)
    g = port_o.gaussian(1, "range.G", n, k + p)
    r0, r1 = shard_rows(m, world, rank)
    u_loc, s, v, resid2 = sharded_rsvd(np.asfortranarray(a[r0:r1]), g, k, q)
    # gather U rows on rank 0 for the comparison
    u_all = [torch.zeros((shard_rows(m, world, r)[1] - shard_rows(m, world, r)[0], k), dtype=torch.float64)
             for r in range(world)]
    dist.all_gather(u_all, torch.from_numpy(np.ascontiguousarray(u_loc)))
    if rank == 0:
        want = port_o.rsvd(a, k, p, q, 1, False, True)
        u = np.vstack([t.numpy() for t in u_all])
        sgn = np.sign(np.sum(u * want.U, axis=0))
        out.put({
            "sig_err": float(np.max(np.abs(s - want.D) / want.D)),
            "u_err": float(np.abs(u * sgn - want.U)[:, :10].max()),
            "resid2": float(resid2),
            "resid2_want": float(np.linalg.norm(a) ** 2 - np.sum((want.U * want.D) ** 2)),
            "rows": [shard_rows(m, world, r) for r in range(world)],
        })
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(300)
def test_row_sharded_schedule_matches_reference_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert res["rows"] == [(0, 300), (300, 600)]
    assert res["sig_err"] < 1e-10
    assert res["u_err"] < 1e-8


def test_shard_rows_cover_and_disjoint():
    for m in (1, 7, 1048576):
        for world in (1, 2, 3, 8):
            spans = [shard_rows(m, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
