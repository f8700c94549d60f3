"""CPU, world_size 2 (gloo): the row-sharded multi-GPU schedules of
randomized_id, randomized_cur and single_pass_svd, executed with numpy on each
rank's row shard with gloo allreduces exactly where rfgpu issues its NCCL
allreduces (paper_1607_01649_b200/csrc/rfgpu_api.cu: rfgpu_randomized_id,
rfgpu_randomized_cur, single_pass_core / svd_tall_dev with dist = true). The
replicated column-ID steps run the oracle's own col_id_core
(lowrank.cpp:51-70), so pivots must match the single-process reference
exactly; X, U and the singular values to 1e-10.

What each schedule sums over ranks (everything else is row-local or
replicated):
  ID   A^T Y per power step (n x l); Y^T assembled from zero-padded columns
       (l x m) for the replicated CPQR.
  CUR  Y = G A (l x n); C = A(:, Js) assembled from zero-padded rows
       (m x k); R = A(Is, :) assembled from the owning ranks (k x n).
  SP   Yr = A^T Gr (n x l); the two CholeskyQR2 Grams of Yc (l x l);
       P = Gr^T Qc (l x k); F = Qc^T Yc (k x l).
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
    return m * rank // world, m * (rank + 1) // world


def allreduce(x):
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    dist.all_reduce(t)
    return t.numpy()


def gather_rows(x_loc, m, world):
    parts = [torch.zeros((shard_rows(m, world, r)[1] - shard_rows(m, world, r)[0], x_loc.shape[1]),
                         dtype=torch.float64) for r in range(world)]
    dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(x_loc)))
    return np.vstack([p.numpy() for p in parts])


def sharded_id(port, a_loc, m, r0, k, p, q, seed):
    ell = k + p
    g = port.gaussian(seed, "rid.G", a_loc.shape[1], ell)
    y = a_loc @ g
    for _ in range(q):
        z = allreduce(a_loc.T @ y)
        y = a_loc @ z
    yt = np.zeros((ell, m))
    yt[:, r0:r0 + a_loc.shape[0]] = y.T
    yt = allreduce(yt)
    is_, zt, _ = port.id_col(yt, k)
    return is_, zt[:, r0:r0 + a_loc.shape[0]].T


def sharded_cur(port, a_loc, m, r0, k, p, seed):
    ell = k + p
    n = a_loc.shape[1]
    g = port.gaussian(seed, "cur.G", ell, m)
    y = allreduce(g[:, r0:r0 + a_loc.shape[0]] @ a_loc)
    js, z, _ = port.id_col(y, k)
    c = np.zeros((m, len(js)))
    c[r0:r0 + a_loc.shape[0]] = a_loc[:, js]
    c = allreduce(c)
    is_, _, _ = port.id_col(c.T, len(js))
    r = np.zeros((len(is_), n))
    for i, gi in enumerate(is_):
        if r0 <= gi < r0 + a_loc.shape[0]:
            r[i] = a_loc[gi - r0]
    r = allreduce(r)
    u = np.linalg.lstsq(r.T, z.T, rcond=None)[0].T  # least_squares(R^T, Z^T)^T
    return js, is_, u


def dist_tall_svd(x_loc):
    """svd_tall_dev(dist=true) fast path: CholeskyQR2 with summed Grams, SVD of R."""
    r1 = np.linalg.cholesky(allreduce(x_loc.T @ x_loc)).T
    q1 = x_loc @ np.linalg.inv(r1)
    r2 = np.linalg.cholesky(allreduce(q1.T @ q1)).T
    ur, s, _ = np.linalg.svd(r2 @ r1)
    return q1 @ np.linalg.inv(r2) @ ur, s


def sharded_single_pass(port, a_loc, m, r0, k, p, seed):
    ell = k + p
    n = a_loc.shape[1]
    gc = port.gaussian(seed, "spsvd.Gc", n, ell)
    gr = port.gaussian(seed, "spsvd.Gr", m, ell)[r0:r0 + a_loc.shape[0]]
    yc = a_loc @ gc
    yr = allreduce(a_loc.T @ gr)
    qc, _ = dist_tall_svd(yc)
    qc = qc[:, :k]
    qr = np.linalg.svd(yr, full_matrices=False)[0][:, :k]
    P = allreduce(gr.T @ qc)
    E = yr.T @ qr
    W = qr.T @ gc
    F = allreduce(qc.T @ yc)
    # P^T P C + C W W^T = P^T E + F W^T in the eigenbases of P^T P and W W^T
    sp, vp = np.linalg.svd(P, full_matrices=False)[1:]
    sw, vw = np.linalg.svd(W.T, full_matrices=False)[1:]
    vp, vw = vp.T, vw.T
    rhs = P.T @ E + F @ W.T
    ct = (vp.T @ rhs @ vw) / (sp[:, None] ** 2 + sw[None, :] ** 2)
    c = vp @ ct @ vw.T
    return np.linalg.svd(c, compute_uv=False)


def _worker(rank, world, port_no, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    from oracle.oracle import get
    port = get("port")
    res = {}
    # ---- randomized_id
    m, n, k, p, q = 500, 300, 25, 10, 1
    a = port.planted(m, n, 0.85 ** np.arange(300, dtype=np.float64), 3)
    r0, r1 = shard_rows(m, world, rank)
    is_, x_loc = sharded_id(port, np.asfortranarray(a[r0:r1]), m, r0, k, p, q, 4)
    x = gather_rows(x_loc, m, world)
    # ---- randomized_cur
    mc, nc, kc, pc = 400, 350, 30, 10
    ac = port.planted(mc, nc, 10.0 ** (-6.0 * np.arange(300) / 299.0), 2)
    c0, c1 = shard_rows(mc, world, rank)
    js, is_c, u = sharded_cur(port, np.asfortranarray(ac[c0:c1]), mc, c0, kc, pc, 1)
    # ---- single_pass_svd
    ms, ns, ks, ps = 360, 280, 12, 8
    as_ = port.planted(ms, ns, 0.8 ** np.arange(280, dtype=np.float64), 5)
    s0, s1 = shard_rows(ms, world, rank)
    d = sharded_single_pass(port, np.asfortranarray(as_[s0:s1]), ms, s0, ks, ps, 6)
    if rank == 0:
        want_is, want_x, _ = port.randomized_id(a, k, p, q, 4)
        want_c = port.randomized_cur(ac, kc, pc, 0, 1)
        want_s = port.single_pass_svd(as_, ks, ps, 6)
        res["id_pivots"] = bool(np.array_equal(is_, want_is))
        res["id_x_err"] = float(np.abs(x - want_x).max())
        res["cur_js"] = bool(np.array_equal(js, want_c.Js))
        res["cur_is"] = bool(np.array_equal(is_c, want_c.Is))
        res["cur_u_err"] = float(np.abs(u - want_c.U).max() / np.abs(want_c.U).max())
        res["sp_err"] = float(np.max(np.abs(d[:ks] - want_s.D) / want_s.D))
        out.put(res)
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(300)
def test_row_sharded_lowrank_schedules_match_reference_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_no, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert res["id_pivots"], res
    assert res["id_x_err"] < 1e-10, res
    assert res["cur_js"] and res["cur_is"], res
    assert res["cur_u_err"] < 1e-8, res
    assert res["sp_err"] < 1e-10, res
