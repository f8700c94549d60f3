"""One rank of the world-size-2 GPU test (tests/test_gpu_dist_world2.py).

Runs librfgpu's OWN row-sharded code (the `dist` branches of range_core /
orth / svd_tall_dev / single_pass_core, global_rows, the zero-padded gathers
of randomized_id / randomized_cur) with the host-staged reduction backend
(rfgpu_ctx_create_hostsum): every sum over ranks that the NCCL context would
issue goes through a torch.distributed gloo all_reduce instead, so two ranks
can share one B200 (NCCL cannot place two ranks on one device). Each rank
holds a contiguous row block of A, exactly as bench.py shards config 3.

The same process also runs the single-process call on the whole A (a world-1
context) and records the deviation of its rows / replicated outputs; the
parent test asserts the bounds. Test infrastructure only.

usage: python tests/dist_worker.py RANK WORLD PORT OUT_JSON CASE
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rel_sigma(a, b):
    return float(np.max(np.abs(a - b) / np.abs(b))) if len(b) else 0.0


def sign_aligned(x, ref):
    """max |x - ref| after flipping each column of x to ref's sign."""
    if x.size == 0:
        return 0.0
    s = np.sign(np.sum(x * ref, axis=0))
    s[s == 0] = 1.0
    return float(np.max(np.abs(x * s - ref)))


def planted(m, n, sigma, seed, noise=0.0):
    rng = np.random.default_rng(seed)
    r = len(sigma)
    u, _ = np.linalg.qr(rng.standard_normal((m, r)))
    v, _ = np.linalg.qr(rng.standard_normal((n, r)))
    a = (u * sigma) @ v.T
    if noise:
        a += noise * rng.standard_normal((m, n))
    return np.asfortranarray(a)


def main():
    rank, world, port, out, case = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4], sys.argv[5]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=port)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1607_01649_b200 as rf

    calls = {"n": 0}

    def host_sum(buf):
        calls["n"] += 1
        dist.all_reduce(torch.from_numpy(buf))  # in place on the library's pinned staging buffer

    ctx = rf.Context(0, rank, world, host_sum=host_sum)
    solo = rf.Context(0)
    res = {"rank": rank, "case": case}

    m, n = 3001, 640
    r0, r1 = m * rank // world, m * (rank + 1) // world
    if case.startswith("rsvd"):
        # rsvd_reorth_{dmma,digits}, rsvd_plain_{dmma,digits}: power iterations, both orth modes
        os.environ["RFGPU_OZAKI"] = "1" if case.endswith("digits") else "0"
        reorth = "reorth" in case
        a = planted(m, n, 1.0 / np.arange(1, 301) ** 1.5, 7, noise=1e-9)
        dm = rf.DeviceMatrix.upload(ctx, a[r0:r1])
        assert (dm.m, dm.m_global, dm.row0) == (r1 - r0, m, r0), (dm.m, dm.m_global, dm.row0)
        got = rf.rsvd(dm, 40, 12, 1, 5, reorthonormalize=reorth)
        want = rf.rsvd(rf.DeviceMatrix.upload(solo, a), 40, 12, 1, 5, reorthonormalize=reorth)
        res.update(rank_got=len(got.D), rank_want=len(want.D), sigma=rel_sigma(got.D, want.D),
                   V=sign_aligned(got.V, want.V), U_rows=sign_aligned(got.U, want.U[r0:r1]))
        pr = rf.power_range(dm, 40, 12, 1, 5, reorthonormalize=True)
        pw = rf.power_range(rf.DeviceMatrix.upload(solo, a), 40, 12, 1, 5, reorthonormalize=True)
        res.update(range_cols=[pr.Q.shape[1], pw.Q.shape[1]],
                   resid_rel=abs(pr.residual_frob - pw.residual_frob) / pw.residual_frob,
                   B=float(np.max(np.abs(np.abs(pr.B) - np.abs(pw.B)))))
    elif case == "exact_rank":
        # rank-deficient sketch: the distributed Gram-Schmidt fallback with the drop rule
        os.environ["RFGPU_OZAKI"] = "0"
        a = planted(m, n, np.array([5.0, 4.0, 3.0, 2.0, 1.0] * 2) / np.arange(1, 11), 3)
        got = rf.rsvd(rf.DeviceMatrix.upload(ctx, a[r0:r1]), 12, 6, 1, 9)
        want = rf.rsvd(rf.DeviceMatrix.upload(solo, a), 12, 6, 1, 9)
        res.update(rank_got=len(got.D), rank_want=len(want.D), sigma=rel_sigma(got.D[:10], want.D[:10]),
                   U_rows=sign_aligned(got.U[:, :10], want.U[r0:r1, :10]))
    elif case in ("id", "cur"):
        os.environ["RFGPU_OZAKI"] = "0"
        sig = 10.0 ** (-6.0 * np.arange(200) / 199)
        a = planted(m, n, sig, 11)
        if case == "id":
            got = rf.randomized_id(rf.DeviceMatrix.upload(ctx, a[r0:r1]), 60, 10, 1, 3)
            want = rf.randomized_id(rf.DeviceMatrix.upload(solo, a), 60, 10, 1, 3)
            res.update(pivots_equal=bool(np.array_equal(got.Is, want.Is)), X_rows=float(np.max(np.abs(got.X - want.X[r0:r1]))))
        else:
            got = rf.randomized_cur(rf.DeviceMatrix.upload(ctx, a[r0:r1]), 60, 10, 0, 3)
            want = rf.randomized_cur(rf.DeviceMatrix.upload(solo, a), 60, 10, 0, 3)
            res.update(js_equal=bool(np.array_equal(got.Js, want.Js)), is_equal=bool(np.array_equal(got.Is, want.Is)),
                       U=float(np.max(np.abs(got.U - want.U)) / np.max(np.abs(want.U))),
                       cond=[abs(got.cond_C - want.cond_C) / want.cond_C, abs(got.cond_R - want.cond_R) / want.cond_R])
    elif case == "single_pass":
        os.environ["RFGPU_OZAKI"] = "0"
        a = planted(m, n, np.exp(-np.arange(1, 301) / 10.0), 13, noise=1e-8)
        got = rf.single_pass_svd(rf.MatrixStream(a[r0:r1], 96), 20, 20, 17, ctx=ctx, m_global=m)
        want = rf.single_pass_svd(rf.MatrixStream(a, 96), 20, 20, 17, ctx=solo)
        res.update(sigma=rel_sigma(got.D, want.D), V=sign_aligned(got.V, want.V),
                   U_rows=sign_aligned(got.U, want.U[r0:r1]))
    else:
        raise SystemExit(f"unknown case {case}")
    res["host_sums"] = calls["n"]
    json.dump(res, open(out, "w"))
    solo.close()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
