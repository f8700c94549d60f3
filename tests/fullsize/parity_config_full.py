#!/usr/bin/env python
"""One-off full-size parity runs at the BASELINE configurations (GPU box).

For each requested workload: build A with the bench's generator (the reference
recipe planted_matrix + noise, paper_1607_01649_b200/planted.py) on the
device, run the product call on the default path (INT8-digit passes), copy the
SAME bytes to the host and run the compiled, unmodified reference
(oracle/_ref/librfref.so) on all host cores, timed: rsvd for c1-c3, the
column ID of G A for c5 (multiply + id_deterministic, lowrank.cpp:351-357),
the restated single pass for c4 (the reference's own single_pass_svd is
infeasible at k = 300; the port restatement is used).

Writes profiles/r02_parity_<workload>.json (deviations, timings) and merges
the oracle's singular values / pivots into tests/golden/config_golden.json,
which bench.py's self-check reads.

usage: python tests/fullsize/parity_config_full.py c3 [c5 c2 c4 ...]
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (workload table and generator)
import paper_1607_01649_b200 as rf  # noqa: E402
from oracle.oracle import get  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden", "config_golden.json")


def sign_aligned_rows(torch, x, ref):
    s = torch.sign(torch.sum(x * ref, dim=1, keepdim=True))
    s[s == 0] = 1
    return float(torch.max(torch.abs(x * s - ref)))


def residual(torch, at, u, d, v):
    """||A - U diag(d) V^T||_F on the device in row blocks; u (k, m), v (k, n) device."""
    n, m = at.shape
    tot = 0.0
    for r0 in range(0, m, 65536):
        r1 = min(m, r0 + 65536)
        blk = at[:, r0:r1].double().T - (u[:, r0:r1].T * d) @ v
        tot += float(torch.sum(blk * blk))
    return tot ** 0.5


def run(workload, threads):
    import torch
    w = bench.WORKLOADS[workload]
    m, n, k, p, q = w["m"], w["n"], w["k"], w["p"], w["q"]
    ell = k + p
    dev = torch.device("cuda", 0)
    t0 = time.perf_counter()
    at = bench.gen_shard(torch, None, w, 0, m, dev)
    torch.cuda.synchronize()
    out = {"workload": workload, "config": bench.config_of(w, 1, type("A", (), {"workload": workload})()),
           "gen_s": time.perf_counter() - t0, "host_threads": threads}
    ctx = rf.Context(0)
    A = rf.DeviceMatrix.wrap(ctx, at.data_ptr(), m, n, m, f32=bool(w.get("f32")), keep=at)
    ref = get("reference")
    port = get("port")
    ref.set_threads(threads)
    port.set_threads(threads)
    gold = {"source": f"tests/fullsize/parity_config_full.py {workload}: compiled reference (oracle/_ref) on the bench's A, "
                      f"{threads} host threads"}
    if w["kind"] == "rsvd":
        got = rf.rsvd(A, k, p, q, 1, reorthonormalize=True)
        ctx.synchronize()
        a = np.asfortranarray(at.T.cpu().numpy())
        t1 = time.perf_counter()
        want = ref.rsvd(a, k, p, q, 1, False, True)
        out["reference_s"] = time.perf_counter() - t1
        del a
        ug = torch.from_numpy(np.ascontiguousarray(got.U.T)).to(dev)
        uw = torch.from_numpy(np.ascontiguousarray(want.U.T)).to(dev)
        vg = torch.from_numpy(np.ascontiguousarray(got.V.T)).to(dev)
        vw = torch.from_numpy(np.ascontiguousarray(want.V.T)).to(dev)
        res_g = residual(torch, at, ug, torch.from_numpy(got.D).to(dev), vg)
        res_w = residual(torch, at, uw, torch.from_numpy(want.D).to(dev), vw)
        out.update(rank=[len(got.D), len(want.D)],
                   sigma_max_rel=float(np.max(np.abs(got.D - want.D) / want.D)),
                   U_max_abs=sign_aligned_rows(torch, ug, uw), V_max_abs=sign_aligned_rows(torch, vg, vw),
                   residual_gpu=res_g, residual_reference=res_w, residual_rel_diff=abs(res_g - res_w) / res_w)
        out["ok"] = bool(out["sigma_max_rel"] <= 1e-10 and out["residual_rel_diff"] <= 0.01)
        gold["D"] = want.D.tolist()
    elif w["kind"] == "cur":
        y_gpu = rf.row_sketch(A, ell, 1, ctx=ctx)
        idg = rf.id_deterministic(y_gpu, k, ctx=ctx)
        a = np.asfortranarray(at.T.cpu().numpy())
        t1 = time.perf_counter()
        g = ref.gaussian(1, "cur.G", ell, m)
        y_ref = ref.multiply(g, a)
        js, z, tr = ref.id_col(y_ref, k)
        out["reference_s"] = time.perf_counter() - t1
        out.update(Y_max_rel=float(np.max(np.abs(y_gpu - y_ref)) / np.max(np.abs(y_ref))),
                   pivots_equal=bool(np.array_equal(idg.Js, js)), Z_max_abs=float(np.max(np.abs(idg.Z - z))),
                   truncated=bool(tr))
        out["ok"] = bool(out["pivots_equal"] and out["Z_max_abs"] <= 1e-8)
        gold["Js"] = js.tolist()
    else:  # single pass, fp32 A
        gc = torch.from_numpy(rf.gaussian(1, "spsvd.Gc", n, ell).reshape(-1, order="F")).to(dev)
        gr = torch.from_numpy(rf.gaussian(1, "spsvd.Gr", m, ell).reshape(-1, order="F")).to(dev)
        U = torch.empty(m * k, dtype=torch.float64, device=dev)
        D = torch.empty(k, dtype=torch.float64, device=dev)
        V = torch.empty(n * k, dtype=torch.float64, device=dev)
        r = rf._i64()
        rf._check(rf.lib().rfgpu_single_pass_svd_device(ctx.handle, A.handle, rf._vp(gc.data_ptr()),
                                                        rf._vp(gr.data_ptr()), k, ell, rf._vp(U.data_ptr()),
                                                        rf._vp(D.data_ptr()), rf._vp(V.data_ptr()), rf.C.byref(r)))
        ctx.synchronize()
        d = D.cpu().numpy()[: r.value]
        a = np.asfortranarray(at.T.double().cpu().numpy())
        t1 = time.perf_counter()
        want = port.single_pass_svd(a, k, p, 1, block=1024)
        out["reference_s"] = time.perf_counter() - t1
        out["reference_kind"] = "port restatement (oracle/rf_oracle.c single_pass_svd, Sylvester core)"
        rel = np.abs(d - want.D) / want.D
        out.update(sigma_max_rel=float(rel.max()), sigma_rel_at_k=float(rel[-1]))
        out["ok"] = bool(rel.max() <= 1e-4)
        gold["D"] = want.D.tolist()
    A.free()
    ctx.close()
    json.dump(out, open(os.path.join(ROOT, "profiles", f"r02_parity_{workload}.json"), "w"), indent=1)
    allg = json.load(open(GOLDEN)) if os.path.exists(GOLDEN) else {}
    allg[workload] = gold
    json.dump(allg, open(GOLDEN, "w"), indent=0)
    print(json.dumps({k: v for k, v in out.items() if k != "config"}), flush=True)


if __name__ == "__main__":
    for wl in sys.argv[1:]:
        run(wl, os.cpu_count() or 1)
