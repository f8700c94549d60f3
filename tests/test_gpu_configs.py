"""GPU parity at the BASELINE configuration sizes, on the DEFAULT path (the FP64
passes over A run as INT8 digit products on tcgen05 whenever m n >= 2^26,
which every config below is).

A is the reference fixture recipe (planted_matrix, diagnostics.cpp:124-136,
built by paper_1607_01649_b200/planted.py, pinned to the compiled reference by
tests/test_planted.py), generated once on the device; the oracle (test
infrastructure) gets the same bytes on the host.

* C5 at full size (32768^2, r = 1000, s_j = 10^(-6(j-1)/999), k = 300, p = 20):
  the GPU's own row sketch Y = G A (digit path) -> device CPQR column ID and the
  full randomized_cur, against the oracle's Y = multiply(G, A) and
  col_id_core (lowrank.cpp:51-70, :351-357): pivots IDENTICAL, Z within 1e-8.
* C2 at full size (20000 x 10000, q = 2) and C3/16 (65536 x 4096, q = 1),
  reorthonormalised, against the oracle rsvd (lowrank.cpp:74-96): singular
  values 1e-10 relative, residual ||A - U S V^T||_F within 1% of the
  oracle's, U and V sign-aligned within 1e-9; C3/16 also through the
  host-matrix call (rfgpu_rsvd_host: A streamed in row panels behind pass 1).
* C4 at 16384^2, k = 300, p = 30, FP32 A (4-digit path):
  singular values within the north star's FP32 bar 1e-4 of the restated
  single-pass oracle (lowrank.cpp:160-220 + the Sylvester core), the margin at
  j = k reported.

Every test prints its measured deviations (`-s` shows them); DESIGN.md §3
lists the results. The full-size C3 comparison is a one-off
(tools/parity_c3_full.py -> profiles/r02_parity_c3.json).
"""
import json
import os

import numpy as np
import pytest

import paper_1607_01649_b200 as rf
from paper_1607_01649_b200 import planted as pl

pytestmark = pytest.mark.gpu


def device_planted(m, n, spec, r, noise, f32=False):
    import torch
    at = pl.planted_matrix(m, n, pl.spectrum(spec, r), 1, noise=noise, device="cuda")
    if f32:
        at = at.float().contiguous()
    torch.cuda.synchronize()
    return at


def host_copy(at):
    """The same bytes as a column-major (m, n) float64 numpy array (At is n x m row-major)."""
    return np.asfortranarray(at.double().cpu().numpy().T)


def sign_aligned(x, ref):
    s = np.sign(np.sum(x * ref, axis=0))
    s[s == 0] = 1.0
    return float(np.max(np.abs(x * s - ref)))


def residual(at, f):
    """||A - U diag(D) V^T||_F on the device, in row blocks."""
    import torch
    n, m = at.shape
    u = torch.from_numpy(np.ascontiguousarray(f.U)).cuda()
    v = torch.from_numpy(np.ascontiguousarray(f.V)).cuda()
    d = torch.from_numpy(f.D).cuda()
    tot = 0.0
    for r0 in range(0, m, 65536):
        r1 = min(m, r0 + 65536)
        blk = at[:, r0:r1].double().T - (u[r0:r1] * d) @ v.T
        tot += float(torch.sum(blk * blk))
    return tot ** 0.5


def report(name, **kv):
    print(f"[config parity] {name}: " + json.dumps(kv), flush=True)


def check_rsvd(ctx, port, at, k, p, q, name, host_call=False):
    n, m = at.shape
    a = host_copy(at)
    want = port.rsvd(a, k, p, q, 1, False, True)
    dm = rf.DeviceMatrix.wrap(ctx, at.data_ptr(), m, n, m, keep=at)
    got = rf.rsvd(dm, k, p, q, 1, reorthonormalize=True)
    sig = float(np.max(np.abs(got.D - want.D) / want.D))
    res_g, res_w = residual(at, got), residual(at, want)
    du, dv = sign_aligned(got.U, want.U), sign_aligned(got.V, want.V)
    out = dict(sigma_max_rel=sig, residual_gpu=res_g, residual_oracle=res_w,
               residual_rel_diff=abs(res_g - res_w) / res_w, U_max_abs=du, V_max_abs=dv)
    assert len(got.D) == len(want.D) == k
    assert sig <= 1e-10
    assert abs(res_g - res_w) <= 0.01 * res_w
    assert du <= 1e-9 and dv <= 1e-9
    if host_call:  # the drop-in's host-matrix call: A streamed in row panels behind pass 1
        gh = rf.rsvd(a, k, p, q, 1, reorthonormalize=True, ctx=ctx)
        out.update(host_sigma_max_rel=float(np.max(np.abs(gh.D - want.D) / want.D)),
                   host_U_max_abs=sign_aligned(gh.U, want.U))
        assert out["host_sigma_max_rel"] <= 1e-10 and out["host_U_max_abs"] <= 1e-9
    dm.free()
    report(name, **out)


def test_c2_full_size_rsvd(ctx, port):
    at = device_planted(20000, 10000, "exp20", 500, 1e-6)
    check_rsvd(ctx, port, at, 100, 10, 2, "C2 20000x10000 k=100 p=10 q=2")


def test_c3_sixteenth_rsvd(ctx, port):
    at = device_planted(65536, 4096, "pow1.5", 1024, 1e-8)
    check_rsvd(ctx, port, at, 200, 20, 1, "C3/16 65536x4096 k=200 p=20 q=1", host_call=True)


def test_c5_full_size_column_id_pivots_exact(ctx, port):
    m = n = 32768
    k, p = 300, 20
    at = device_planted(m, n, "decade6", 1000, 0.0)
    dm = rf.DeviceMatrix.wrap(ctx, at.data_ptr(), m, n, m, keep=at)
    y_gpu = rf.row_sketch(dm, k + p, 1, ctx=ctx)               # G A on the digit path
    idg = rf.id_deterministic(y_gpu, k, ctx=ctx)               # device CPQR + Z
    cur = rf.randomized_cur(dm, k, p, 0, 1, ctx=ctx)           # the whole call (its own sketch)
    dm.free()
    a = host_copy(at)
    del at
    g = port.gaussian(1, "cur.G", k + p, m)
    y_ref = port.multiply(g, a)                                # the reference's sketch
    del a
    js_ref, z_ref, tr = port.id_col(y_ref, k)
    js_on_gpu_y, _, _ = port.id_col(y_gpu, k)                  # oracle CPQR on the GPU's sketch
    out = dict(Y_max_rel=float(np.max(np.abs(y_gpu - y_ref)) / np.max(np.abs(y_ref))),
               pivots_equal_sketch_id=bool(np.array_equal(idg.Js, js_ref)),
               pivots_equal_cur=bool(np.array_equal(cur.Js, js_ref)),
               pivots_equal_oracle_on_gpu_y=bool(np.array_equal(js_on_gpu_y, js_ref)),
               Z_max_abs=float(np.max(np.abs(idg.Z - z_ref))), truncated=bool(tr),
               cond_C=cur.cond_C, cond_R=cur.cond_R)
    report("C5 32768^2 k=300 p=20", **out)
    assert not tr and len(js_ref) == k
    assert out["pivots_equal_sketch_id"] and out["pivots_equal_cur"]
    assert out["Z_max_abs"] <= 1e-8


def test_c4_16384_single_pass_fp32(ctx, port):
    import torch
    m = n = 16384
    k, p = 300, 30
    at = device_planted(m, n, "exp100", 2000, 1e-4, f32=True)
    ell = k + p
    gc = torch.from_numpy(rf.gaussian(1, "spsvd.Gc", n, ell).reshape(-1, order="F")).cuda()
    gr = torch.from_numpy(rf.gaussian(1, "spsvd.Gr", m, ell).reshape(-1, order="F")).cuda()
    U = torch.empty(m * k, dtype=torch.float64, device="cuda")
    D = torch.empty(k, dtype=torch.float64, device="cuda")
    V = torch.empty(n * k, dtype=torch.float64, device="cuda")
    dm = rf.DeviceMatrix.wrap(ctx, at.data_ptr(), m, n, m, f32=True, keep=at)
    r = rf._i64()
    L = rf.lib()
    rf._check(L.rfgpu_single_pass_svd_device(ctx.handle, dm.handle, rf._vp(gc.data_ptr()), rf._vp(gr.data_ptr()), k,
                                             ell, rf._vp(U.data_ptr()), rf._vp(D.data_ptr()), rf._vp(V.data_ptr()),
                                             rf.C.byref(r)))
    ctx.synchronize()
    d_gpu = D.cpu().numpy()[: r.value]
    dm.free()
    a = host_copy(at)  # the fp32 values, widened
    del at
    want = port.single_pass_svd(a, k, p, 1, block=1024)
    rel = np.abs(d_gpu - want.D) / want.D
    out = dict(sigma_max_rel=float(rel.max()), sigma_rel_at_k=float(rel[-1]), margin_at_k=float(1e-4 / max(rel[-1], 1e-300)),
               sigma_median_rel=float(np.median(rel)))
    report("C4/16 16384^2 fp32 k=300 p=30", **out)
    assert r.value == k
    assert out["sigma_max_rel"] <= 1e-4
