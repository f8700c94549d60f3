"""GPU: the reference's own known-answer / edge tests for this path, re-expressed
against the device implementation.

* svd_dense on a spectrum spanning 23 orders of magnitude
  (proj/tests/test_dense.cpp:222-236): converges (per-sweep norm ordering,
  dense.cpp:597-618), orthonormal factors, reconstruction 1e-13, every
  singular value above 1e-10 sigma_1 to 1e-10 relative.
* frob_residual's guards (proj/tests/test_rangefinder.cpp:39,
  rangefinder.cpp:45-54): NumericalError when the projection exceeds the total
  norm, ParameterError on a negative norm, the down-dated value otherwise.
* cpqr's recompute rule (dense.cpp:503-518): columns nearly parallel to the
  first pivot shrink below 1e-8 of their original norm, forcing exact
  recomputation; pivots must still equal the reference's.
* the FP32 dual sketch entry point rfgpu_dual_sketch_f32 (Yc = A Gc,
  Yr = A^T Gr from one read of an fp32 A; lowrank.cpp:170-176).
"""
import numpy as np
import pytest

import paper_1607_01649_b200 as rf

pytestmark = pytest.mark.gpu


def orthonormality_defect(q):
    return float(np.max(np.abs(q.T @ q - np.eye(q.shape[1]))))


def test_svd_dense_23_decade_spectrum(ctx, ref):
    sigma = 0.7 ** np.arange(150, dtype=np.float64)  # support::geometric_sigma(150, 0.7): 1 .. 1e-23
    a = ref.test_planted(200, 150, sigma, 1)  # the reference test's own matrix (support::planted, Haar factors)
    f = rf.svd_dense(a, ctx=ctx)
    assert f.U.shape == (200, 150) and f.V.shape == (150, 150) and len(f.D) == 150
    assert orthonormality_defect(f.U) < 1e-12
    assert orthonormality_defect(f.V) < 1e-12
    rec = (f.U * f.D) @ f.V.T
    assert np.linalg.norm(rec - a) / np.linalg.norm(a) < 1e-13
    # CHECK(f.D[j] == doctest::Approx(sigma[j]).epsilon(1e-10)): |d - s| < 1e-10 (1 + max(|d|, |s|))
    for j, s in enumerate(sigma):
        if s < 1e-10 * sigma[0]:
            break
        assert abs(f.D[j] - s) < 1e-10 * (1.0 + max(abs(f.D[j]), s)), (j, f.D[j], s)
    want = ref.svd(a)
    assert np.max(np.abs(f.D - want.D) / (1.0 + want.D)) < 1e-14


def test_frob_residual_guards(ctx):
    b = np.array([[3.0, 0.0], [0.0, 4.0]])  # ||B||_F = 5
    with pytest.raises(rf.NumericalError):
        rf.frob_residual(3.0, b, ctx=ctx)
    with pytest.raises(rf.ParameterError):
        rf.frob_residual(-1.0, b, ctx=ctx)
    assert rf.frob_residual(13.0, b, ctx=ctx) == pytest.approx(12.0, rel=1e-15)
    assert rf.frob_residual(5.0 * (1 + 1e-9), b, ctx=ctx) == pytest.approx(0.0, abs=1e-3)  # inside the 1e-8 slack


def test_cpqr_recompute_rule_keeps_reference_pivots(ctx, port):
    rng = np.random.default_rng(5)
    m, n, k = 40, 300, 30
    # a rank-one matrix plus 1e-5 noise: once the first pivot removes the common direction, every
    # remaining column has lost all but ~1e-13 of its squared norm, so (a numpy restatement of the
    # rule counts it) 28 of the 30 steps recompute the norms exactly
    v, c = rng.standard_normal(m), rng.standard_normal(n)
    y = np.asfortranarray(10.0 * np.outer(v, c) + 1e-5 * rng.standard_normal((m, n)))
    js_ref, z_ref, tr_ref = port.id_col(y, k)
    got = rf.id_deterministic(y, k, ctx=ctx)
    assert np.array_equal(got.Js, js_ref)
    assert got.rank_truncated == tr_ref
    assert np.max(np.abs(got.Z - z_ref)) <= 1e-8 * max(1.0, np.max(np.abs(z_ref)))


def test_dual_sketch_f32_entry_point(ctx):
    rng = np.random.default_rng(9)
    m, n, ell = 1500, 1100, 48
    a = np.asfortranarray(rng.standard_normal((m, n)).astype(np.float32))
    gc = np.asfortranarray(rng.standard_normal((n, ell)).astype(np.float32))
    gr = np.asfortranarray(rng.standard_normal((m, ell)).astype(np.float32))
    dm = rf.DeviceMatrix.upload(ctx, a, f32=True)
    yc = np.zeros(m * ell, dtype=np.float32)
    yr = np.zeros(n * ell, dtype=np.float32)
    rf._check(rf.lib().rfgpu_dual_sketch_f32(ctx.handle, dm.handle, rf._fp(gc.reshape(-1, order="F")),
                                             rf._fp(gr.reshape(-1, order="F")), ell, rf._fp(yc), rf._fp(yr)))
    dm.free()
    a64 = a.astype(np.float64)
    want_c = a64 @ gc.astype(np.float64)
    want_r = a64.T @ gr.astype(np.float64)
    assert np.max(np.abs(yc.reshape((m, ell), order="F") - want_c)) <= 1e-6 * np.max(np.abs(want_c))
    assert np.max(np.abs(yr.reshape((n, ell), order="F") - want_r)) <= 1e-6 * np.max(np.abs(want_r))


def test_wide_sketches_beyond_352(port):
    """l = k + p above 352 (the single-CTA triangular inverse's range) runs on the blocked l x l kernels up
    to 736; above that the call is refused with the reference's parameter error class, not a CUDA failure."""
    ctx = rf.Context(0)
    try:
        ell = 400
        rng = np.random.default_rng(ell)
        u, _ = np.linalg.qr(rng.standard_normal((2 * ell, ell)))
        v, _ = np.linalg.qr(rng.standard_normal((ell, ell)))
        a = np.asfortranarray((u * np.arange(1, ell + 1) ** -1.0) @ v.T)
        f = rf.svd_dense(a, ctx=ctx)
        s = np.linalg.svd(a, compute_uv=False)
        assert np.max(np.abs(f.D - s) / s) < 1e-12
        big = port.planted(3000, 1500, 1.0 / np.arange(1, 801) ** 1.2, 1)
        got = rf.rsvd(big, 380, 20, 1, 7, reorthonormalize=True, ctx=ctx)
        want = port.rsvd(big, 380, 20, 1, 7, False, True)
        assert got.D.shape == want.D.shape and np.max(np.abs(got.D - want.D) / want.D) < 1e-10
        with pytest.raises(rf.ParameterError):
            rf.rsvd(port.planted(900, 800, 1.0 / np.arange(1, 801), 1), 730, 10, 0, 1, ctx=ctx)
    finally:
        ctx.close()
