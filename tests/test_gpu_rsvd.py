"""GPU parity: the CUDA range finder / RSVD through the C ABI vs the CPU oracle.

Tolerances (north star): singular values 1e-10 relative in FP64 (reorthonormalised
mode, the only mode with that parity floor — SURVEY.md §0.4), residual
||A - U S V^T||_F within 1% of the reference's. Reference tests mirrored:
proj/tests/test_lowrank.cpp:42-105, proj/tests/test_rangefinder.cpp:43-185.
"""
import numpy as np
import pytest

import paper_1607_01649_b200 as rf

pytestmark = pytest.mark.gpu


def planted(port, m, n, sigma, seed=1, noise=0.0, tag="noise.N"):
    a = port.planted(m, n, np.asarray(sigma, dtype=np.float64), seed)
    if noise:
        a = a + noise * port.gaussian(seed, tag, m, n)
    return np.asfortranarray(a)


def geometric(count, ratio):
    return ratio ** np.arange(count, dtype=np.float64)


def recon(f, k=None):
    k = len(f.D) if k is None else k
    return (f.U[:, :k] * f.D[:k]) @ f.V[:, :k].T


def rel(a, b):
    return np.abs(a - b) / np.maximum(np.abs(b), 1e-300)


@pytest.mark.parametrize("m,n,k,p", [(300, 200, 20, 10), (257, 129, 7, 5), (1000, 777, 50, 14), (130, 300, 16, 8)])
@pytest.mark.parametrize("trans", [False, True])
def test_multiply_matches_numpy(ctx, m, n, k, p, trans):
    rng = np.random.default_rng(m * 7 + n)
    a = np.asfortranarray(rng.standard_normal((m, n)))
    x = np.asfortranarray(rng.standard_normal((m if trans else n, k + p)))
    got = rf.multiply(a, x, trans=trans, ctx=ctx)
    want = (a.T @ x) if trans else (a @ x)
    scale = np.abs(a).max() * np.abs(x).max() * (m if trans else n)
    assert np.abs(got - want).max() <= 1e-14 * scale


@pytest.mark.parametrize("case", ["c1", "c2s", "c3s"])
def test_rsvd_reorth_matches_oracle(ctx, port, case):
    if case == "c1":  # BASELINE config 1, full size
        m, n, k, p, q = 2000, 2000, 50, 10, 1
        sig = 1.0 / np.arange(1, 2001, dtype=np.float64) ** 2
        a = planted(port, m, n, sig)
    elif case == "c2s":  # config 2 shape family at 1/10 rows
        m, n, k, p, q = 2000, 1000, 100, 10, 2
        sig = np.exp(-np.arange(1, 501) / 20.0)
        a = planted(port, m, n, sig, noise=1e-6)
    else:  # config 3 family at 1/256 rows, 1/4 cols
        m, n, k, p, q = 4096, 1024, 200, 20, 1
        sig = np.arange(1, 1025, dtype=np.float64) ** -1.5
        a = planted(port, m, n, sig, noise=1e-8)
    want = port.rsvd(a, k, p, q, 1, False, True)
    got = rf.rsvd(a, k, p, q, 1, reorthonormalize=True, ctx=ctx)
    assert got.D.shape == want.D.shape == (k,)
    assert rel(got.D, want.D).max() <= 1e-10
    r_got = np.linalg.norm(a - recon(got))
    r_want = np.linalg.norm(a - recon(want))
    assert abs(r_got - r_want) <= 0.01 * r_want
    # orthonormal factors
    assert np.abs(got.U.T @ got.U - np.eye(k)).max() < 1e-12
    assert np.abs(got.V.T @ got.V - np.eye(k)).max() < 1e-12
    # singular vectors agree up to sign
    s = np.sign(np.sum(got.U * want.U, axis=0))
    assert np.abs(got.U * s - want.U)[:, : k // 2].max() < 1e-9


def test_power_range_matches_oracle(ctx, port):
    sig = 1.0 / np.arange(1, 401, dtype=np.float64) ** 2
    a = planted(port, 600, 400, sig)
    for q in (0, 1, 2):
        want = port.power_range(a, 30, 10, q, 5, reorth=True)
        got = rf.power_range(a, 30, 10, q, 5, reorthonormalize=True, ctx=ctx)
        assert got.Q.shape == want.Q.shape
        # same subspace: Q_ref^T Q has singular values 1
        s = np.linalg.svd(want.Q.T @ got.Q, compute_uv=False)
        assert np.abs(s - 1).max() < 1e-8
        assert abs(got.residual_frob - want.residual_frob) <= 1e-6 * np.linalg.norm(a)


@pytest.mark.parametrize("ell", [1, 2, 3, 33, 97, 220, 235, 236, 237])
def test_power_range_all_sketch_widths(ctx, port, ell):
    """CholeskyQR2 at every sketch-width class: the single-CTA Cholesky (odd
    and even widths, one and several rows per lane, up to the largest width
    whose packed triangle fits in shared memory, 236) and the blocked one just
    above it. Q must be orthonormal and span the oracle's."""
    p = min(5, ell - 1)
    k = ell - p
    sig = 0.97 ** np.arange(300, dtype=np.float64)
    a = planted(port, 1200, 300, sig, seed=ell)
    want = port.power_range(a, k, p, 0, 3, reorth=True)
    got = rf.power_range(a, k, p, 0, 3, reorthonormalize=True, ctx=ctx)
    assert got.Q.shape == want.Q.shape == (1200, ell)
    assert np.abs(got.Q.T @ got.Q - np.eye(ell)).max() < 1e-12
    s = np.linalg.svd(want.Q.T @ got.Q, compute_uv=False)
    assert np.abs(s - 1).max() < 1e-8


def test_basic_range_tracks_residual(ctx):
    # test_rangefinder.cpp:43-71
    sig = geometric(12, 0.5)
    from oracle.oracle import get
    a = planted(get("port"), 30, 20, sig, seed=11)
    rb = rf.basic_range(a, 8, 4, 3, ctx=ctx)
    assert rb.Q.shape == (30, 12)
    assert np.abs(rb.Q.T @ rb.Q - np.eye(12)).max() < 1e-13
    assert np.linalg.norm(a - rb.Q @ rb.B) < 1e-12 * np.linalg.norm(a)
    assert rb.residual_frob < 1e-7 * np.linalg.norm(a)
    pb = rf.basic_range(a, 6, 2, 3, ctx=ctx)
    direct = np.linalg.norm(a - pb.Q @ pb.B)
    assert direct > 1e-4 * np.linalg.norm(a)
    assert abs(pb.residual_frob - direct) <= 1e-9 * direct


def test_rsvd_exact_rank_recovery(ctx, port):
    # test_lowrank.cpp:42-55: planted rank 6, k=6, p=4 -> orth drops columns
    sig = geometric(6, 0.7)
    a = planted(port, 30, 20, sig, seed=3)
    f = rf.rsvd(a, 6, 4, 0, 11, ctx=ctx)
    assert f.U.shape == (30, 6) and f.V.shape == (20, 6) and f.D.shape == (6,)
    assert np.abs(f.U.T @ f.U - np.eye(6)).max() < 1e-12
    assert np.abs(f.V.T @ f.V - np.eye(6)).max() < 1e-12
    assert np.linalg.norm(a - recon(f)) < 1e-10 * np.linalg.norm(a)
    assert rel(f.D, sig).max() < 1e-9


def test_rsvd_keep_oversamples_matches_projection(ctx, port):
    # test_lowrank.cpp:68-87
    sig = geometric(16, 0.6)
    a = planted(port, 35, 25, sig, seed=9)
    f = rf.rsvd(a, 5, 4, 1, 13, keep_oversamples=True, ctx=ctx)
    assert f.D.shape == (9,)
    rb = rf.power_range(a, 5, 4, 1, 13, ctx=ctx)
    e1 = np.linalg.norm(a - recon(f))
    e2 = np.linalg.norm(a - rb.Q @ (rb.Q.T @ a))
    assert abs(e1 - e2) <= 1e-10 * e2


def test_rsvd_plain_power_mode_matches_oracle(ctx, port):
    # reorthonormalize = false (reference default): sketch (A A^T)^q A G then
    # one orth; ill-conditioned for q >= 1, exercised through the
    # Gram-Schmidt fallback. Parity floor ~1e-7 per value.
    sig = 1.0 / np.arange(1, 301, dtype=np.float64) ** 2
    a = planted(port, 400, 300, sig)
    for q in (0, 1):
        want = port.rsvd(a, 20, 10, q, 7, False, False)
        got = rf.rsvd(a, 20, 10, q, 7, ctx=ctx)
        assert got.D.shape == want.D.shape
        assert rel(got.D, want.D).max() < 1e-6
        r1, r2 = np.linalg.norm(a - recon(got)), np.linalg.norm(a - recon(want))
        assert abs(r1 - r2) <= 0.01 * r2


def test_plain_mode_orth_runs_shifted_choleskyqr3(port):
    """The plain power mode's sketch (A A^T) A G is far too ill-conditioned for CholeskyQR2 (kappa ~ 1e9 here)
    but has full rank: orth takes the shifted CholeskyQR3 path (three Grams, no column-by-column work), keeps
    every column like the reference's Gram-Schmidt (dense.cpp:402-431) and gives the reference's factors. An
    exactly rank-deficient sketch is rejected by the same path and falls through to Gram-Schmidt, which
    drops the reference's columns."""
    sig = 1.0 / np.arange(1, 301, dtype=np.float64) ** 2
    a = planted(port, 2000, 300, sig)
    c = rf.Context(0)
    c.profile(True)
    try:
        want = port.rsvd(a, 20, 10, 1, 7, False, False)
        got = rf.rsvd(a, 20, 10, 1, 7, ctx=c)
        n3, _ = c.profile_read("scholqr3")
        assert n3 >= 1
        assert got.D.shape == want.D.shape and rel(got.D, want.D).max() < 1e-6
        r1, r2 = np.linalg.norm(a - recon(got)), np.linalg.norm(a - recon(want))
        assert abs(r1 - r2) <= 0.01 * r2
        assert np.abs(got.U.T @ got.U - np.eye(20)).max() < 1e-12
        # exact rank 6 < l = 12: every path but Gram-Schmidt must refuse it
        low = planted(port, 500, 200, np.array([5.0, 4.0, 3.0, 2.0, 1.0, 0.5]), seed=3)
        c.profile_reset()
        w2 = port.rsvd(low, 8, 4, 1, 7, False, False)
        g2 = rf.rsvd(low, 8, 4, 1, 7, ctx=c)
        assert g2.D.shape == w2.D.shape and rel(g2.D, w2.D).max() < 1e-6
    finally:
        c.close()


def test_rsvd_deterministic(ctx, port):
    sig = geometric(10, 0.5)
    a = planted(port, 25, 20, sig, seed=2)
    f1 = rf.rsvd(a, 4, 4, 1, 7, ctx=ctx)
    f2 = rf.rsvd(a, 4, 4, 1, 7, ctx=ctx)
    assert np.array_equal(f1.U, f2.U) and np.array_equal(f1.D, f2.D)
    f3 = rf.rsvd(a, 4, 4, 1, 8, ctx=ctx)
    assert not np.array_equal(f1.U, f3.U)


@pytest.mark.parametrize("m", [70000, 600000])
def test_rsvd_host_streamed_matches_device_path(ctx, m):
    """rfgpu_rsvd_host streams A in row panels behind pass 1 (4 / 16 panels
    here); the factors must match the device-resident call and the cached
    device buffer must be reusable across calls of different sizes."""
    n, k, p = 96, 10, 6
    rng = np.random.default_rng(m)
    u, _ = np.linalg.qr(rng.standard_normal((m, 40)))
    v, _ = np.linalg.qr(rng.standard_normal((n, 40)))
    a = np.asfortranarray((u * 0.8 ** np.arange(40)) @ v.T)
    host = rf.rsvd(a, k, p, 1, 3, reorthonormalize=True, ctx=ctx)
    dm = ctx.matrix(a)
    try:
        dev = rf.rsvd(dm, k, p, 1, 3, reorthonormalize=True, ctx=ctx)
    finally:
        dm.free()
    assert rel(host.D, dev.D).max() < 1e-12
    assert np.abs(np.abs(host.U) - np.abs(dev.U)).max() < 1e-9
    assert np.abs(np.abs(host.V) - np.abs(dev.V)).max() < 1e-9
    a5 = np.asfortranarray(a[:5000])
    small = rf.rsvd(a5, k, p, 1, 3, reorthonormalize=True, ctx=ctx)  # reuses the larger cached buffer
    dm = ctx.matrix(a5)
    try:
        want = rf.rsvd(dm, k, p, 1, 3, reorthonormalize=True, ctx=ctx)
    finally:
        dm.free()
    assert np.array_equal(small.D, want.D) and np.array_equal(small.U, want.U)


def test_rsvd_host_staging_odd_rows_misaligned_base(ctx):
    """The pinned staging ring copies caller columns with non-temporal stores (32-byte aligned bodies, plain
    heads and tails): an odd row count and a base 8 bytes off a 32-byte boundary walk every alignment."""
    m, n, k, p = 70001, 64, 8, 4
    rng = np.random.default_rng(11)
    buf = np.empty(m * n + 3)
    a = buf[1:1 + m * n].reshape((m, n), order="F")
    u, _ = np.linalg.qr(rng.standard_normal((m, 20)))
    v, _ = np.linalg.qr(rng.standard_normal((n, 20)))
    a[...] = (u * 0.7 ** np.arange(20)) @ v.T
    assert a.ctypes.data % 32 != 0 and a.flags.f_contiguous
    host = rf.rsvd(a, k, p, 1, 3, reorthonormalize=True, ctx=ctx)
    dm = ctx.matrix(np.asfortranarray(a.copy(order="F")))
    try:
        dev = rf.rsvd(dm, k, p, 1, 3, reorthonormalize=True, ctx=ctx)
    finally:
        dm.free()
    assert rel(host.D, dev.D).max() < 1e-12
    assert np.abs(np.abs(host.U) - np.abs(dev.U)).max() < 1e-9


def test_rsvd_zero_matrix(ctx):
    f = rf.rsvd(np.zeros((12, 9)), 3, 2, 0, 1, ctx=ctx)
    assert f.U.shape[1] == 0 and f.D.size == 0


def test_rsvd_validation(ctx, port):
    a = planted(port, 10, 8, geometric(4, 0.5), seed=1)
    with pytest.raises(rf.ParameterError):
        rf.rsvd(a, 0, 2, 0, 1, ctx=ctx)
    with pytest.raises(rf.ParameterError):
        rf.rsvd(a, 5, 4, 0, 1, ctx=ctx)
    with pytest.raises(rf.ParameterError):
        rf.rsvd(a, 2, 2, -1, 1, ctx=ctx)
    with pytest.raises(rf.ParameterError):
        rf.basic_range(a, 2, 2, 1, q=1, ctx=ctx)


# ----------------------------------------------------------- single pass ---
def test_single_pass_matches_reference_small_k(ctx, ref):
    # the reference's own stacked least squares is feasible at small k
    a = ref.planted(300, 250, np.exp(-np.arange(1, 101) / 10.0), 1)
    want = ref.single_pass_svd(a, 10, 10, 3, block=32)
    s = rf.MatrixStream(a, 32)
    got = rf.single_pass_svd(s, 10, 10, 3, ctx=ctx)
    assert s.passes_completed() == 1 and s.entries_served == 300 * 250
    assert rel(got.D, want.D).max() < 1e-10
    r1, r2 = np.linalg.norm(a - recon(got)), np.linalg.norm(a - recon(want))
    assert abs(r1 - r2) <= 0.01 * r2


def test_single_pass_matches_restated_oracle(ctx, port):
    # config-4 family at reduced size: r = 200, s_j = exp(-j/10), noise 1e-4
    m, n, k, p = 1500, 1200, 60, 10
    a = planted(port, m, n, np.exp(-np.arange(1, 201) / 10.0), seed=1, noise=1e-4)
    want = port.single_pass_svd(a, k, p, 1, block=64)
    got = rf.single_pass_svd(rf.MatrixStream(a, 64), k, p, 1, ctx=ctx)
    assert got.D.shape == want.D.shape == (k,)
    assert rel(got.D, want.D).max() < 1e-8
    assert np.abs(got.U.T @ got.U - np.eye(k)).max() < 1e-10


def test_single_pass_exact_rank(ctx, port):
    # test_lowrank.cpp:144-160
    sig = 0.5 ** np.arange(5.0)
    a = planted(port, 35, 25, sig, seed=6)
    s = rf.MatrixStream(a, 6)
    f = rf.single_pass_svd(s, 5, 5, 29, ctx=ctx)
    assert s.passes_completed() == 1 and s.entries_served == 35 * 25
    assert rel(f.D, sig).max() < 1e-7
    assert np.linalg.norm(a - recon(f)) < 1e-7 * np.linalg.norm(a)


def test_single_pass_stream_contract(ctx, port):
    a = planted(port, 20, 16, geometric(4, 0.5), seed=2)
    s = rf.MatrixStream(a, 7)
    rf.single_pass_svd(s, 3, 2, 1, ctx=ctx)
    with pytest.raises(rf.StreamContractError):
        s.next_block()


@pytest.mark.parametrize("m,n", [(60, 60), (500, 110), (220, 220), (2000, 300), (330, 330), (5000, 64)])
def test_svd_dense_matches_oracle(ctx, port, m, n):
    rng = np.random.default_rng(m + n)
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = np.arange(1, n + 1, dtype=np.float64) ** -1.5
    a = np.asfortranarray((u * s) @ v.T)
    want = port.svd(a)
    got = rf.svd_dense(a, ctx=ctx)
    assert rel(got.D, want.D).max() < 1e-12
    assert np.abs(got.U.T @ got.U - np.eye(n)).max() < 1e-12
    assert np.abs(got.V.T @ got.V - np.eye(n)).max() < 1e-12
    assert np.linalg.norm(a - (got.U * got.D) @ got.V.T) < 1e-13 * np.linalg.norm(a) * np.sqrt(n)
