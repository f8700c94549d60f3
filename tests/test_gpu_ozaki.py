"""GPU: the FP64 passes on the INT8 tensor cores (csrc/ozaki.cu, Ozaki digit
splitting + tcgen05 kind::i8). Forced on with RFGPU_OZAKI=1 at sizes where the
size rule would pick DMMA, so every case here runs the digit GEMM.

Bars: products within 1e-14 of an extended-precision reference, relative to
max|A(i,:)| max|X(:,c)| * sqrt(K) (the digit truncation bound, ~2^-53 per
term); rsvd singular values 1e-10 vs the oracle (the north-star bar); the
reference's exact-rank residual identity (test_rangefinder.cpp:43-71).
"""
import numpy as np
import pytest

import paper_1607_01649_b200 as rf

pytestmark = pytest.mark.gpu


def planted(port, m, n, sigma, seed=1, noise=0.0):
    a = port.planted(m, n, np.asarray(sigma, dtype=np.float64), seed)
    if noise:
        a = a + noise * port.gaussian(seed, "noise.N", m, n)
    return np.asfortranarray(a)


@pytest.fixture
def ozaki(monkeypatch):
    monkeypatch.setenv("RFGPU_OZAKI", "1")


def exact_product(a, x, trans):
    a = a.astype(np.longdouble)
    x = x.astype(np.longdouble)
    return (a.T @ x) if trans else (a @ x)


def scaled_err(got, want, a, x, trans):
    rows = np.abs(a).max(axis=0 if trans else 1)
    cols = np.abs(x).max(axis=0)
    k = a.shape[0] if trans else a.shape[1]
    scale = np.outer(rows, cols) * np.sqrt(k)
    scale[scale == 0] = 1.0
    return float(np.max(np.abs(got.astype(np.longdouble) - want) / scale))


@pytest.mark.parametrize("m,n,cols", [(1000, 777, 40), (4096, 300, 64), (257, 20000, 3), (40000, 129, 70)])
@pytest.mark.parametrize("trans", [False, True])
def test_digit_gemm_matches_extended_precision(ctx, ozaki, m, n, cols, trans):
    rng = np.random.default_rng(m + n + cols)
    a = rng.standard_normal((m, n))
    a[3] *= 1e120             # wide dynamic range across rows
    a[5] *= 1e-150
    a[7] = 0.0                # zero row
    a[:, 2] *= 1e-8           # small column inside every row
    x = rng.standard_normal((m if trans else n, cols))
    x[:, 1] *= 1e80
    x[:, 2] = 0.0
    a = np.asfortranarray(a)
    got = rf.multiply(a, x, trans=trans, ctx=ctx)
    want = exact_product(a, x, trans)
    assert scaled_err(got, want, a, x, trans) < 1e-14
    if not trans:
        assert np.all(got[7] == 0.0)
    assert np.all(got[:, 2] == 0.0)


@pytest.mark.parametrize("shared", ["0", "1", None])
@pytest.mark.parametrize("m,n,cols", [(1000, 777, 40), (40000, 129, 70)])
@pytest.mark.parametrize("trans", [False, True])
def test_digit_gemm_one_or_two_digit_sets(ctx, ozaki, monkeypatch, shared, m, n, cols, trans):
    """Columns of comparable scale (exponents within 2 bits): A^T Q may run on
    the row-scaled digits with the row factors moved onto Q (one digit set for
    both passes; the library does so when the second set does not fit in HBM).
    Forced on (RFGPU_OZAKI_SHARED=1), off, and by default (row-major second
    set), the products stay within the column-scaled bar."""
    if shared is None:
        monkeypatch.delenv("RFGPU_OZAKI_SHARED", raising=False)
    else:
        monkeypatch.setenv("RFGPU_OZAKI_SHARED", shared)
    rng = np.random.default_rng(m + cols)
    a = rng.standard_normal((m, n))
    a[3] *= 8.0              # a dominant row keeps every column maximum in one binade
    a[5] *= 1e-150           # tiny row
    a[7] = 0.0               # zero row
    x = rng.standard_normal((m if trans else n, cols))
    x[:, 1] *= 1e80
    x[:, 2] = 0.0
    a = np.asfortranarray(a)
    got = rf.multiply(a, x, trans=trans, ctx=ctx)
    want = exact_product(a, x, trans)
    assert scaled_err(got, want, a, x, trans) < 1e-14
    assert np.all(got[:, 2] == 0.0)


def test_graded_columns_keep_two_digit_sets(ctx, ozaki, monkeypatch):
    """A column 2^-30 below the others: A^T Q must use the column-scaled set
    (the shared set would lose ~30 bits there; it is only a fallback for
    column exponents within 2 bits)."""
    monkeypatch.delenv("RFGPU_OZAKI_SHARED", raising=False)
    rng = np.random.default_rng(9)
    a = rng.standard_normal((3000, 300))
    a[:, 4] *= 2.0 ** -30
    q = rng.standard_normal((3000, 16))
    a = np.asfortranarray(a)
    got = rf.multiply(a, q, trans=True, ctx=ctx)
    want = exact_product(a, q, True)
    assert scaled_err(got, want, a, q, True) < 1e-14


@pytest.mark.parametrize("case", [(600, 400, 20, 10, 1), (2000, 2000, 50, 10, 1), (5000, 1500, 100, 10, 2)])
def test_rsvd_on_digit_gemm_matches_oracle(ctx, port, ozaki, case):
    m, n, k, p, q = case
    sig = np.arange(1, min(m, n) + 1, dtype=np.float64) ** -1.5
    a = np.asfortranarray(port.planted(m, n, sig, 3))
    want = port.rsvd(a, k, p, q, 7, False, True)
    got = rf.rsvd(a, k, p, q, 7, reorthonormalize=True, ctx=ctx)
    assert np.max(np.abs(got.D - want.D) / want.D) < 1e-10
    r1 = np.linalg.norm(a - (got.U * got.D) @ got.V.T)
    r2 = np.linalg.norm(a - (want.U * want.D) @ want.V.T)
    assert abs(r1 - r2) <= 0.01 * r2


def test_exact_rank_residual_on_digit_gemm(ctx, port, ozaki):
    # test_rangefinder.cpp:43-71 with every pass on the INT8 tensor cores
    sig = 0.5 ** np.arange(12, dtype=np.float64)
    a = np.asfortranarray(port.planted(30, 20, sig, 11))
    rb = rf.basic_range(a, 8, 4, 3, ctx=ctx)
    assert rb.residual_frob < 1e-7 * np.linalg.norm(a)
    assert np.linalg.norm(a - rb.Q @ rb.B) < 1e-12 * np.linalg.norm(a)


def test_streamed_panels_on_digit_gemm(ctx, ozaki, monkeypatch):
    # host matrix -> rfgpu_rsvd_host: 4 upload panels, each sliced and multiplied as it lands
    m, n, k, p = 70000, 96, 10, 6
    rng = np.random.default_rng(5)
    u, _ = np.linalg.qr(rng.standard_normal((m, 40)))
    v, _ = np.linalg.qr(rng.standard_normal((n, 40)))
    a = np.asfortranarray((u * 0.8 ** np.arange(40)) @ v.T)
    host = rf.rsvd(a, k, p, 1, 3, reorthonormalize=True, ctx=ctx)
    monkeypatch.setenv("RFGPU_OZAKI", "0")
    dm = ctx.matrix(a)
    try:
        dev = rf.rsvd(dm, k, p, 1, 3, reorthonormalize=True, ctx=ctx)
    finally:
        dm.free()
    assert np.max(np.abs(host.D - dev.D) / dev.D) < 1e-12


@pytest.mark.parametrize("m", [1500, 1501])
@pytest.mark.parametrize("f32", [False, True])
def test_single_pass_device_on_digit_gemm(ctx, port, ozaki, f32, m):
    """rfgpu_single_pass_svd_device with both sketches on the digit path:
    FP64 data (7 digits) within 1e-8 of the restated oracle, FP32 data (4
    digits, 10 products) within the FP32 bar 1e-4 of the oracle run on the
    same rounded data. m = 1501 gives columns that do not start 16-byte
    aligned, so A is sliced by the register-prefetch slicer instead of the
    cp.async one."""
    import ctypes as C
    import torch
    n, k, p = 1200, 60, 10
    ell = k + p
    a = planted(port, m, n, np.exp(-np.arange(1, 201) / 10.0), seed=1, noise=1e-4)
    if f32:
        a = np.asfortranarray(a.astype(np.float32).astype(np.float64))
    want = port.single_pass_svd(a, k, p, 1, block=64)
    dev = torch.device("cuda")
    At = torch.from_numpy(np.ascontiguousarray(a.T)).to(dev)  # column-major A as rows of A^T
    if f32:
        At = At.float()
    dm = rf.DeviceMatrix.wrap(ctx, At.data_ptr(), m, n, m, f32=f32, keep=At)
    gc = torch.from_numpy(np.asfortranarray(rf.gaussian(1, "spsvd.Gc", n, ell)).reshape(-1, order="F")).to(dev)
    gr = torch.from_numpy(np.asfortranarray(rf.gaussian(1, "spsvd.Gr", m, ell)).reshape(-1, order="F")).to(dev)
    U = torch.empty(m * ell, device=dev, dtype=torch.float64)
    D = torch.empty(ell, device=dev, dtype=torch.float64)
    V = torch.empty(n * ell, device=dev, dtype=torch.float64)
    r = C.c_int64()
    rf._check(rf.lib().rfgpu_single_pass_svd_device(ctx.handle, dm.handle, C.c_void_p(gc.data_ptr()),
                                                      C.c_void_p(gr.data_ptr()), k, ell, C.c_void_p(U.data_ptr()),
                                                      C.c_void_p(D.data_ptr()), C.c_void_p(V.data_ptr()), C.byref(r)))
    torch.cuda.synchronize()
    got = D.cpu().numpy()[: r.value]
    tol = 1e-4 if f32 else 1e-8
    assert r.value == k
    assert np.max(np.abs(got - want.D) / want.D) < tol
