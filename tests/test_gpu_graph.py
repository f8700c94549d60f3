"""GPU: the device-resident rsvd as a replayed CUDA graph (rfgpu_rsvd_device: the
second call with the same arguments is captured, later calls replay it) and
the speculative CholeskyQR2 that makes the call capturable (one host round
trip, at the end): the graph replays give the eager, non-speculative result
bit for bit, and an input whose sketch fails the CholeskyQR gate (exact rank
below l: the reference's orth drops columns, dense.cpp:402-431) falls back to
the eager Gram-Schmidt path on every replay with the reference's kept rank."""
import os

import numpy as np
import pytest

import paper_1607_01649_b200 as rf

pytestmark = pytest.mark.gpu


def device_rsvd(ctx, at, m, n, k, p, q, reorth, calls, env=None):
    import torch
    old = {}
    for kk, v in (env or {}).items():
        old[kk] = os.environ.get(kk)
        os.environ[kk] = v
    try:
        ell = k + p
        A = rf.DeviceMatrix.wrap(ctx, at.data_ptr(), m, n, m, keep=at)
        g = torch.from_numpy(rf.gaussian(1, "range.G", n, ell).reshape(-1, order="F")).cuda()
        U = torch.zeros(m * ell, dtype=torch.float64, device="cuda")
        D = torch.zeros(ell, dtype=torch.float64, device="cuda")
        V = torch.zeros(n * ell, dtype=torch.float64, device="cuda")
        r = rf._i64()
        outs = []
        for _ in range(calls):
            U.zero_(), D.zero_(), V.zero_()
            rf._check(rf.lib().rfgpu_rsvd_device(ctx.handle, A.handle, rf._vp(g.data_ptr()), k, ell, q, 0, int(reorth),
                                                 rf._vp(U.data_ptr()), rf._vp(D.data_ptr()), rf._vp(V.data_ptr()),
                                                 rf.C.byref(r)))
            ctx.synchronize()
            outs.append((r.value, D.cpu().numpy()[: r.value].copy(), U.cpu().numpy()[: m * r.value].copy()))
        A.free()
        return outs
    finally:
        for kk, v in old.items():
            if v is None:
                os.environ.pop(kk, None)
            else:
                os.environ[kk] = v


@pytest.mark.parametrize("ozaki", ["0", "1"])
def test_graph_replays_match_eager(port, ozaki):
    import torch
    m, n = 3000, 700
    a = port.planted(m, n, 1.0 / np.arange(1, 401) ** 1.5, 1) + 1e-9 * port.gaussian(1, "noise.N", m, n)
    at = torch.from_numpy(np.ascontiguousarray(a.T)).cuda()
    ctx = rf.Context(0)
    env = {"RFGPU_OZAKI": ozaki}
    got = device_rsvd(ctx, at, m, n, 30, 10, 1, True, 4, env)
    launches = ctx.launch_count()
    ctx.close()
    ctx2 = rf.Context(0)
    want = device_rsvd(ctx2, at, m, n, 30, 10, 1, True, 1, {**env, "RFGPU_GRAPH": "0", "RFGPU_SPECULATE": "0"})[0]
    ctx2.close()
    assert launches > 0
    for r, d, u in got:
        assert r == want[0] == 30
        assert np.array_equal(d, want[1]) and np.array_equal(u, want[2])
    ref = port.rsvd(a, 30, 10, 1, 1, False, True)
    assert np.max(np.abs(got[-1][1] - ref.D) / ref.D) <= 1e-10


def test_graph_falls_back_when_speculation_fails(port):
    import torch
    m, n = 2500, 600
    a = port.planted(m, n, np.array([3.0, 2.0, 1.0, 0.5, 0.25] * 3), 2)  # exact rank 15 < l = 30
    at = torch.from_numpy(np.ascontiguousarray(a.T)).cuda()
    ctx = rf.Context(0)
    got = device_rsvd(ctx, at, m, n, 20, 10, 1, True, 4, {"RFGPU_OZAKI": "0"})
    ctx.close()
    want = port.rsvd(a, 20, 10, 1, 1, False, True)
    for r, d, _ in got:
        assert r == len(want.D) == 15
        assert np.max(np.abs(d - want.D) / want.D) <= 1e-9


def test_graph_is_keyed_by_the_path_switches(port):
    """A graph recorded on the digit path must not be replayed when the same call is made with
    RFGPU_OZAKI=0 (bench.py's DMMA self-check does exactly that): the replies differ in the last bits,
    and the DMMA reply equals the eager DMMA call bit for bit."""
    import torch
    m, n = 3000, 700
    a = port.planted(m, n, 1.0 / np.arange(1, 401) ** 1.5, 1) + 1e-9 * port.gaussian(1, "noise.N", m, n)
    at = torch.from_numpy(np.ascontiguousarray(a.T)).cuda()
    ctx = rf.Context(0)
    # same context, same buffers: 4 calls on the digits (graph recorded and replayed), then the DMMA call
    ell = 40
    A = rf.DeviceMatrix.wrap(ctx, at.data_ptr(), m, n, m, keep=at)
    g = torch.from_numpy(rf.gaussian(1, "range.G", n, ell).reshape(-1, order="F")).cuda()
    U = torch.zeros(m * ell, dtype=torch.float64, device="cuda")
    D = torch.zeros(ell, dtype=torch.float64, device="cuda")
    V = torch.zeros(n * ell, dtype=torch.float64, device="cuda")
    r = rf._i64()

    def call():
        rf._check(rf.lib().rfgpu_rsvd_device(ctx.handle, A.handle, rf._vp(g.data_ptr()), 30, ell, 1, 0, 1,
                                             rf._vp(U.data_ptr()), rf._vp(D.data_ptr()), rf._vp(V.data_ptr()),
                                             rf.C.byref(r)))
        ctx.synchronize()
        return D.cpu().numpy()[:30].copy()

    old = os.environ.get("RFGPU_OZAKI")
    try:
        os.environ["RFGPU_OZAKI"] = "1"
        digits = [call() for _ in range(4)][-1]
        os.environ["RFGPU_OZAKI"] = "0"
        dmma = call()
    finally:
        if old is None:
            os.environ.pop("RFGPU_OZAKI", None)
        else:
            os.environ["RFGPU_OZAKI"] = old
    A.free()
    ctx.close()
    ctx2 = rf.Context(0)
    want = device_rsvd(ctx2, at, m, n, 30, 10, 1, True, 1, {"RFGPU_OZAKI": "0", "RFGPU_GRAPH": "0"})[0][1]
    ctx2.close()
    assert np.array_equal(dmma, want)
    assert not np.array_equal(dmma, digits)
    assert np.max(np.abs(dmma - digits) / dmma) <= 1e-12
