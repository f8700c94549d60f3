"""The C++ drop-in: a probe compiled against the REFERENCE headers and linked
only against librandfact_b200.so (oracle/Makefile target dropin_probe)."""
import os
import subprocess
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROBE = os.path.join(ROOT, "oracle", "_ref", "dropin_probe")
needs_probe = pytest.mark.skipif(not os.path.exists(PROBE), reason="dropin_probe not built (needs /root/reference)")


def run(*args):
    return subprocess.run([PROBE, *map(str, args)], capture_output=True, text=True, timeout=600)


@needs_probe
def test_probe_links_and_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    r = run("cpu")
    assert r.returncode == 0, r.stderr
    assert "DEVICE_ERROR" in r.stdout and "no CPU fallback" in r.stdout
    assert "VALIDATION_OK" in r.stdout  # reference ParameterError class caught by reference-compiled code


@needs_probe
@pytest.mark.gpu
def test_probe_rsvd_matches_oracle(port):
    sig = 1.0 / np.arange(1, 301, dtype=np.float64) ** 2
    a = port.planted(500, 300, sig, 1)
    with tempfile.TemporaryDirectory() as d:
        ain, out = os.path.join(d, "a.bin"), os.path.join(d, "o.bin")
        np.asfortranarray(a).reshape(-1, order="F").tofile(ain)
        r = run("rsvd", ain, 500, 300, 20, 10, 1, 1, out)
        assert r.returncode == 0, r.stdout + r.stderr
        got = np.fromfile(out)
    want = port.rsvd(a, 20, 10, 1, 1, False, True)
    assert np.max(np.abs(got[:20] - want.D) / want.D) < 1e-10
    rb = port.power_range(a, 20, 10, 1, 1, reorth=True)
    resid = float(r.stdout.split("resid")[1])
    assert abs(resid - rb.residual_frob) <= 1e-6 * np.linalg.norm(a)


@needs_probe
@pytest.mark.gpu
def test_probe_cur_matches_oracle(port):
    a = port.planted(400, 300, 10.0 ** (-6.0 * np.arange(200) / 199.0), 2)
    with tempfile.TemporaryDirectory() as d:
        ain, out = os.path.join(d, "a.bin"), os.path.join(d, "o.bin")
        np.asfortranarray(a).reshape(-1, order="F").tofile(ain)
        r = run("cur", ain, 400, 300, 30, 10, out)
        assert r.returncode == 0, r.stdout + r.stderr
        got = np.fromfile(out).astype(np.int64)
    want = port.randomized_cur(a, 30, 10, 0, 1)
    assert np.array_equal(got[:30], want.Js) and np.array_equal(got[30:], want.Is)


@needs_probe
@pytest.mark.gpu
def test_probe_single_pass_stream_telemetry(port):
    """single_pass_svd(MatrixStream&) through the drop-in (which reads the stream's matrix in slabs): the
    stream ends exactly as if drained block by block (acceptance #8, acceptance.cpp:296-316), a second
    pass raises StreamContractError, and the singular values match the oracle's single pass."""
    m, n, k, p, b = 700, 520, 12, 12, 32
    a = port.planted(m, n, np.exp(-np.arange(1, 301) / 12.0), 3) + 1e-9 * port.gaussian(3, "noise.N", m, n)
    with tempfile.TemporaryDirectory() as d:
        ain, out = os.path.join(d, "a.bin"), os.path.join(d, "o.bin")
        np.asfortranarray(a).reshape(-1, order="F").tofile(ain)
        r = run("spsvd", ain, m, n, k, p, b, out)
        assert r.returncode == 0, r.stdout + r.stderr
        got = np.fromfile(out)
    assert f"rank {k} entries_served {m * n} passes_completed 1 has_next 0" in r.stdout
    assert "STREAM_CONTRACT_OK" in r.stdout
    want = port.single_pass_svd(a, k, p, 1, block=b)
    assert np.max(np.abs(got - want.D) / want.D) <= 1e-8
