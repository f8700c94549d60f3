"""CPU: the C-ABI library loads, exports every entry point include/rfgpu.h
declares, and fails loudly (no CPU fallback) when no GPU is present. The host
generator (rfgpu_gaussian, product code: the drop-in needs the reference
stream to build G) is bitwise the reference's."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1607_01649_b200 as rf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rfgpu.h")


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(rfgpu_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_entry_points():
    names = declared_functions()
    for want in ("rfgpu_rsvd", "rfgpu_range_finder", "rfgpu_row_sketch", "rfgpu_col_id", "rfgpu_dual_sketch_f32",
                 "rfgpu_gaussian", "rfgpu_ctx_create_dist"):
        assert want in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(rf.library_path())
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, f"librfgpu.so lacks {missing}"


def test_python_mirror_binds_every_symbol():
    assert set(declared_functions()) <= set(rf._SIGS)


def test_gaussian_is_bitwise_reference(port):
    for seed, tag, m, n in [(1, "range.G", 2000, 60), (7, "g", 5, 4), (1, "cur.G", 33, 17), (2**63 + 5, "x", 3, 3)]:
        assert np.array_equal(rf.gaussian(seed, tag, m, n), port.gaussian(seed, tag, m, n))


def test_gaussian_range_is_seekable():
    full = rf.gaussian(11, "spsvd.Gc", 77, 13).reshape(-1, order="F")
    part = np.empty(101)
    rf._check(rf.lib().rfgpu_gaussian_range(11, b"spsvd.Gc", 333, 101, rf._dp(part)))
    assert np.array_equal(part, full[333:434])


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(rf.DeviceError):
        rf.Context(0)


def test_staging_copy_non_temporal_paths():
    """csrc/host_copy.cpp: the pinned ring's staging copy (AVX-512 / AVX2 non-temporal stores with plain heads
    and tails, memcpy below 4 KB) at every destination alignment and odd lengths. CPU only."""
    import ctypes as C
    lib = rf.lib()
    fn = getattr(lib, "_ZN5rfgpu16host_stream_copyEPvPKvm")
    fn.restype = None
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
    rng = np.random.default_rng(3)
    src = rng.integers(0, 256, size=(1 << 20) + 64, dtype=np.uint8)
    for off in (0, 1, 8, 31, 33, 63):
        for n in (0, 1, 100, 4095, 4096, 4097, 70001, 1 << 20):
            dst = np.zeros(n + off + 64, dtype=np.uint8)
            fn(dst.ctypes.data + off, src.ctypes.data + 5, n)
            assert np.array_equal(dst[off:off + n], src[5:5 + n])
            assert not dst[:off].any() and not dst[off + n:].any()
