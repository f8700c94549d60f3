"""B200-native randomized range finder — Python host mirror of the reference API.

The product is the CUDA library ``librfgpu.so`` behind the C ABI in
``include/rfgpu.h`` (and the C++ drop-in ``librandfact_b200.so`` for C++
callers of the reference ``randfact`` API). This module binds that C ABI with
ctypes and mirrors the reference entry points (``proj/include/randfact/``):

* :func:`gaussian`       <- ``randfact::gaussian``       (sketch.hpp:25)
* :func:`basic_range`    <- ``randfact::basic_range``    (rangefinder.hpp:50)
* :func:`power_range`    <- ``randfact::power_range``    (rangefinder.hpp:55)
* :func:`rsvd`           <- ``randfact::rsvd``           (lowrank.hpp:15-16)
* :func:`randomized_id`  <- ``randfact::randomized_id``  (lowrank.hpp:78)
* :func:`randomized_cur` <- ``randfact::randomized_cur`` (lowrank.hpp:102)
* :func:`id_deterministic` (column side) <- ``col_id_core`` (lowrank.cpp:51-70)
* :func:`single_pass_svd` <- ``randfact::single_pass_svd`` (lowrank.hpp:41)

Same argument meaning, same defaults, same error classes (``ParameterError``,
``NumericalError``, ``ConvergenceError``, ...). Matrices are numpy arrays in
the reference's column-major layout. There is no CPU fallback: without the
built extension or without a B200 every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
import weakref
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Error", "ParameterError", "NumericalError", "ConvergenceError", "NotPositiveDefiniteError",
    "StreamContractError", "DeviceError", "Context", "DeviceMatrix", "SvdFactors", "RangeBasis", "IdFactors",
    "CurFactors", "gaussian", "basic_range", "power_range", "rsvd", "randomized_id", "randomized_cur",
    "id_deterministic", "single_pass_svd", "MatrixStream", "library_path", "default_context", "row_sketch",
    "multiply", "svd_dense", "frob_residual",
]

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(HERE, "librfgpu.so")


# ----------------------------------------------------------------- errors ---
class Error(RuntimeError):
    """randfact::Error (proj/include/randfact/common.hpp:11-14)."""


class ParameterError(Error):
    pass


class NumericalError(Error):
    pass


class ConvergenceError(NumericalError):
    pass


class NotPositiveDefiniteError(NumericalError):
    pass


class StreamContractError(Error):
    pass


class DeviceError(Error):
    """CUDA / NCCL failure (no reference counterpart: the reference is CPU-only)."""


_ERRORS = {3: ParameterError, 4: NumericalError, 5: ConvergenceError, 6: NotPositiveDefiniteError, 7: DeviceError,
           8: StreamContractError, 9: DeviceError}

# ------------------------------------------------------------------ loader ---
_lib = None
_lib_lock = threading.Lock()

_i64, _u64, _int, _vp = C.c_int64, C.c_uint64, C.c_int, C.c_void_p
_pd, _pf, _pi = C.POINTER(C.c_double), C.POINTER(C.c_float), C.POINTER(C.c_int64)

_SIGS = {
    "rfgpu_last_error": (C.c_char_p, []),
    "rfgpu_version": (_int, []),
    "rfgpu_gaussian": (_int, [_u64, C.c_char_p, _i64, _i64, _pd]),
    "rfgpu_gaussian_range": (_int, [_u64, C.c_char_p, _i64, _i64, _pd]),
    "rfgpu_ctx_create": (_int, [_int, C.POINTER(_vp)]),
    "rfgpu_nccl_unique_id": (_int, [_vp, C.c_size_t]),
    "rfgpu_nccl_selftest": (_int, [_int, _pd, _i64, _pd]),
    "rfgpu_ctx_create_dist": (_int, [_int, _int, _int, _vp, C.c_size_t, C.POINTER(_vp)]),
    "rfgpu_ctx_create_hostsum": (_int, [_int, _int, _int, _vp, _vp, C.POINTER(_vp)]),
    "rfgpu_ctx_destroy": (_int, [_vp]),
    "rfgpu_ctx_release_memory": (_int, [_vp]),
    "rfgpu_ctx_pool_bytes": (_i64, [_vp]),
    "rfgpu_ctx_rank": (_int, [_vp]),
    "rfgpu_ctx_world": (_int, [_vp]),
    "rfgpu_ctx_synchronize": (_int, [_vp]),
    "rfgpu_ctx_stream": (_vp, [_vp]),
    "rfgpu_profile_enable": (_int, [_vp, _int]),
    "rfgpu_profile_reset": (_int, [_vp]),
    "rfgpu_profile_read": (_int, [_vp, C.c_char_p, _pi, _pd]),
    "rfgpu_launch_count": (_i64, [_vp]),
    "rfgpu_matrix_upload": (_int, [_vp, _pd, _i64, _i64, _i64, C.POINTER(_vp)]),
    "rfgpu_matrix_wrap_device": (_int, [_vp, _vp, _i64, _i64, _i64, C.POINTER(_vp)]),
    "rfgpu_matrix_upload_f32": (_int, [_vp, _pf, _i64, _i64, _i64, C.POINTER(_vp)]),
    "rfgpu_matrix_wrap_device_f32": (_int, [_vp, _vp, _i64, _i64, _i64, C.POINTER(_vp)]),
    "rfgpu_matrix_free": (_int, [_vp]),
    "rfgpu_matrix_shape": (_int, [_vp, _pi, _pi, _pi, _pi]),
    "rfgpu_multiply": (_int, [_vp, _vp, _int, _pd, _i64, _pd]),
    "rfgpu_range_finder": (_int, [_vp, _vp, _pd, _i64, _i64, _int, _pd, _pd, _pd, _pi]),
    "rfgpu_rsvd": (_int, [_vp, _vp, _pd, _i64, _i64, _i64, _int, _int, _pd, _pd, _pd, _pi]),
    "rfgpu_rsvd_host": (_int, [_vp, _pd, _i64, _i64, _i64, _pd, _i64, _i64, _i64, _int, _int, _pd, _pd, _pd, _pi]),
    "rfgpu_rsvd_device": (_int, [_vp, _vp, _vp, _i64, _i64, _i64, _int, _int, _vp, _vp, _vp, _pi]),
    "rfgpu_row_sketch": (_int, [_vp, _vp, _pd, _i64, _pd]),
    "rfgpu_row_sketch_device": (_int, [_vp, _vp, _vp, _i64, _vp]),
    "rfgpu_col_id": (_int, [_vp, _pd, _i64, _i64, _i64, _pi, _pd, _pi, C.POINTER(_int)]),
    "rfgpu_col_id_device": (_int, [_vp, _vp, _i64, _i64, _i64, _pi, _vp, _pi, C.POINTER(_int)]),
    "rfgpu_dual_sketch_f32": (_int, [_vp, _vp, _pf, _pf, _i64, _pf, _pf]),
    "rfgpu_single_pass_begin": (_int, [_vp, _i64, _i64, _i64, _pd, _pd, C.POINTER(_vp)]),
    "rfgpu_single_pass_push": (_int, [_vp, _i64, _pd, _i64]),
    "rfgpu_single_pass_finish": (_int, [_vp, _i64, _pd, _pd, _pd, _pi]),
    "rfgpu_single_pass_abort": (_int, [_vp]),
    "rfgpu_single_pass_svd_device": (_int, [_vp, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _pi]),
    "rfgpu_svd": (_int, [_vp, _pd, _i64, _i64, _pd, _pd, _pd, C.POINTER(_int)]),
    "rfgpu_frob_residual": (_int, [_vp, C.c_double, _pd, _i64, _pd]),
    "rfgpu_lowrank_error": (_int, [_vp, _vp, _pd, _pd, _i64, _pd, _i64, _pd, _pd]),
    "rfgpu_randomized_id": (_int, [_vp, _vp, _pd, _i64, _i64, _i64, _pi, _pd, _pi, C.POINTER(_int)]),
    "rfgpu_randomized_cur": (_int, [_vp, _vp, _pd, _i64, _i64, _i64, _pi, _pi, _pd, _pd, _pd, C.POINTER(_int), _pi,
                                     _pi]),
}


def library_path() -> str:
    return _LIB_PATH


def lib():
    """Load librfgpu.so (raises ImportError if it was never built)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(_LIB_PATH):
                raise ImportError(f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                                  f"g.build()'` (there is no CPU fallback)")
            L = C.CDLL(_LIB_PATH)
            for name, (res, args) in _SIGS.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        msg = lib().rfgpu_last_error().decode(errors="replace")
        raise _ERRORS.get(status, Error)(msg)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_pd)


def _fp(a: np.ndarray):
    return a.ctypes.data_as(_pf)


def _ip(a: np.ndarray):
    return a.ctypes.data_as(_pi)


def _fmat(a, dtype=np.float64) -> np.ndarray:
    a = np.asarray(a, dtype=dtype)
    if a.ndim != 2:
        raise ParameterError("expected a 2-D matrix")
    if not np.isfinite(a).all():
        raise ParameterError("from_data: non-finite entry")
    return np.asfortranarray(a)


def _flat(a: np.ndarray) -> np.ndarray:
    return a.reshape(-1, order="F")


# ------------------------------------------------------------------ results ---
@dataclass
class SvdFactors:
    """randfact::SvdFactors (dense.hpp:76-80)."""
    U: np.ndarray
    D: np.ndarray
    V: np.ndarray


@dataclass
class RangeBasis:
    """randfact::RangeBasis (rangefinder.hpp:26-34)."""
    Q: np.ndarray
    B: np.ndarray | None = None
    residual_frob: float | None = None
    picks: list = field(default_factory=list)


@dataclass
class IdFactors:
    """randfact::IdFactors (lowrank.hpp:60-67)."""
    side: str
    Js: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int64))
    Is: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int64))
    Z: np.ndarray = field(default_factory=lambda: np.zeros((0, 0)))
    X: np.ndarray = field(default_factory=lambda: np.zeros((0, 0)))
    rank_truncated: bool = False


@dataclass
class CurFactors:
    """randfact::CurFactors (lowrank.hpp:90-97)."""
    Js: np.ndarray
    Is: np.ndarray
    U: np.ndarray
    cond_C: float
    cond_R: float
    warning: bool


# ------------------------------------------------------------------ context ---
class Context:
    """One GPU (and, for world > 1, one NCCL communicator). Not re-entrant:
    the C layer serialises calls on the same context."""

    HOST_SUM = C.CFUNCTYPE(C.c_int, C.c_void_p, _pd, C.c_int64)

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 host_sum=None):
        """host_sum: optional callable(np.ndarray) -> None that sums the float64
        buffer over all ranks in place (the host-staged reduction backend,
        rfgpu_ctx_create_hostsum); otherwise world > 1 uses NCCL with nccl_id."""
        self._h = _vp()
        self._cb = None
        self._mats = weakref.WeakSet()  # device matrices of this context: freed before the context
        if host_sum is not None:
            def _sum(_user, buf, count):
                try:
                    host_sum(np.ctypeslib.as_array(buf, shape=(count,)))
                    return 0
                except BaseException:  # never unwind through the C library
                    return 1
            self._cb = Context.HOST_SUM(_sum)
            _check(lib().rfgpu_ctx_create_hostsum(device, rank, world, C.cast(self._cb, _vp), None,
                                                  C.byref(self._h)))
        elif world == 1:
            _check(lib().rfgpu_ctx_create(device, C.byref(self._h)))
        else:
            buf = C.create_string_buffer(nccl_id, 128)
            _check(lib().rfgpu_ctx_create_dist(device, rank, world, C.cast(buf, _vp), 128, C.byref(self._h)))
        self.device, self.rank, self.world = device, rank, world

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib().rfgpu_nccl_unique_id(C.cast(buf, _vp), 128))
        return buf.raw

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        return lib().rfgpu_ctx_stream(self._h) or 0

    def synchronize(self):
        _check(lib().rfgpu_ctx_synchronize(self._h))

    def profile(self, on: bool = True):
        _check(lib().rfgpu_profile_enable(self._h, int(on)))

    def profile_reset(self):
        _check(lib().rfgpu_profile_reset(self._h))

    def profile_read(self, name: str) -> tuple[int, float]:
        n, ms = _i64(), C.c_double()
        _check(lib().rfgpu_profile_read(self._h, name.encode(), C.byref(n), C.byref(ms)))
        return n.value, ms.value

    def launch_count(self) -> int:
        return int(lib().rfgpu_launch_count(self._h))

    def release_memory(self):
        """Return the context's cached device memory (pools, host-call A buffer) to the driver."""
        _check(lib().rfgpu_ctx_release_memory(self._h))

    def pool_bytes(self) -> int:
        return int(lib().rfgpu_ctx_pool_bytes(self._h))

    def matrix(self, a, f32: bool = False) -> "DeviceMatrix":
        return DeviceMatrix.upload(self, a, f32=f32)

    def close(self):
        if self._h:
            for mat in list(self._mats):  # a handle must never outlive its context
                mat.free()
            lib().rfgpu_ctx_destroy(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(int(os.environ.get("LOCAL_RANK", "0")))
    return _default_ctx


class DeviceMatrix:
    """Device-resident A (this rank's rows): upload from host or wrap a device pointer."""

    def __init__(self, ctx: Context, handle, m: int, n: int, f32: bool, keep=None):
        self.ctx, self._h, self.f32 = ctx, handle, f32
        self._keep = keep
        ctx._mats.add(self)
        ml, nn, mg, r0 = _i64(), _i64(), _i64(), _i64()
        _check(lib().rfgpu_matrix_shape(handle, C.byref(ml), C.byref(nn), C.byref(mg), C.byref(r0)))
        self.m, self.n, self.m_global, self.row0 = ml.value, nn.value, mg.value, r0.value

    @classmethod
    def upload(cls, ctx: Context, a, f32: bool = False):
        dt = np.float32 if f32 else np.float64
        a = _fmat(a, dt)
        m, n = a.shape
        h = _vp()
        if f32:
            _check(lib().rfgpu_matrix_upload_f32(ctx.handle, _fp(_flat(a)), m, n, max(1, m), C.byref(h)))
        else:
            _check(lib().rfgpu_matrix_upload(ctx.handle, _dp(_flat(a)), m, n, max(1, m), C.byref(h)))
        return cls(ctx, h, m, n, f32)

    @classmethod
    def wrap(cls, ctx: Context, dev_ptr: int, m: int, n: int, lda: int, f32: bool = False, keep=None):
        h = _vp()
        fn = lib().rfgpu_matrix_wrap_device_f32 if f32 else lib().rfgpu_matrix_wrap_device
        _check(fn(ctx.handle, _vp(dev_ptr), m, n, lda, C.byref(h)))
        return cls(ctx, h, m, n, f32, keep=keep)

    @property
    def handle(self):
        return self._h

    def free(self):
        if self._h:
            lib().rfgpu_matrix_free(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


# --------------------------------------------------------------- functions ---
def gaussian(seed: int, tag: str, m: int, n: int) -> np.ndarray:
    """randfact::gaussian(seed, tag, m, n) — bit-identical host generator."""
    if m < 0 or n < 0:
        raise ParameterError("gaussian: negative dimension")
    out = np.empty(m * n)
    _check(lib().rfgpu_gaussian(seed & (2**64 - 1), tag.encode(), m, n, _dp(out)))
    return out.reshape((m, n), order="F")


def _as_device(a, ctx: Context | None):
    if isinstance(a, DeviceMatrix):
        return a, False
    ctx = ctx or default_context()
    return DeviceMatrix.upload(ctx, a), True


def _check_sample(k, p, m, n, where):
    if k < 1:
        raise ParameterError(f"{where}: k must be at least 1")
    if p < 0:
        raise ParameterError(f"{where}: p must be non-negative")
    if k + p > min(m, n):
        raise ParameterError(f"{where}: k + p exceeds min(m, n)")


def power_range(a, k: int, p: int = 10, q: int = 0, seed: int = 0, reorthonormalize: bool = False,
                ctx: Context | None = None) -> RangeBasis:
    """randfact::power_range(a, RangeConfig{k, p, q, reorthonormalize, seed})."""
    if q < 0:
        raise ParameterError("power_range: q must be non-negative")
    dm, tmp = _as_device(a, ctx)
    try:
        _check_sample(k, p, dm.m_global, dm.n, "power_range")
        ell = k + p
        g = gaussian(seed, "range.G", dm.n, ell)
        Q = np.zeros(max(1, dm.m * ell))
        B = np.zeros(max(1, ell * dm.n))
        res, r = C.c_double(), _i64()
        _check(lib().rfgpu_range_finder(dm.ctx.handle, dm.handle, _dp(_flat(g)), ell, q, int(reorthonormalize),
                                        _dp(Q), _dp(B), C.byref(res), C.byref(r)))
        rr = r.value
        return RangeBasis(Q[: dm.m * rr].reshape((dm.m, rr), order="F"),
                          B[: rr * dm.n].reshape((rr, dm.n), order="F"), res.value)
    finally:
        if tmp:
            dm.free()


def basic_range(a, k: int, p: int = 10, seed: int = 0, q: int = 0, ctx: Context | None = None) -> RangeBasis:
    """randfact::basic_range (requires q == 0): bitwise power_range with q = 0."""
    if q != 0:
        raise ParameterError("basic_range: q must be 0 (use power_range)")
    return power_range(a, k, p, 0, seed, False, ctx)


def rsvd(a, k: int, p: int, q: int, seed: int, keep_oversamples: bool = False, reorthonormalize: bool = False,
         ctx: Context | None = None) -> SvdFactors:
    """randfact::rsvd(a, k, p, q, seed, keep_oversamples, reorthonormalize)."""
    if q < 0:
        raise ParameterError("power_range: q must be non-negative")
    if not isinstance(a, DeviceMatrix):
        # host matrix: one call that streams A in behind the first pass
        if k < 1 or p < 0:
            _check_sample(k, p, k + max(p, 0), k + max(p, 0), "power_range")
        ctx = ctx or default_context()
        a = _fmat(a)
        m, n = a.shape
        ell = k + p
        g = gaussian(seed, "range.G", n, ell)
        U = np.zeros(max(1, m * ell))
        D = np.zeros(ell)
        V = np.zeros(max(1, n * ell))
        r = _i64()
        _check(lib().rfgpu_rsvd_host(ctx.handle, _dp(_flat(a)), m, n, max(1, m), _dp(_flat(g)), k, ell, q,
                                     int(keep_oversamples), int(reorthonormalize), _dp(U), _dp(D), _dp(V),
                                     C.byref(r)))
        rr = r.value
        return SvdFactors(U[: m * rr].reshape((m, rr), order="F"), D[:rr].copy(),
                          V[: n * rr].reshape((n, rr), order="F"))
    dm, tmp = _as_device(a, ctx)
    try:
        _check_sample(k, p, dm.m_global, dm.n, "power_range")
        ell = k + p
        g = gaussian(seed, "range.G", dm.n, ell)
        U = np.zeros(max(1, dm.m * ell))
        D = np.zeros(ell)
        V = np.zeros(max(1, dm.n * ell))
        r = _i64()
        _check(lib().rfgpu_rsvd(dm.ctx.handle, dm.handle, _dp(_flat(g)), k, ell, q, int(keep_oversamples),
                                int(reorthonormalize), _dp(U), _dp(D), _dp(V), C.byref(r)))
        rr = r.value
        return SvdFactors(U[: dm.m * rr].reshape((dm.m, rr), order="F"), D[:rr].copy(),
                          V[: dm.n * rr].reshape((dm.n, rr), order="F"))
    finally:
        if tmp:
            dm.free()


def multiply(a, x, trans: bool = False, ctx: Context | None = None) -> np.ndarray:
    """C = A X (trans=False) or A^T X on the device (randfact::multiply for the pass shapes)."""
    dm, tmp = _as_device(a, ctx)
    try:
        x = _fmat(x)
        rows_out = dm.n if trans else dm.m
        out = np.zeros(max(1, rows_out * x.shape[1]))
        _check(lib().rfgpu_multiply(dm.ctx.handle, dm.handle, int(trans), _dp(_flat(x)), x.shape[1], _dp(out)))
        return out[: rows_out * x.shape[1]].reshape((rows_out, x.shape[1]), order="F")
    finally:
        if tmp:
            dm.free()


def svd_dense(a, ctx: Context | None = None) -> SvdFactors:
    """randfact::svd_dense (dense.hpp:117) on the device: thin SVD, D non-increasing."""
    a = _fmat(a)
    m, n = a.shape
    wide = m < n
    x = np.asfortranarray(a.T) if wide else a
    r, c = x.shape
    ctx = ctx or default_context()
    U, S, V = np.zeros(r * c), np.zeros(c), np.zeros(c * c)
    sw = C.c_int()
    _check(lib().rfgpu_svd(ctx.handle, _dp(_flat(x)), r, c, _dp(U), _dp(S), _dp(V), C.byref(sw)))
    U, V = U.reshape((r, c), order="F"), V.reshape((c, c), order="F")
    return SvdFactors(V, S, U) if wide else SvdFactors(U, S, V)


def frob_residual(a_frob: float, b, ctx: Context | None = None) -> float:
    """randfact::frob_residual(a_frob, B) (rangefinder.cpp:45-54): ||B||_F summed on the device."""
    if not (a_frob >= 0.0):
        raise ParameterError("frob_residual: norm must be non-negative")
    b = _fmat(b)
    ctx = ctx or default_context()
    out = C.c_double()
    _check(lib().rfgpu_frob_residual(ctx.handle, float(a_frob), _dp(_flat(b)), b.size, C.byref(out)))
    return out.value


def id_deterministic(a, k: int, side: str = "Col", ctx: Context | None = None) -> IdFactors:
    """randfact::id_deterministic(a, k, IdSide::Col) — the column ID core on the device."""
    if side != "Col":
        raise ParameterError("id_deterministic: only IdSide::Col is on the device path")
    a = _fmat(a)
    m, n = a.shape
    if k < 1:
        raise ParameterError("id_deterministic: k must be at least 1")
    if k > min(m, n):
        raise ParameterError("id_deterministic: k exceeds min(m, n)")
    ctx = ctx or default_context()
    js = np.zeros(k, dtype=np.int64)
    z = np.zeros(k * n)
    r, tr = _i64(), C.c_int()
    _check(lib().rfgpu_col_id(ctx.handle, _dp(_flat(a)), m, n, k, _ip(js), _dp(z), C.byref(r), C.byref(tr)))
    ke = r.value
    return IdFactors("Col", Js=js[:ke].copy(), Z=z[: ke * n].reshape((ke, n), order="F"),
                     rank_truncated=bool(tr.value))


def randomized_id(a, k: int, p: int, q: int, seed: int, ctx: Context | None = None) -> IdFactors:
    """randfact::randomized_id(a, k, p, q, seed): row ID from the tall sketch."""
    dm, tmp = _as_device(a, ctx)
    try:
        _check_sample(k, p, dm.m_global, dm.n, "randomized_id")
        if q < 0:
            raise ParameterError("randomized_id: q must be non-negative")
        ell = k + p
        g = gaussian(seed, "rid.G", dm.n, ell)
        is_ = np.zeros(k, dtype=np.int64)
        x = np.zeros(dm.m * k)
        r, tr = _i64(), C.c_int()
        _check(lib().rfgpu_randomized_id(dm.ctx.handle, dm.handle, _dp(_flat(g)), k, ell, q, _ip(is_), _dp(x),
                                         C.byref(r), C.byref(tr)))
        ke = r.value
        return IdFactors("Row", Is=is_[:ke].copy(), X=x[: dm.m * ke].reshape((dm.m, ke), order="F"),
                         rank_truncated=bool(tr.value))
    finally:
        if tmp:
            dm.free()


def randomized_cur(a, k: int, p: int, q: int, seed: int, ctx: Context | None = None) -> CurFactors:
    """randfact::randomized_cur(a, k, p, q, seed)."""
    dm, tmp = _as_device(a, ctx)
    try:
        _check_sample(k, p, dm.m_global, dm.n, "randomized_cur")
        if q < 0:
            raise ParameterError("randomized_cur: q must be non-negative")
        ell = k + p
        g = gaussian(seed, "cur.G", ell, dm.m_global)
        js, is_ = np.zeros(k, dtype=np.int64), np.zeros(k, dtype=np.int64)
        u = np.zeros(k * k)
        cc, cr, w = C.c_double(), C.c_double(), C.c_int()
        kc, kr = _i64(), _i64()
        _check(lib().rfgpu_randomized_cur(dm.ctx.handle, dm.handle, _dp(_flat(g)), k, ell, q, _ip(js), _ip(is_),
                                          _dp(u), C.byref(cc), C.byref(cr), C.byref(w), C.byref(kc), C.byref(kr)))
        return CurFactors(js[: kc.value].copy(), is_[: kr.value].copy(),
                          u[: kc.value * kr.value].reshape((kc.value, kr.value), order="F"), cc.value, cr.value,
                          bool(w.value))
    finally:
        if tmp:
            dm.free()


def row_sketch(a, ell: int, seed: int, ctx: Context | None = None) -> np.ndarray:
    """Y = G A with G = gaussian(seed, "cur.G", ell, m) (randomized_cur's pass over A)."""
    dm, tmp = _as_device(a, ctx)
    try:
        g = gaussian(seed, "cur.G", ell, dm.m_global)
        y = np.zeros(ell * dm.n)
        _check(lib().rfgpu_row_sketch(dm.ctx.handle, dm.handle, _dp(_flat(g)), ell, _dp(y)))
        return y.reshape((ell, dm.n), order="F")
    finally:
        if tmp:
            dm.free()


class MatrixStream:
    """randfact::MatrixStream (stream.hpp:13-41): one-shot column-block view."""

    def __init__(self, a, block_cols: int = 32):
        if block_cols < 1:
            raise ParameterError("MatrixStream: block width must be positive")
        self.a = _fmat(a)
        self.block_cols = block_cols
        self.next_col = 0
        self.entries_served = 0

    def rows(self):
        return self.a.shape[0]

    def cols(self):
        return self.a.shape[1]

    def has_next(self):
        return self.next_col < self.a.shape[1]

    def next_block(self):
        if self.next_col >= self.a.shape[1]:
            raise StreamContractError("MatrixStream: single pass already consumed")
        c0 = self.next_col
        c1 = min(self.a.shape[1], c0 + self.block_cols)
        self.next_col = c1
        self.entries_served += self.a.shape[0] * (c1 - c0)
        return c0, self.a[:, c0:c1]

    def passes_completed(self):
        return 1 if self.next_col >= self.a.shape[1] else 0


def single_pass_svd(stream: MatrixStream, k: int, p: int, seed: int, ctx: Context | None = None,
                    m_global: int | None = None) -> SvdFactors:
    """randfact::single_pass_svd(stream, k, p, seed): one traversal of the stream;
    every block is pushed to the device once (Yc += A_blk Gc_blk, Yr_blk = A_blk^T Gr)
    and the core is solved on the device. On a multi-rank context the stream
    holds this rank's rows of A and m_global is the row count of the whole A
    (Gr is drawn for all of it; each rank uses its rows)."""
    m, n = stream.rows(), stream.cols()
    mg = m if m_global is None else m_global
    _check_sample(k, p, mg, n, "single_pass_svd")
    ctx = ctx or default_context()
    ell = k + p
    gc = gaussian(seed, "spsvd.Gc", n, ell)
    gr = gaussian(seed, "spsvd.Gr", mg, ell)
    h = _vp()
    _check(lib().rfgpu_single_pass_begin(ctx.handle, m, n, ell, _dp(_flat(gc)), _dp(_flat(gr)), C.byref(h)))
    try:
        while stream.has_next():
            c0, blk = stream.next_block()
            blk = np.asfortranarray(blk)
            _check(lib().rfgpu_single_pass_push(h, c0, _dp(_flat(blk)), blk.shape[1]))
    except BaseException:
        lib().rfgpu_single_pass_abort(h)
        raise
    kk = min(k, ell)
    U, D, V = np.zeros(m * kk), np.zeros(kk), np.zeros(n * kk)
    r = _i64()
    _check(lib().rfgpu_single_pass_finish(h, k, _dp(U), _dp(D), _dp(V), C.byref(r)))
    rr = r.value
    return SvdFactors(U[: m * rr].reshape((m, rr), order="F"), D[:rr].copy(), V[: n * rr].reshape((n, rr), order="F"))
