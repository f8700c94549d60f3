"""TEST INFRASTRUCTURE ONLY — CPU checkers for the randomized range-finder path.

Two independent CPU implementations, both loaded through ctypes:

* ``Oracle("port")``      -> ``oracle/_build/librforacle.so``: the plain-C
  restatement (``oracle/rf_oracle.c``) of the reference algorithms, written to
  reproduce the reference's floating-point order.
* ``Oracle("reference")`` -> ``oracle/_ref/librfref.so``: the unmodified
  reference sources (``/root/reference/proj/src``) compiled by
  ``oracle/Makefile`` with the ``ref_shim.cpp`` C entry points.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg
and ``--impl reference``) may import this module; the product path
(``paper_1607_01649_b200``) never does.

Both expose the same numpy-level API, named after the reference functions
(``proj/include/randfact/*.hpp``) and raising the same error classes as the
product wrapper so parity tests read like the reference's own tests.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "port": os.path.join(HERE, "_build", "librforacle.so"),
    "reference": os.path.join(HERE, "_ref", "librfref.so"),
}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_i64 = C.c_int64
_u64 = C.c_uint64
_pd = C.POINTER(C.c_double)
_pi = C.POINTER(C.c_int64)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_pd)


def _ip(a: np.ndarray):
    return a.ctypes.data_as(_pi)


def fmat(a) -> np.ndarray:
    """Column-major float64 copy (the reference DenseMatrix layout)."""
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _flat(a: np.ndarray) -> np.ndarray:
    return np.asfortranarray(a).reshape(-1, order="F")


@dataclass
class Svd:
    U: np.ndarray
    D: np.ndarray
    V: np.ndarray


@dataclass
class Range:
    Q: np.ndarray
    B: np.ndarray
    residual_frob: float


@dataclass
class Cur:
    Js: np.ndarray
    Is: np.ndarray
    U: np.ndarray
    cond_C: float
    cond_R: float
    warning: bool


class Oracle:
    def __init__(self, kind: str = "port"):
        path = LIBS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
        self.kind = kind
        self.lib = C.CDLL(path)
        self.p = "rfo_" if kind == "port" else "rfref_"
        self._err = getattr(self.lib, self.p + "last_error")
        self._err.restype = C.c_char_p

    def _fn(self, name):
        f = getattr(self.lib, self.p + name)
        f.restype = C.c_int
        return f

    def _check(self, st: int):
        if st != 0:
            raise OracleError(st, self._err().decode())

    def set_threads(self, n: int):
        getattr(self.lib, self.p + "set_threads")(C.c_int(n))

    # ---------------------------------------------------------------- rng
    def gaussian(self, seed: int, tag: str, m: int, n: int) -> np.ndarray:
        out = np.empty(m * n)
        self._check(self._fn("gaussian")(_u64(seed), tag.encode(), _i64(m), _i64(n), _dp(out)))
        return out.reshape((m, n), order="F")

    def planted(self, m: int, n: int, sigma, seed: int) -> np.ndarray:
        s = np.ascontiguousarray(sigma, dtype=np.float64)
        out = np.empty(m * n)
        self._check(self._fn("planted")(_i64(m), _i64(n), _dp(s), _i64(len(s)), _u64(seed), _dp(out)))
        return out.reshape((m, n), order="F")

    def test_planted(self, m: int, n: int, sigma, seed: int) -> np.ndarray:
        """The reference test suite's planted() (tests/test_support.hpp:37-46; reference only)."""
        s = np.ascontiguousarray(sigma, dtype=np.float64)
        out = np.empty(m * n)
        self._check(self._fn("test_planted")(_i64(m), _i64(n), _dp(s), _i64(len(s)), _u64(seed), _dp(out)))
        return out.reshape((m, n), order="F")

    # ---------------------------------------------------------------- dense
    def multiply(self, a, b, ta=False, tb=False) -> np.ndarray:
        a, b = fmat(a), fmat(b)
        m = a.shape[1] if ta else a.shape[0]
        n = b.shape[0] if tb else b.shape[1]
        out = np.zeros(m * n)
        self._check(self._fn("multiply")(_dp(_flat(a)), _i64(a.shape[0]), _i64(a.shape[1]),
                                         _dp(_flat(b)), _i64(b.shape[0]), _i64(b.shape[1]),
                                         C.c_int(int(ta)), C.c_int(int(tb)), _dp(out)))
        return out.reshape((m, n), order="F")

    def orth(self, x) -> np.ndarray:
        x = fmat(x)
        m, n = x.shape
        out = np.zeros(m * n)
        r = _i64()
        self._check(self._fn("orth")(_dp(_flat(x)), _i64(m), _i64(n), _dp(out), C.byref(r)))
        return out[: m * r.value].reshape((m, r.value), order="F")

    def svd(self, a) -> Svd:
        a = fmat(a)
        m, n = a.shape
        r = min(m, n)
        U, D, V = np.zeros(m * r), np.zeros(r), np.zeros(n * r)
        self._check(self._fn("svd")(_dp(_flat(a)), _i64(m), _i64(n), _dp(U), _dp(D), _dp(V)))
        return Svd(U.reshape((m, r), order="F"), D, V.reshape((n, r), order="F"))

    def cpqr_rank(self, a, k: int):
        """Returns (perm, R (rank x n), stopped_rank)."""
        a = fmat(a)
        m, n = a.shape
        perm = np.zeros(n, dtype=np.int64)
        rank = _i64()
        if self.kind == "port":
            R = np.zeros(max(k, 1) * n)
            self._check(self._fn("cpqr_rank")(_dp(_flat(a)), _i64(m), _i64(n), _i64(k), _ip(perm),
                                              _dp(R), C.byref(rank)))
            Rm = R[: k * n].reshape((k, n), order="F")[: rank.value]
        else:
            R = np.zeros(max(k, 1) * n)
            Q = np.zeros(m * max(k, 1))
            res = C.c_double()
            self._check(self._fn("cpqr_rank")(_dp(_flat(a)), _i64(m), _i64(n), _i64(k), _ip(perm), _dp(R),
                                              _dp(Q), C.byref(rank), C.byref(res)))
            Rm = R[: rank.value * n].reshape((rank.value, n), order="F")
        return perm, Rm, rank.value

    # ------------------------------------------------------------ algorithms
    def power_range(self, a, k, p, q, seed, reorth=False, basic=False) -> Range:
        a = fmat(a)
        m, n = a.shape
        ell = k + p
        Q, B = np.zeros(m * max(ell, 1)), np.zeros(max(ell, 1) * n)
        res, r = C.c_double(), _i64()
        self._check(self._fn("power_range")(_dp(_flat(a)), _i64(m), _i64(n), _i64(k), _i64(p), _i64(q),
                                            C.c_int(int(reorth)), _u64(seed), C.c_int(int(basic)),
                                            _dp(Q), _dp(B), C.byref(res), C.byref(r)))
        rr = r.value
        return Range(Q[: m * rr].reshape((m, rr), order="F"), B[: rr * n].reshape((rr, n), order="F"),
                     res.value)

    def basic_range(self, a, k, p, seed) -> Range:
        return self.power_range(a, k, p, 0, seed, reorth=False, basic=True)

    def rsvd(self, a, k, p, q, seed, keep_oversamples=False, reorthonormalize=False) -> Svd:
        a = fmat(a)
        m, n = a.shape
        ell = max(k + p, 1)
        U, D, V = np.zeros(m * ell), np.zeros(ell), np.zeros(n * ell)
        r = _i64()
        self._check(self._fn("rsvd")(_dp(_flat(a)), _i64(m), _i64(n), _i64(k), _i64(p), _i64(q), _u64(seed),
                                     C.c_int(int(keep_oversamples)), C.c_int(int(reorthonormalize)),
                                     _dp(U), _dp(D), _dp(V), C.byref(r)))
        rr = r.value
        return Svd(U[: m * rr].reshape((m, rr), order="F"), D[:rr].copy(), V[: n * rr].reshape((n, rr), order="F"))

    def id_col(self, a, k):
        """id_deterministic(a, k, IdSide::Col) == col_id_core. (Js, Z, truncated)."""
        a = fmat(a)
        m, n = a.shape
        js = np.zeros(max(k, 1), dtype=np.int64)
        z = np.zeros(max(k, 1) * n)
        r, tr = _i64(), C.c_int()
        fn = "col_id" if self.kind == "port" else "id_col"
        self._check(self._fn(fn)(_dp(_flat(a)), _i64(m), _i64(n), _i64(k), _ip(js), _dp(z), C.byref(r),
                                 C.byref(tr)))
        ke = r.value
        return js[:ke].copy(), z[: ke * n].reshape((ke, n), order="F"), bool(tr.value)

    def randomized_id(self, a, k, p, q, seed):
        """(Is, X (m x ke), truncated)."""
        a = fmat(a)
        m, n = a.shape
        is_ = np.zeros(max(k, 1), dtype=np.int64)
        x = np.zeros(m * max(k, 1))
        r, tr = _i64(), C.c_int()
        self._check(self._fn("randomized_id")(_dp(_flat(a)), _i64(m), _i64(n), _i64(k), _i64(p), _i64(q),
                                              _u64(seed), _ip(is_), _dp(x), C.byref(r), C.byref(tr)))
        ke = r.value
        return is_[:ke].copy(), x[: m * ke].reshape((m, ke), order="F"), bool(tr.value)

    def cur_col_id(self, a, k, p, seed):
        """Column-ID part of randomized_cur (port only): (Js, Z, truncated, Y)."""
        if self.kind != "port":
            g = self.gaussian(seed, "cur.G", k + p, a.shape[0])
            y = self.multiply(g, a)
            js, z, tr = self.id_col(y, k)
            return js, z, tr, y
        a = fmat(a)
        m, n = a.shape
        ell = k + p
        js = np.zeros(k, dtype=np.int64)
        z = np.zeros(k * n)
        y = np.zeros(ell * n)
        r, tr = _i64(), C.c_int()
        self._check(self._fn("cur_col_id")(_dp(_flat(a)), _i64(m), _i64(n), _i64(k), _i64(p), _u64(seed),
                                           _ip(js), _dp(z), C.byref(r), C.byref(tr), _dp(y)))
        ke = r.value
        return js[:ke].copy(), z[: ke * n].reshape((ke, n), order="F"), bool(tr.value), y.reshape((ell, n), order="F")

    def randomized_cur(self, a, k, p, q, seed) -> Cur:
        a = fmat(a)
        m, n = a.shape
        js, is_ = np.zeros(k, dtype=np.int64), np.zeros(k, dtype=np.int64)
        u = np.zeros(k * k)
        cc, cr, w = C.c_double(), C.c_double(), C.c_int()
        kc, kr = _i64(), _i64()
        if self.kind == "port":
            if q != 0:
                raise OracleError(3, "port restates randomized_cur for q = 0 only")
            st = self._fn("randomized_cur")(_dp(_flat(a)), _i64(m), _i64(n), _i64(k), _i64(p), _u64(seed),
                                            _ip(js), _ip(is_), _dp(u), C.byref(cc), C.byref(cr), C.byref(w),
                                            C.byref(kc), C.byref(kr))
        else:
            st = self._fn("randomized_cur")(_dp(_flat(a)), _i64(m), _i64(n), _i64(k), _i64(p), _i64(q),
                                            _u64(seed), _ip(js), _ip(is_), _dp(u), C.byref(cc), C.byref(cr),
                                            C.byref(w), C.byref(kc), C.byref(kr))
        self._check(st)
        return Cur(js[: kc.value].copy(), is_[: kr.value].copy(),
                   u[: kc.value * kr.value].reshape((kc.value, kr.value), order="F"),
                   cc.value, cr.value, bool(w.value))

    def single_pass_svd(self, a, k, p, seed, block=32) -> Svd:
        a = fmat(a)
        m, n = a.shape
        ell = k + p
        U, D, V = np.zeros(m * ell), np.zeros(ell), np.zeros(n * ell)
        r = _i64()
        if self.kind == "port":
            st = self._fn("single_pass_svd")(_dp(_flat(a)), _i64(m), _i64(n), _i64(k), _i64(p), _u64(seed),
                                             _i64(block), _dp(U), _dp(D), _dp(V), C.byref(r))
        else:
            es, ps = _u64(), C.c_int()
            st = self._fn("single_pass_svd")(_dp(_flat(a)), _i64(m), _i64(n), _i64(k), _i64(p), _u64(seed),
                                             _i64(block), _dp(U), _dp(D), _dp(V), C.byref(r), C.byref(es),
                                             C.byref(ps))
        self._check(st)
        rr = r.value
        return Svd(U[: m * rr].reshape((m, rr), order="F"), D[:rr].copy(), V[: n * rr].reshape((n, rr), order="F"))

    def read_matrix(self, path: str):
        """reference read_matrix (matrix_io.cpp) -> (status, message, array or None) (reference only)."""
        rows, cols, data = _i64(), _i64(), C.POINTER(C.c_double)()
        st = self._fn("read_matrix")(path.encode(), C.byref(rows), C.byref(cols), C.byref(data))
        if st != 0:
            return st, self._err().decode(), None
        m, n = rows.value, cols.value
        arr = np.ctypeslib.as_array(data, shape=(max(1, m * n),))[: m * n].copy().reshape((m, n), order="F")
        self.lib.rfref_free(data)
        return 0, "", arr

    def write_matrix(self, path: str, a) -> tuple[int, str]:
        a = fmat(a)
        st = self._fn("write_matrix")(path.encode(), _dp(_flat(a)), _i64(a.shape[0]), _i64(a.shape[1]))
        return st, (self._err().decode() if st else "")

    def dual_sketch(self, a, gc, gr, block=32):
        """(Yc = A Gc, Yr = A^T Gr) accumulated in MatrixStream block order (port only)."""
        a, gc, gr = fmat(a), fmat(gc), fmat(gr)
        m, n = a.shape
        ell = gc.shape[1]
        yc, yr = np.zeros(m * ell), np.zeros(n * ell)
        self._check(self._fn("dual_sketch")(_dp(_flat(a)), _i64(m), _i64(n), _dp(_flat(gc)), _dp(_flat(gr)),
                                            _i64(ell), _i64(block), _dp(yc), _dp(yr)))
        return yc.reshape((m, ell), order="F"), yr.reshape((n, ell), order="F")


_cache: dict[str, Oracle] = {}


def get(kind: str = "port") -> Oracle:
    if kind not in _cache:
        _cache[kind] = Oracle(kind)
    return _cache[kind]
