"""CPU oracle for the rsvd hot path — TEST INFRASTRUCTURE ONLY.

ctypes front end of oracle/_build/liboracle_rsvd.so (built from
oracle/rsvd_oracle.cpp by oracle/Makefile).  Only tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline / reference arm may import this package; the
product path (paper_2402_17794_b200 + librsvd_b200.so) never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle_rsvd.so")

BASIC, POWER, POWER_ORTHO = 0, 1, 2


class OracleError(RuntimeError):
    pass


class DimensionError(OracleError):
    pass


class ParameterError(OracleError):
    pass


class NumericError(OracleError):
    pass


_ERRS = {1: DimensionError, 2: ParameterError, 3: NumericError}


class RngState(ctypes.Structure):
    """Same layout as rsvd_rng_state in include/rsvd_b200.h."""
    _fields_ = [("mt", ctypes.c_uint64 * 312), ("pos", ctypes.c_uint64),
                ("has_cached", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("cached", ctypes.c_double)]


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P, I64, I, U64, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint64, ctypes.c_double
        L.orc_last_error.restype = ctypes.c_char_p
        L.orc_rng_new.restype = P
        L.orc_rng_new.argtypes = [U64]
        L.orc_rng_free.argtypes = [P]
        L.orc_rng_normal.restype = D
        L.orc_rng_normal.argtypes = [P]
        L.orc_rng_raw.restype = U64
        L.orc_rng_raw.argtypes = [P]
        L.orc_polar_r2_log.argtypes = [P, ctypes.c_int64, P, P]
        L.orc_polar_r2_log.restype = None
        L.orc_rng_get_state.argtypes = [P, ctypes.POINTER(RngState)]
        L.orc_rng_set_state.argtypes = [P, ctypes.POINTER(RngState)]
        L.orc_set_threads.argtypes = [I]
        L.orc_compiler.restype = ctypes.c_char_p
        L.orc_gaussian.argtypes = [I64, I64, P, P]
        L.orc_gemm.argtypes = [I64, I64, I64, P, I, P, I, P]
        L.orc_orthonormalize.argtypes = [I64, I64, P, P]
        L.orc_svd_small.argtypes = [I64, I64, P, P, P, P]
        L.orc_evd_symmetric.argtypes = [I64, P, P, P]
        L.orc_solve_ls.argtypes = [I64, I64, P, I64, P, P]
        L.orc_range_basis.argtypes = [I64, I64, P, I64, I64, I, I, P, P]
        L.orc_rsvd.argtypes = [I64, I64, P, I64, I64, I, I, P, P, P, P]
        L.orc_spevd.argtypes = [I64, P, I64, I64, P, P, P, ctypes.POINTER(I)]
        L.orc_spsvd.argtypes = [I64, I64, P, I64, I64, P, P, P, P, ctypes.POINTER(I), ctypes.POINTER(I)]
        L.orc_solve_joint_core.argtypes = [I64, P, P, P, P, I, P]
        L.orc_singular_values.argtypes = [I64, I64, P, P]
        L.orc_spectral_norm.argtypes = [I64, I64, P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I)]
        L.orc_computed_range_error.argtypes = [I64, I64, P, I64, P, ctypes.POINTER(ctypes.c_double)]
        L.orc_canonical_sines.argtypes = [I64, I64, P, I64, P, P]
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        msg = lib().orc_last_error().decode()
        raise _ERRS.get(rc, OracleError)(msg)


def _f(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def compiler() -> str:
    return lib().orc_compiler().decode()


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


class Rng:
    """The reference's rsvd::Rng (sketch.hpp:19-45): std::mt19937_64 +
    std::normal_distribution<double> from the host libstdc++."""

    def __init__(self, seed: int):
        self._h = lib().orc_rng_new(ctypes.c_uint64(seed & (2**64 - 1)))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_rng_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def normal(self) -> float:
        return lib().orc_rng_normal(self._h)

    def raw(self) -> int:
        return lib().orc_rng_raw(self._h)

    def polar_r2_log(self, count: int):
        """(r2, glibc log(r2)) of the next `count` accepted polar attempts."""
        r2 = np.empty(count)
        lg = np.empty(count)
        lib().orc_polar_r2_log(self._h, count, _p(r2), _p(lg))
        return r2, lg

    def get_state(self) -> RngState:
        st = RngState()
        lib().orc_rng_get_state(self._h, ctypes.byref(st))
        return st

    def set_state(self, st: RngState) -> None:
        lib().orc_rng_set_state(self._h, ctypes.byref(st))


def gaussian(n: int, l: int, rng: Rng) -> np.ndarray:
    out = np.empty((max(n, 0), max(l, 0)), dtype=np.float64, order="F")
    _check(lib().orc_gaussian(n, l, rng.handle, _p(out)))
    return out


def gemm(a, b, ta=False, tb=False):
    a, b = _f(a), _f(b)
    m = a.shape[1] if ta else a.shape[0]
    k = a.shape[0] if ta else a.shape[1]
    n = b.shape[0] if tb else b.shape[1]
    c = np.empty((m, n), order="F")
    _check(lib().orc_gemm(m, n, k, _p(a), int(ta), _p(b), int(tb), _p(c)))
    return c


def orthonormalize(m) -> np.ndarray:
    m = _f(m)
    q = np.empty_like(m, order="F")
    _check(lib().orc_orthonormalize(m.shape[0], m.shape[1], _p(m), _p(q)))
    return q


def svd_small(m):
    m = _f(m)
    r = min(m.shape)
    u = np.empty((m.shape[0], r), order="F")
    s = np.empty(r)
    v = np.empty((m.shape[1], r), order="F")
    _check(lib().orc_svd_small(m.shape[0], m.shape[1], _p(m), _p(u), _p(s), _p(v)))
    return u, s, v


def evd_symmetric(c):
    c = _f(c)
    if c.ndim != 2 or c.shape[0] != c.shape[1]:
        raise DimensionError("evd_symmetric: matrix is not square")
    n = c.shape[0]
    u = np.empty((n, n), order="F")
    lam = np.empty(n)
    _check(lib().orc_evd_symmetric(n, _p(c), _p(u), _p(lam)))
    return u, lam


def solve_ls(g, h):
    g, h = _f(g), _f(h)
    x = np.empty((g.shape[1], h.shape[1]), order="F")
    if g.shape[0] != h.shape[0]:
        raise DimensionError("solve_ls: row counts differ")
    _check(lib().orc_solve_ls(g.shape[0], g.shape[1], _p(g), h.shape[1], _p(h), _p(x)))
    return x


def range_basis(a, k, p, q, mode, rng: Rng):
    a = _f(a)
    out = np.empty((a.shape[0], max(k + p, 0)), order="F")
    _check(lib().orc_range_basis(a.shape[0], a.shape[1], _p(a), k, p, q, mode, rng.handle, _p(out)))
    return out


def rsvd(a, k, p, q, mode, rng: Rng):
    a = _f(a)
    l = k + p
    u = np.empty((a.shape[0], max(l, 0)), order="F")
    s = np.empty(max(l, 0))
    v = np.empty((a.shape[1], max(l, 0)), order="F")
    _check(lib().orc_rsvd(a.shape[0], a.shape[1], _p(a), k, p, q, mode, rng.handle, _p(u), _p(s), _p(v)))
    return u, s, v


def spevd_hermitian(a, k, p, rng: Rng, counters=None):
    a = _f(a)
    n = a.shape[0]
    u = np.empty((n, max(k, 0)), order="F")
    lam = np.empty(max(k, 0))
    applies = ctypes.c_int(0)
    if a.shape[0] != a.shape[1]:
        raise DimensionError("spevd_hermitian: matrix is not square")
    _check(lib().orc_spevd(n, _p(a), k, p, rng.handle, _p(u), _p(lam), ctypes.byref(applies)))
    if counters is not None:
        counters["apply"] = applies.value
    return u, lam


def spsvd_general(a, k, p, rng: Rng, counters=None):
    a = _f(a)
    m, n = a.shape
    u = np.empty((m, max(k, 0)), order="F")
    s = np.empty(max(k, 0))
    v = np.empty((n, max(k, 0)), order="F")
    ap, ad = ctypes.c_int(0), ctypes.c_int(0)
    _check(lib().orc_spsvd(m, n, _p(a), k, p, rng.handle, _p(u), _p(s), _p(v), ctypes.byref(ap), ctypes.byref(ad)))
    if counters is not None:
        counters["apply"], counters["adjoint"] = ap.value, ad.value
    return u, s, v


def solve_joint_core(g1, h1, g2, h2, route: int = 2):
    """route 0 = literal stacked (singlepass.hpp:84-101), 1 = Kronecker, 2 = auto."""
    g1, h1, g2, h2 = map(_f, (g1, h1, g2, h2))
    l = g1.shape[0]
    c = np.empty((l, l), order="F")
    _check(lib().orc_solve_joint_core(l, _p(g1), _p(h1), _p(g2), _p(h2), route, _p(c)))
    return c


# ------------------------------------------------ diagnostics (core/bounds/angles)
def singular_values(m):
    """reference core.hpp:180-183"""
    m = _f(m)
    s = np.empty(min(m.shape))
    _check(lib().orc_singular_values(m.shape[0], m.shape[1], _p(m), _p(s)))
    return s


def spectral_norm(m, with_iterations=False):
    """reference core.hpp:188-221"""
    m = _f(m)
    out, it = ctypes.c_double(0.0), ctypes.c_int(0)
    _check(lib().orc_spectral_norm(m.shape[0], m.shape[1], _p(m), ctypes.byref(out), ctypes.byref(it)))
    return (out.value, it.value) if with_iterations else out.value


def computed_range_error(a, q):
    """reference bounds.hpp:107-120"""
    a, q = _f(a), _f(q)
    if a.shape[0] != q.shape[0]:
        raise DimensionError("computed_range_error: row counts differ")
    out = ctypes.c_double(0.0)
    _check(lib().orc_computed_range_error(a.shape[0], a.shape[1], _p(a), q.shape[1], _p(q),
                                          ctypes.byref(out)))
    return out.value


def canonical_sines(x, y):
    """reference angles.hpp:42-60"""
    x, y = _f(x), _f(y)
    if x.shape[0] != y.shape[0]:
        raise DimensionError("canonical_sines: ambient dimensions differ")
    out = np.empty(min(x.shape[1], y.shape[1]))
    _check(lib().orc_canonical_sines(x.shape[0], x.shape[1], _p(x), y.shape[1], _p(y), _p(out)))
    return out
