"""rsvd-b200: B200-native randomized SVD (Algorithms 2-6 of arXiv:2402.17794).

Python mirror of the reference's C++ API (namespace ``rsvd``,
/root/reference/proj/include/rsvd/{sketch,rangefinder,factor,singlepass,core}.hpp)
over the C ABI of ``lib/librsvd_b200.so`` (include/rsvd_b200.h).  Same names,
argument meaning and exception types as the reference:

    Rng(seed), gaussian(n, l, rng)                        sketch.hpp:19-59
    orthonormalize, svd_small, evd_symmetric, solve_ls    core.hpp:96-177
    singular_values, spectral_norm                        core.hpp:180-221
    computed_range_error                                  bounds.hpp:107-120
    canonical_sines, subspace_quality, AngleReport        angles.hpp:11-78
    reconstruction_error                                  drivers.hpp:145-151
    range_basis_trials, rsvd_trials, range_error_trials   drivers.hpp:340-356, 400-431
    fixed_rank_range, power_range, subspace_iter_range,
    range_basis, SketchConfig, RangeMode                  rangefinder.hpp:13-105
    rsvd, truncate, SvdApprox                             factor.hpp:12-34
    CountingOperator, spevd_hermitian, spsvd_general      singlepass.hpp:15-137

Matrices are column-major float64: either host numpy arrays or torch CUDA
tensors (device-resident, zero-copy; a column-major tensor is a transposed
contiguous tensor or any tensor with stride (1, ld)).  Results come back in the
same kind as the input.  There is no CPU fallback: if the CUDA library is
missing or no GPU is visible, calls raise ``EngineUnavailable``.
"""
from __future__ import annotations

import ctypes
import enum
import os
import threading
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = [
    "DimensionError", "ParameterError", "NumericError", "EngineError", "EngineUnavailable",
    "Rng", "RngState", "gaussian", "orthonormalize", "svd_small", "evd_symmetric", "solve_ls",
    "solve_joint_core", "RangeMode", "SketchConfig", "fixed_rank_range", "power_range",
    "subspace_iter_range", "range_basis", "SvdApprox", "EvdApprox", "rsvd", "truncate",
    "CountingOperator", "spevd_hermitian", "spsvd_general", "apply", "apply_adjoint", "Engine",
    "default_engine", "VirtualComm", "lib_path", "build", "using_engine", "rsvd_host", "singular_values",
    "spectral_norm", "computed_range_error", "canonical_sines", "subspace_quality", "AngleReport",
    "reconstruction_error", "range_basis_trials", "rsvd_trials", "range_error_trials",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# RSVD_B200_LIB: an alternative build of the same library (A/B experiments)
_LIB = os.environ.get("RSVD_B200_LIB") or os.path.join(_HERE, "lib", "librsvd_b200.so")


def lib_path() -> str:
    return _LIB


def build(quiet: bool = True) -> str:
    """Compile csrc/ for sm_100a into lib/librsvd_b200.so (nvcc, in-tree)."""
    import subprocess
    cmd = ["make", "-j8", "-C", os.path.join(_HERE, "csrc")]
    subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL if quiet else None)
    return _LIB


# ---------------------------------------------------------------- errors
class DimensionError(ValueError):
    """Bad shape (reference core.hpp:23-26, std::invalid_argument)."""


class ParameterError(ValueError):
    """Invalid parameter value (reference core.hpp:29-32, std::invalid_argument)."""


class NumericError(RuntimeError):
    """Numerical failure (reference core.hpp:35-39, std::runtime_error)."""


class EngineError(RuntimeError):
    """CUDA / NCCL / internal failure of the engine."""


class EngineUnavailable(RuntimeError):
    """The CUDA library or a GPU is missing (no CPU fallback exists)."""


_STATUS = {1: DimensionError, 2: ParameterError, 3: NumericError, 4: EngineError, 5: EngineError,
           9: EngineError}


class RngState(ctypes.Structure):
    """rsvd_rng_state: mt19937_64 vector + index + cached polar variate."""
    _fields_ = [("mt", ctypes.c_uint64 * 312), ("pos", ctypes.c_uint64),
                ("has_cached", ctypes.c_int32), ("pad_", ctypes.c_int32),
                ("cached", ctypes.c_double)]


class Counters(ctypes.Structure):
    _fields_ = [("apply", ctypes.c_int64), ("adjoint", ctypes.c_int64),
                ("physical_passes", ctypes.c_int64), ("kernel_launches", ctypes.c_int64),
                ("robust_reruns", ctypes.c_int64)]


_lib = None
_lib_lock = threading.Lock()


def _load():
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(_LIB):
            raise EngineUnavailable(f"{_LIB} not built (run __graft_entry__.build())")
        L = ctypes.CDLL(_LIB)
        P, I64, I, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        PS = ctypes.POINTER(RngState)
        sigs = {
            "rsvd_create": [ctypes.POINTER(P), I],
            "rsvd_nccl_unique_id": [P],
            "rsvd_create_dist": [ctypes.POINTER(P), I, I, I, P],
            "rsvd_vcomm_create": [ctypes.POINTER(P), I],
            "rsvd_create_virtual": [ctypes.POINTER(P), I, I, P],
            "rsvd_set_shard": [P, I64, I64],
            "rsvd_set_stream": [P, P],
            "rsvd_synchronize": [P],
            "rsvd_get_counters": [P, ctypes.POINTER(Counters)],
            "rsvd_reset_counters": [P],
            "rsvd_dist_info": [P, ctypes.POINTER(I), ctypes.POINTER(I)],
            "rsvd_profile_enable": [P, I],
            "rsvd_trace_enable": [P, I],
            "rsvd_trace_report": [P, ctypes.c_char_p, I64],
            "rsvd_profile_read": [P, I, ctypes.POINTER(I64), ctypes.POINTER(D), ctypes.POINTER(D),
                                  ctypes.POINTER(D)],
            "rsvd_gaussian_dev": [P, I64, I64, PS, P, I64],
            "rsvd_orthonormalize_dev": [P, I64, I64, P, I64, P, I64],
            "rsvd_svd_small_dev": [P, I64, I64, P, I64, P, I64, P, P, I64],
            "rsvd_evd_symmetric_dev": [P, I64, P, I64, P, I64, P],
            "rsvd_solve_ls_dev": [P, I64, I64, P, I64, I64, P, I64, P, I64],
            "rsvd_solve_joint_core_dev": [P, I64, P, P, P, P, P],
            "rsvd_apply_dev": [P, I64, I64, P, I64, I64, P, I64, P, I64],
            "rsvd_apply_adjoint_dev": [P, I64, I64, P, I64, I64, P, I64, P, I64],
            "rsvd_range_basis_dev": [P, I64, I64, P, I64, I64, I64, I, I, PS, P, I64],
            "rsvd_rsvd_dev": [P, I64, I64, P, I64, I64, I64, I, I, PS, P, I64, P, P, I64],
            "rsvd_rsvd_host": [P, I64, I64, P, I64, I64, I64, I, I, PS, P, I64, P, P, I64],
            "rsvd_spevd_dev": [P, I64, P, I64, I64, I64, PS, I, P, I64, P],
            "rsvd_spevd_shard_dev": [P, I64, I64, P, I64, I64, I64, PS, I, P, I64, P],
            "rsvd_spevd_shard_host": [P, I64, I64, P, I64, I64, I64, PS, P, I64, P],
            "rsvd_spevd_host": [P, I64, P, I64, I64, I64, PS, P, I64, P],
            "rsvd_spsvd_dev": [P, I64, I64, P, I64, I64, I64, PS, P, I64, P, P, I64],
            "rsvd_spsvd_host": [P, I64, I64, P, I64, I64, I64, PS, P, I64, P, P, I64],
            "rsvd_singular_values_dev": [P, I64, I64, P, I64, P],
            "rsvd_spectral_norm_dev": [P, I64, I64, P, I64, ctypes.POINTER(D)],
            "rsvd_computed_range_error_dev": [P, I64, I64, P, I64, I64, P, I64, ctypes.POINTER(D)],
            "rsvd_canonical_sines_dev": [P, I64, I64, P, I64, I64, P, I64, P],
            "rsvd_singular_values_host": [P, I64, I64, P, I64, P],
            "rsvd_spectral_norm_host": [P, I64, I64, P, I64, ctypes.POINTER(D)],
            "rsvd_computed_range_error_host": [P, I64, I64, P, I64, I64, P, I64, ctypes.POINTER(D)],
            "rsvd_canonical_sines_host": [P, I64, I64, P, I64, I64, P, I64, P],
            "rsvd_reconstruction_error_dev": [P, I64, I64, P, I64, I64, P, I64, P, P, I64,
                                              ctypes.POINTER(D), ctypes.POINTER(D)],
            "rsvd_range_basis_trials_dev": [P, I64, I64, P, I64, I64, I64, I, I, ctypes.c_uint64,
                                            I64, P, I64],
            "rsvd_rsvd_trials_dev": [P, I64, I64, P, I64, I64, I64, I, I, ctypes.c_uint64, I64, P,
                                     I64, P, P, I64],
            "rsvd_range_error_trials_dev": [P, I64, I64, P, I64, I64, I64, I, I, ctypes.c_uint64,
                                            I64, P],
        }
        for name, argt in sigs.items():
            f = getattr(L, name)
            f.argtypes = argt
            f.restype = ctypes.c_int
        L.rsvd_destroy.argtypes = [P]
        L.rsvd_destroy.restype = None
        L.rsvd_vcomm_destroy.argtypes = [P]
        L.rsvd_vcomm_destroy.restype = None
        L.rsvd_last_error.restype = ctypes.c_char_p
        L.rsvd_version.restype = ctypes.c_char_p
        L.rsvd_debug_log_cr.argtypes = [D]
        L.rsvd_debug_log_cr.restype = D
        L.rsvd_debug_dual_pass_dev.argtypes = [P, I64, I64, I64, P, I64, P, I64, P, I64, P, I64, P, I64, I64, I]
        L.rsvd_debug_dual_pass_dev.restype = ctypes.c_int
        L.rsvd_set_ozaki_slices.argtypes = [P, I]
        L.rsvd_set_ozaki_slices.restype = ctypes.c_int
        L.rsvd_debug_ozaki_kernel.argtypes = [I]
        L.rsvd_debug_ozaki_kernel.restype = ctypes.c_int
        L.rsvd_debug_ozaki_gemm_dev.argtypes = [P, I, I64, I64, P, I64, I64, P, I64, P, I64, I]
        L.rsvd_debug_ozaki_gemm_dev.restype = ctypes.c_int
        L.rsvd_debug_log_window.argtypes = [ctypes.c_void_p, I64, ctypes.c_void_p, ctypes.c_void_p]
        L.rsvd_debug_log_window.restype = None
        _lib = L
        return _lib


def _check(rc: int) -> None:
    if rc != 0:
        msg = _load().rsvd_last_error().decode(errors="replace")
        raise _STATUS.get(rc, EngineError)(msg)


# ---------------------------------------------------------------- engine
class VirtualComm:
    """nranks ranks of the row-sharded engine in this process on one device
    (rsvd_vcomm_create): one Engine per rank, each driven by its own thread;
    fixed-order device reductions stand in for NCCL.  For tests of the
    multi-GPU code path without several GPUs."""

    def __init__(self, nranks: int, device: int = 0):
        self.nranks = nranks
        self.ptr = ctypes.c_void_p()
        _check(_load().rsvd_vcomm_create(ctypes.byref(self.ptr), nranks))
        self.engines = [Engine(device, r, nranks, vcomm=self) for r in range(nranks)]

    def run(self, fn):
        """fn(rank, engine) on one thread per rank (the module-level API
        routed through that rank's engine); returns the per-rank results."""
        import threading
        out = [None] * self.nranks
        err = [None] * self.nranks

        def body(r):
            try:
                with using_engine(self.engines[r]):
                    out[r] = fn(r, self.engines[r])
            except BaseException as ex:  # noqa: BLE001
                err[r] = ex
        th = [threading.Thread(target=body, args=(r,)) for r in range(self.nranks)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        # the root cause first: a failing rank releases its peers with
        # "a peer rank failed"
        errs = [e for e in err if e is not None]
        errs.sort(key=lambda e: "peer rank failed" in str(e))
        if errs:
            raise errs[0]
        return out

    def close(self):
        for e in self.engines:
            e.close()
        self.engines = []
        if self.ptr.value:
            _load().rsvd_vcomm_destroy(self.ptr)
            self.ptr = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Engine:
    """Owns one rsvd_handle (one GPU; a row shard when created distributed)."""

    def __init__(self, device: int = 0, rank: int = 0, nranks: int = 1,
                 nccl_id: Optional[bytes] = None, vcomm: Optional["VirtualComm"] = None):
        L = _load()
        self._h = ctypes.c_void_p()
        self.device = device
        self.virtual = vcomm is not None
        self._vcomm = vcomm  # keeps the communicator alive
        # nranks == 1 with an id: a one-rank NCCL communicator, i.e. the
        # row-sharded code path (every exchange included) on one GPU
        if vcomm is not None:
            _check(L.rsvd_create_virtual(ctypes.byref(self._h), device, rank, vcomm.ptr))
            nranks = vcomm.nranks
        elif nranks > 1 or nccl_id is not None:
            buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            _check(L.rsvd_create_dist(ctypes.byref(self._h), device, rank, nranks, buf))
        else:
            _check(L.rsvd_create(ctypes.byref(self._h), device))
        self.rank, self.nranks = rank, nranks

    def set_shard(self, m_global: int, row_offset: int) -> None:
        """Shard descriptor: global rows and this rank's first row (no per-call
        row-count exchange)."""
        _check(_load().rsvd_set_shard(self._h, int(m_global), int(row_offset)))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(_load().rsvd_nccl_unique_id(buf))
        return buf.raw

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _load().rsvd_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int) -> None:
        _check(_load().rsvd_set_stream(self._h, ctypes.c_void_p(stream_ptr)))

    def counters(self) -> dict:
        c = Counters()
        _check(_load().rsvd_get_counters(self._h, ctypes.byref(c)))
        return {"apply": c.apply, "adjoint": c.adjoint, "physical_passes": c.physical_passes,
                "kernel_launches": c.kernel_launches, "robust_reruns": c.robust_reruns}

    def reset_counters(self) -> None:
        _check(_load().rsvd_reset_counters(self._h))

    def profile(self, on: bool = True) -> None:
        """Time every streaming-pass launch with CUDA events (resets totals)."""
        _check(_load().rsvd_profile_enable(self._h, 1 if on else 0))

    def profile_read(self) -> dict:
        out = {}
        for kind, name in ((0, "apply"), (1, "adjoint"), (2, "other"), (3, "fused"), (4, "int8")):
            n, ms, fl, by = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
            _check(_load().rsvd_profile_read(self._h, kind, ctypes.byref(n), ctypes.byref(ms),
                                             ctypes.byref(fl), ctypes.byref(by)))
            out[name] = {"launches": n.value, "ms": ms.value, "flops": fl.value, "bytes": by.value}
        return out

    def trace(self, on: bool = True) -> None:
        """Charge device time between consecutive launches to launch sites."""
        _check(_load().rsvd_trace_enable(self._h, 1 if on else 0))

    def trace_report(self) -> list:
        buf = ctypes.create_string_buffer(1 << 16)
        _check(_load().rsvd_trace_report(self._h, buf, len(buf)))
        rows = []
        for line in buf.value.decode().splitlines():
            site, cnt, ms = line.rsplit(" ", 2)
            rows.append((site, int(cnt), float(ms)))
        return sorted(rows, key=lambda r: -r[2])

    def synchronize(self) -> None:
        _check(_load().rsvd_synchronize(self._h))


_engines: dict = {}
_eng_lock = threading.Lock()


def default_engine(device: Optional[int] = None) -> Engine:
    import torch
    if not torch.cuda.is_available():
        raise EngineUnavailable("no CUDA device visible; the rsvd engine has no CPU fallback")
    if device is None:
        device = torch.cuda.current_device()
    with _eng_lock:
        e = _engines.get(device)
        if e is None:
            e = Engine(device)
            _engines[device] = e
        return e


# ------------------------------------------------------------------- RNG
_MT_F = 6364136223846793005
_M64 = (1 << 64) - 1


class Rng:
    """The reference's rsvd::Rng (sketch.hpp:19-45): std::mt19937_64(seed)
    feeding std::normal_distribution<double>, as an explicit state that the
    device generator advances exactly like the host library would."""

    _seeded: dict = {}  # seed -> freshly seeded state (the 312-step seeding
                        # recurrence costs ~100 us in Python; a copy ~1 us)

    def __init__(self, seed: int):
        seed &= _M64
        base = Rng._seeded.get(seed)
        if base is None:
            st = RngState()
            x = seed
            st.mt[0] = x
            for i in range(1, 312):
                x = (_MT_F * (x ^ (x >> 62)) + i) & _M64
                st.mt[i] = x
            st.pos = 312
            st.has_cached = 0
            st.cached = 0.0
            if len(Rng._seeded) >= 4096:
                Rng._seeded.clear()
            base = Rng._seeded[seed] = bytes(st)
        self.state = RngState.from_buffer_copy(base)

    @staticmethod
    def identity() -> str:
        return "mt19937_64/std-normal/v1"

    @staticmethod
    def for_trial(seed_base: int, trial: int) -> "Rng":
        return Rng((seed_base + trial) & _M64)

    def normal(self) -> float:
        return float(gaussian(1, 1, self)[0, 0])

    def copy(self) -> "Rng":
        r = Rng.__new__(Rng)
        r.state = RngState.from_buffer_copy(self.state)
        return r


# ---------------------------------------------------------- array plumbing
def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


class _Dev:
    """A device view (ptr, rows, cols, ld) of a numpy or torch input."""

    def __init__(self, x, name="matrix"):
        import torch
        self.host = not _is_torch(x)
        if self.host:
            a = np.asarray(x, dtype=np.float64)
            if a.ndim == 1:
                a = a.reshape(-1, 1)
            if a.ndim != 2:
                raise DimensionError(f"{name}: expected a matrix")
            self.rows, self.cols = a.shape
            t = torch.from_numpy(np.ascontiguousarray(a.T)).cuda()  # (cols, rows) row-major == col-major
            self.t = t
            self.ld = max(self.rows, 1)
        else:
            t = x
            if t.dtype != torch.float64:
                raise ParameterError(f"{name}: expected float64")
            if t.ndim == 1:
                t = t.reshape(-1, 1)
            if not t.is_cuda:
                return self.__init__(t.cpu().numpy(), name)
            self.rows, self.cols = t.shape
            if self.rows * self.cols > 0 and (t.stride(0) != 1 or t.stride(1) < max(self.rows, 1)):
                t = t.t().contiguous().t()  # make column-major
            self.t = t
            self.ld = t.stride(1) if self.cols > 1 else max(self.rows, 1)
            if self.cols == 1:
                self.ld = max(self.rows, 1)
        self.ptr = self.t.data_ptr()


def _empty(rows, cols, like_host, device=None):
    import torch
    t = torch.empty((max(cols, 0), max(rows, 0)), dtype=torch.float64,
                    device=device if device is not None else "cuda").t()
    return t


def _out(t, host: bool):
    if host:
        return np.asfortranarray(t.cpu().numpy())
    return t


def _vec_out(t, host: bool):
    return t.cpu().numpy() if host else t


_engine_override = threading.local()


class using_engine:
    """Context manager routing the module-level API through a given Engine
    (e.g. a row-sharded multi-GPU engine)."""

    def __init__(self, engine: Engine):
        self.engine = engine

    def __enter__(self):
        self.prev = getattr(_engine_override, "e", None)
        _engine_override.e = self.engine
        return self.engine

    def __exit__(self, *exc):
        _engine_override.e = self.prev


def _eng(x=None) -> Engine:
    import torch
    ov = getattr(_engine_override, "e", None)
    if ov is not None:
        ov.set_stream(torch.cuda.current_stream().cuda_stream)
        return ov
    dev = None
    if x is not None and _is_torch(x) and x.is_cuda:
        dev = x.device.index
    e = default_engine(dev)
    if dev is not None:
        torch.cuda.set_device(dev)
    e.set_stream(torch.cuda.current_stream().cuda_stream)
    return e


def _sync_torch():
    import torch
    torch.cuda.current_stream().synchronize()


# ------------------------------------------------------------ sketch.hpp
def gaussian(n: int, l: int, rng: Rng, *, device_out: bool = False):
    """n x l i.i.d. N(0,1), column-major fill (reference sketch.hpp:48-59)."""
    if n < 1 or l < 1:
        raise ParameterError("gaussian: dimensions must be positive")
    e = _eng()
    out = _empty(n, l, True)
    _check(_load().rsvd_gaussian_dev(e.handle, n, l, ctypes.byref(rng.state), out.data_ptr(),
                                     max(n, 1)))
    return out if device_out else np.asfortranarray(out.cpu().numpy())


# -------------------------------------------------------------- core.hpp
def orthonormalize(m):
    """Householder-quality orthonormal basis, padded to full width
    (reference core.hpp:96-105)."""
    d = _Dev(m, "orthonormalize")
    if d.cols > d.rows:
        raise DimensionError(f"orthonormalize: more columns than rows ({d.cols} > {d.rows})")
    e = _eng(None if d.host else m)
    q = _empty(d.rows, d.cols, d.host)
    if d.rows * d.cols:
        _check(_load().rsvd_orthonormalize_dev(e.handle, d.rows, d.cols, d.ptr, d.ld,
                                               q.data_ptr(), max(d.rows, 1)))
    return _out(q, d.host)


@dataclass
class SvdApprox:
    """U * diag(sigma) * V^T (reference core.hpp:43-53)."""
    U: object
    sigma: object
    V: object

    def factor_count(self) -> int:
        return int(self.sigma.shape[0])

    def reconstruct(self):
        if _is_torch(self.U):
            return (self.U * self.sigma) @ self.V.T
        return (self.U * self.sigma) @ self.V.T


@dataclass
class EvdApprox:
    """U * diag(lambda) * U^T (reference core.hpp:57-66)."""
    U: object
    lam: object

    @property
    def lambda_(self):
        return self.lam

    def factor_count(self) -> int:
        return int(self.lam.shape[0])

    def reconstruct(self):
        return (self.U * self.lam) @ self.U.T


def svd_small(m) -> SvdApprox:
    """Thin SVD with the reference sign rule (core.hpp:111-124)."""
    d = _Dev(m, "svd_small")
    e = _eng(None if d.host else m)
    r = min(d.rows, d.cols)
    import torch
    u, v = _empty(d.rows, r, d.host), _empty(d.cols, r, d.host)
    s = torch.empty(max(r, 1), dtype=torch.float64, device="cuda")
    if r:
        _check(_load().rsvd_svd_small_dev(e.handle, d.rows, d.cols, d.ptr, d.ld, u.data_ptr(),
                                          max(d.rows, 1), s.data_ptr(), v.data_ptr(),
                                          max(d.cols, 1)))
    return SvdApprox(_out(u, d.host), _vec_out(s[:r], d.host), _out(v, d.host))


def evd_symmetric(c) -> EvdApprox:
    """Symmetric EVD ordered by |lambda| desc (core.hpp:130-162)."""
    d = _Dev(c, "evd_symmetric")
    if d.rows != d.cols:
        raise DimensionError("evd_symmetric: matrix is not square")
    e = _eng(None if d.host else c)
    import torch
    u = _empty(d.rows, d.rows, d.host)
    lam = torch.empty(max(d.rows, 1), dtype=torch.float64, device="cuda")
    if d.rows:
        _check(_load().rsvd_evd_symmetric_dev(e.handle, d.rows, d.ptr, d.ld, u.data_ptr(),
                                              max(d.rows, 1), lam.data_ptr()))
    return EvdApprox(_out(u, d.host), _vec_out(lam[:d.rows], d.host))


def solve_ls(g, h):
    """Min-norm least squares, cutoff 1e-12 * sigma_max (core.hpp:166-177)."""
    dg, dh = _Dev(g, "solve_ls"), _Dev(h, "solve_ls")
    if dg.rows != dh.rows:
        raise DimensionError(f"solve_ls: row counts differ ({dg.rows} vs {dh.rows})")
    e = _eng(None if dg.host else g)
    x = _empty(dg.cols, dh.cols, dg.host)
    if dg.cols and dh.cols:
        _check(_load().rsvd_solve_ls_dev(e.handle, dg.rows, dg.cols, dg.ptr, dg.ld, dh.cols,
                                         dh.ptr, dh.ld, x.data_ptr(), max(dg.cols, 1)))
    return _out(x, dg.host)


def solve_joint_core(g1, h1, g2, h2):
    """detail::solve_joint_core (singlepass.hpp:84-101), Kronecker route."""
    ds = [_Dev(x, "solve_joint_core") for x in (g1, h1, g2, h2)]
    l = ds[0].rows
    for d in ds:
        if d.rows != l or d.cols != l:
            raise DimensionError("solve_joint_core: blocks must be l x l")
    # the C ABI takes packed l x l blocks
    import torch
    packed = [d.t if d.ld == l else d.t.t().contiguous().t() for d in ds]
    e = _eng(None if ds[0].host else g1)
    c = _empty(l, l, ds[0].host)
    _check(_load().rsvd_solve_joint_core_dev(e.handle, l, *[p.data_ptr() for p in packed],
                                             c.data_ptr()))
    return _out(c, ds[0].host)


# ------------------------------------------------------- rangefinder.hpp
class RangeMode(enum.IntEnum):
    basic = 0
    power = 1
    power_ortho = 2


def to_string(mode: RangeMode) -> str:
    return {RangeMode.basic: "basic", RangeMode.power: "power", RangeMode.power_ortho: "ortho"}[mode]


@dataclass
class SketchConfig:
    """Every Stage-1 tunable (rangefinder.hpp:30-42)."""
    k: int = 1
    p: int = 0
    q: int = 0
    mode: RangeMode = RangeMode.basic
    seed: int = 0

    def normalized(self) -> "SketchConfig":
        c = SketchConfig(self.k, self.p, self.q, self.mode, self.seed)
        if c.mode == RangeMode.basic:
            c.q = 0
        return c


def range_basis(a, cfg: SketchConfig, rng: Rng):
    """Dispatch on the Stage-1 variant (rangefinder.hpp:97-105)."""
    c = cfg.normalized()
    d = _Dev(a, "range_basis")
    e = _eng(None if d.host else a)
    l = c.k + c.p
    q = _empty(d.rows, max(l, 0), d.host)
    _check(_load().rsvd_range_basis_dev(e.handle, d.rows, d.cols, d.ptr, d.ld, c.k, c.p, c.q,
                                        int(c.mode), ctypes.byref(rng.state), q.data_ptr(),
                                        max(d.rows, 1)))
    return _out(q, d.host)


def fixed_rank_range(a, k: int, p: int, rng: Rng):
    """Alg 2 Stage 1 (rangefinder.hpp:60-65)."""
    return range_basis(a, SketchConfig(k, p, 0, RangeMode.basic), rng)


def power_range(a, k: int, p: int, q: int, rng: Rng):
    """Alg 3 Stage 1 (rangefinder.hpp:70-79)."""
    return range_basis(a, SketchConfig(k, p, q, RangeMode.power), rng)


def subspace_iter_range(a, k: int, p: int, q: int, rng: Rng):
    """Alg 4 Stage 1 (rangefinder.hpp:83-94)."""
    return range_basis(a, SketchConfig(k, p, q, RangeMode.power_ortho), rng)


# ------------------------------------------------------------ factor.hpp
def rsvd(a, cfg: SketchConfig, rng: Optional[Rng] = None) -> SvdApprox:
    """Two-stage randomized SVD, full width k+p (factor.hpp:12-24)."""
    if rng is None:
        rng = Rng(cfg.seed)
    d = _Dev(a, "rsvd")
    e = _eng(None if d.host else a)
    import torch
    l = max(cfg.k + cfg.p, 0)
    u, v = _empty(d.rows, l, d.host), _empty(d.cols, l, d.host)
    s = torch.empty(max(l, 1), dtype=torch.float64, device="cuda")
    _check(_load().rsvd_rsvd_dev(e.handle, d.rows, d.cols, d.ptr, d.ld, cfg.k, cfg.p, cfg.q,
                                 int(cfg.mode), ctypes.byref(rng.state), u.data_ptr(),
                                 max(d.rows, 1), s.data_ptr(), v.data_ptr(), max(d.cols, 1)))
    return SvdApprox(_out(u, d.host), _vec_out(s[:l], d.host), _out(v, d.host))


def truncate(f: SvdApprox, k: int) -> SvdApprox:
    """Keep the first k factor triples (factor.hpp:27-34)."""
    if k < 0 or k > f.factor_count():
        raise DimensionError(f"truncate: k = {k} exceeds factor count {f.factor_count()}")
    return SvdApprox(f.U[:, :k], f.sigma[:k], f.V[:, :k])


# -------------------------------------------------------- singlepass.hpp
class CountingOperator:
    """Operator view counting block applications (singlepass.hpp:15-40).  The
    engine counts the passes it makes over A; this wrapper exposes them."""

    def __init__(self, a):
        self._a = a
        self.apply_count_ = 0
        self.adjoint_count_ = 0
        self.physical_passes_ = 0

    def matrix(self):
        return self._a

    def rows(self) -> int:
        return int(self._a.shape[0])

    def cols(self) -> int:
        return int(self._a.shape[1])

    def apply_count(self) -> int:
        return self.apply_count_

    def adjoint_count(self) -> int:
        return self.adjoint_count_

    def physical_passes(self) -> int:
        """Streaming traversals of A (engine extension): Alg 6's fused pass
        counts one apply, one adjoint and ONE physical pass."""
        return self.physical_passes_

    def apply(self, x):
        self.apply_count_ += 1
        return apply(self._a, x)

    def apply_adjoint(self, x):
        self.adjoint_count_ += 1
        return apply_adjoint(self._a, x)


def _counted(a, fn):
    op = a if isinstance(a, CountingOperator) else None
    mat = op.matrix() if op else a
    d = _Dev(mat, "operator")
    e = _eng(None if d.host else mat)
    before = e.counters()
    res = fn(d, e)
    after = e.counters()
    if op is not None:
        op.apply_count_ += after["apply"] - before["apply"]
        op.adjoint_count_ += after["adjoint"] - before["adjoint"]
        op.physical_passes_ += after["physical_passes"] - before["physical_passes"]
    return res


def spevd_hermitian(a, k: int, p: int, rng: Rng) -> EvdApprox:
    """Single-pass symmetric EVD, Alg 5 (singlepass.hpp:45-78)."""
    def run(d, e):
        import torch
        # a distributed engine takes this rank's (m_local x n) row shard;
        # squareness is then m_global == n (checked by the engine)
        if d.rows != d.cols and e.nranks == 1 and not e.virtual:
            raise DimensionError("spevd_hermitian: matrix is not square")
        u = _empty(d.rows, max(k, 0), d.host)
        lam = torch.empty(max(k, 1), dtype=torch.float64, device="cuda")
        _check(_load().rsvd_spevd_shard_dev(e.handle, d.rows, d.cols, d.ptr, d.ld, k, p,
                                            ctypes.byref(rng.state), 1, u.data_ptr(), max(d.rows, 1),
                                            lam.data_ptr()))
        return EvdApprox(_out(u, d.host), _vec_out(lam[:max(k, 0)], d.host))
    return _counted(a, run)


def spsvd_general(a, k: int, p: int, rng: Rng) -> SvdApprox:
    """Single-pass general SVD, Alg 6 (singlepass.hpp:109-137)."""
    def run(d, e):
        import torch
        kk = max(k, 0)
        u, v = _empty(d.rows, kk, d.host), _empty(d.cols, kk, d.host)
        s = torch.empty(max(kk, 1), dtype=torch.float64, device="cuda")
        _check(_load().rsvd_spsvd_dev(e.handle, d.rows, d.cols, d.ptr, d.ld, k, p,
                                      ctypes.byref(rng.state), u.data_ptr(), max(d.rows, 1),
                                      s.data_ptr(), v.data_ptr(), max(d.cols, 1)))
        return SvdApprox(_out(u, d.host), _vec_out(s[:kk], d.host), _out(v, d.host))
    return _counted(a, run)


# ------------------------------------------------------ streaming passes
def apply(a, x):
    """Y = A X on the DMMA pass engine."""
    da, dx = _Dev(a, "apply"), _Dev(x, "apply")
    if da.cols != dx.rows:
        raise DimensionError("apply: inner dimensions differ")
    e = _eng(None if da.host else a)
    y = _empty(da.rows, dx.cols, da.host)
    _check(_load().rsvd_apply_dev(e.handle, da.rows, da.cols, da.ptr, da.ld, dx.cols, dx.ptr,
                                  dx.ld, y.data_ptr(), max(da.rows, 1)))
    return _out(y, da.host)


def apply_adjoint(a, y):
    """Z = A^T Y on the DMMA pass engine."""
    da, dy = _Dev(a, "apply_adjoint"), _Dev(y, "apply_adjoint")
    if da.rows != dy.rows:
        raise DimensionError("apply_adjoint: inner dimensions differ")
    e = _eng(None if da.host else a)
    z = _empty(da.cols, dy.cols, da.host)
    _check(_load().rsvd_apply_adjoint_dev(e.handle, da.rows, da.cols, da.ptr, da.ld, dy.cols,
                                          dy.ptr, dy.ld, z.data_ptr(), max(da.cols, 1)))
    return _out(z, da.host)


def rsvd_host(a: np.ndarray, cfg: SketchConfig, rng: Optional[Rng] = None, out=None):
    """End-to-end host-buffer call (rsvd_rsvd_host): A and the outputs live in
    host memory; the host<->device copies are part of the call.  `a` must be a
    Fortran-ordered float64 array (pinned memory makes the copy fast); `out`
    optionally supplies preallocated (U, sigma, V) host arrays."""
    if rng is None:
        rng = Rng(cfg.seed)
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.f_contiguous):
        a = np.asfortranarray(a, dtype=np.float64)
    m, n = a.shape
    l = max(cfg.k + cfg.p, 0)
    if out is None:
        out = (np.empty((m, l), order="F"), np.empty(l), np.empty((n, l), order="F"))
    u, s, v = out
    e = _eng()
    P = lambda x: x.ctypes.data_as(ctypes.c_void_p)
    _check(_load().rsvd_rsvd_host(e.handle, m, n, P(a), max(m, 1), cfg.k, cfg.p, cfg.q,
                                  int(cfg.mode), ctypes.byref(rng.state), P(u), max(m, 1), P(s),
                                  P(v), max(n, 1)))
    return SvdApprox(u, s, v)


def spevd_host(a: np.ndarray, k: int, p: int, rng: Rng, out=None):
    """End-to-end host-buffer spevd_hermitian (rsvd_spevd_host): A streamed up
    in row panels into the pass; `out` optionally supplies preallocated
    (U, lambda) host arrays (pinned memory makes the copy-back fast)."""
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.f_contiguous):
        a = np.asfortranarray(a, dtype=np.float64)
    m_local, n = a.shape  # a row shard (m_local x n) on a distributed engine
    kk = max(k, 0)
    u, lam = out if out is not None else (np.empty((m_local, kk), order="F"), np.empty(max(kk, 1)))
    e = _eng()
    if m_local != n and e.nranks == 1 and not e.virtual:
        raise DimensionError("spevd_hermitian: matrix is not square")
    P = lambda x: x.ctypes.data_as(ctypes.c_void_p)
    _check(_load().rsvd_spevd_shard_host(e.handle, m_local, n, P(a), max(m_local, 1), k, p,
                                         ctypes.byref(rng.state), P(u), max(m_local, 1), P(lam)))
    return EvdApprox(u, lam[:kk])


def spsvd_host(a: np.ndarray, k: int, p: int, rng: Rng, out=None):
    """End-to-end host-buffer spsvd_general (rsvd_spsvd_host): A streamed up
    in row panels into the fused pass; `out` optionally supplies preallocated
    (U, sigma, V) host arrays (pinned memory makes the copy-back fast)."""
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.f_contiguous):
        a = np.asfortranarray(a, dtype=np.float64)
    m, n = a.shape
    kk = max(k, 0)
    u, s, v = out if out is not None else (np.empty((m, kk), order="F"), np.empty(max(kk, 1)),
                                           np.empty((n, kk), order="F"))
    e = _eng()
    P = lambda x: x.ctypes.data_as(ctypes.c_void_p)
    _check(_load().rsvd_spsvd_host(e.handle, m, n, P(a), max(m, 1), k, p, ctypes.byref(rng.state),
                                   P(u), max(m, 1), P(s), P(v), max(n, 1)))
    return SvdApprox(u, s[:kk], v)


def debug_log_cr(x: float) -> float:
    """Host evaluation of the device polar-sampler log (ddlog.cuh), for tests."""
    return _load().rsvd_debug_log_cr(float(x))


def debug_dual_pass(a, oc, psi, panel_rows: int = 0, macroblock: int = 0):
    """The fused Alg-6 pass alone (fused.cu): returns (A @ oc, A.T @ psi) from
    one traversal of A.  panel_rows > 0 issues A in row panels of that many
    rows (the streamed host path's launch sequence); macroblock > 0 overrides
    the macroblock edge.  Device tensors in, device tensors out."""
    import torch
    e = default_engine()
    m, n = a.shape
    l = oc.shape[1]
    y = torch.empty((l, m), dtype=torch.float64, device="cuda").t()
    w = torch.empty((l, n), dtype=torch.float64, device="cuda").t()
    ld = lambda t: int(t.stride(1)) if t.shape[1] > 1 else max(int(t.shape[0]), 1)  # noqa: E731
    _check(_load().rsvd_debug_dual_pass_dev(e.handle, m, n, l, a.data_ptr(), ld(a), oc.data_ptr(), ld(oc),
                                             psi.data_ptr(), ld(psi), y.data_ptr(), m, w.data_ptr(), n,
                                             int(panel_rows), int(macroblock)))
    return y, w


def set_ozaki_slices(slices: int, engine=None) -> None:
    """Run the wide-sketch products with A on the INT8 tensor cores with
    `slices` exact 8-bit slices per operand (csrc/ozaki.cu): 0 = off (FP64
    DMMA passes), 3..8 = slices (7 = fp64-equivalent, the automatic choice),
    -1 = the automatic policy / the RSVD_OZAKI environment variable."""
    e = engine or default_engine()
    _check(_load().rsvd_set_ozaki_slices(e.handle, int(slices)))


def debug_ozaki_kernel(pair: int) -> None:
    """Select the INT8 GEMM kernel process-wide: 1 = CTA pair (cta_group::2,
    default), 0 = single CTA, -1 = default.  For unit tests."""
    _check(_load().rsvd_debug_ozaki_kernel(int(pair)))


def debug_ozaki_gemm(a, x, trans: bool = False, slices: int = 8):
    """A @ x (or A.T @ x) by the sliced INT8 tensor-core product alone.
    Column-major device tensors in, device tensor out."""
    import torch
    e = default_engine()
    m, n = a.shape
    l = x.shape[1]
    rows = n if trans else m
    c = torch.empty((l, rows), dtype=torch.float64, device="cuda").t()
    ld = lambda t: int(t.stride(1)) if t.shape[1] > 1 else max(int(t.shape[0]), 1)  # noqa: E731
    _check(_load().rsvd_debug_ozaki_gemm_dev(e.handle, int(bool(trans)), m, n, a.data_ptr(), ld(a), l,
                                              x.data_ptr(), ld(x), c.data_ptr(), rows, int(slices)))
    return c


def debug_log_window(x):
    """Host evaluation of the exact-mode flag test (ddlog.cuh log_near_midpoint):
    returns (correctly rounded log(x), flag) arrays; flag marks the inputs whose
    normals the engine recomputes with the host glibc log."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    cr = np.empty_like(x)
    fl = np.empty(x.shape, dtype=np.uint8)
    _load().rsvd_debug_log_window(x.ctypes.data, x.size, cr.ctypes.data, fl.ctypes.data)
    return cr, fl.astype(bool)


# ------------------------------------------------ diagnostics (core/bounds/angles)
def singular_values(m):
    """Singular values, descending (reference core.hpp:180-183)."""
    import torch
    d = _Dev(m, "singular_values")
    e = _eng(None if d.host else m)
    r = min(d.rows, d.cols)
    s = torch.empty(max(r, 1), dtype=torch.float64, device="cuda")
    if r:
        _check(_load().rsvd_singular_values_dev(e.handle, d.rows, d.cols, d.ptr, d.ld, s.data_ptr()))
    return _vec_out(s[:r], d.host)


def spectral_norm(m) -> float:
    """||M||_2: dense SVD when min(m, n) <= 512, else power iteration on M^T M
    from the reference's LCG start vector, tol 1e-10, cap 5000
    (reference core.hpp:188-221)."""
    d = _Dev(m, "spectral_norm")
    e = _eng(None if d.host else m)
    out = ctypes.c_double(0.0)
    _check(_load().rsvd_spectral_norm_dev(e.handle, d.rows, d.cols, d.ptr, d.ld, ctypes.byref(out)))
    return out.value


def computed_range_error(a, q) -> float:
    """Measured Stage-1 residual ||A - Q Q^T A||_2 (reference bounds.hpp:107-120)."""
    da, dq = _Dev(a, "computed_range_error"), _Dev(q, "computed_range_error")
    if dq.rows != da.rows:
        raise DimensionError("computed_range_error: row counts differ")
    e = _eng(None if da.host else a)
    out = ctypes.c_double(0.0)
    _check(_load().rsvd_computed_range_error_dev(e.handle, da.rows, da.cols, da.ptr, da.ld,
                                                 dq.cols, dq.ptr, dq.ld, ctypes.byref(out)))
    return out.value


def canonical_sines(x, y):
    """Sines of the principal angles between range(X) and range(Y), ascending,
    clamped to [0, 1] (reference angles.hpp:42-60, projection route)."""
    import torch
    dx, dy = _Dev(x, "canonical_sines"), _Dev(y, "canonical_sines")
    if dx.rows != dy.rows:
        raise DimensionError("canonical_sines: ambient dimensions differ")
    e = _eng(None if dx.host else x)
    cnt = min(dx.cols, dy.cols)
    out = torch.empty(max(cnt, 1), dtype=torch.float64, device="cuda")
    _check(_load().rsvd_canonical_sines_dev(e.handle, dx.rows, dx.cols, dx.ptr, dx.ld, dy.cols,
                                            dy.ptr, dy.ld, out.data_ptr()))
    return _vec_out(out[:cnt], dx.host)


@dataclass
class AngleReport:
    """Per-index canonical-angle record (reference angles.hpp:11-22)."""
    k: int = 0
    p: int = 0
    q: int = 0
    seed: int = 0
    gap: float = 0.0
    sin_theta: object = None
    sin_nu: object = None
    bound_theta: object = None
    bound_nu: object = None


def subspace_quality(oracle, k: int, result: SvdApprox) -> AngleReport:
    """Angles between the oracle's rank-k singular subspaces and the first k
    computed factors (reference angles.hpp:62-78).  `oracle` is an SvdApprox
    or the matrix itself (then svd_small(oracle) is the oracle)."""
    if k < 1:
        raise ParameterError("subspace_quality: k must be >= 1")
    if not isinstance(oracle, SvdApprox):
        oracle = svd_small(oracle)
    if oracle.factor_count() < k or result.factor_count() < k:
        raise DimensionError("subspace_quality: fewer than k factors available")
    rep = AngleReport(k=k)
    rep.sin_theta = canonical_sines(oracle.U[:, :k], result.U[:, :k])
    rep.sin_nu = canonical_sines(oracle.V[:, :k], result.V[:, :k])
    return rep


def reconstruction_error(a, f):
    """run_svd's error report (reference drivers.hpp:145-151) for an SvdApprox
    (or EvdApprox): (||A - recon||_F / ||A||_F, ||A - recon||_2 / ||A||_2)."""
    da = _Dev(a, "reconstruction_error")
    e = _eng(None if da.host else a)
    if isinstance(f, EvdApprox):
        du, dv, s = _Dev(f.U), _Dev(f.U), f.lambda_
    else:
        du, dv, s = _Dev(f.U), _Dev(f.V), f.sigma
    import torch
    sd = torch.as_tensor(np.asarray(s) if not _is_torch(s) else s, dtype=torch.float64).cuda().contiguous()
    fro, spec = ctypes.c_double(0.0), ctypes.c_double(0.0)
    _check(_load().rsvd_reconstruction_error_dev(e.handle, da.rows, da.cols, da.ptr, da.ld, du.cols,
                                                 du.ptr, du.ld, sd.data_ptr(), dv.ptr, dv.ld,
                                                 ctypes.byref(fro), ctypes.byref(spec)))
    return fro.value, spec.value


# ------------------------------------------------------------ batched trials
def _trial_args(cfg: SketchConfig, trials: int):
    if trials < 1:
        raise ParameterError("trials must be >= 1")
    return cfg.k, cfg.p, cfg.q, int(cfg.mode), ctypes.c_uint64(cfg.seed & (2**64 - 1)), int(trials)


def range_basis_trials(a, cfg: SketchConfig, trials: int):
    """Stage-1 bases of `trials` runs, trial t with Rng(cfg.seed + t) (the
    run_bounds loop, drivers.hpp:340-346): every pass over A shared by all
    trials.  Returns a list of m x (k+p) bases."""
    d = _Dev(a, "range_basis_trials")
    e = _eng(None if d.host else a)
    k, p, q, mode, seed, T = _trial_args(cfg, trials)
    l = max(k + p, 0)
    qall = _empty(d.rows, l * T, d.host)
    _check(_load().rsvd_range_basis_trials_dev(e.handle, d.rows, d.cols, d.ptr, d.ld, k, p, q, mode,
                                               seed, T, qall.data_ptr(), max(d.rows, 1)))
    qall = _out(qall, d.host)
    return [qall[:, t * l:(t + 1) * l] for t in range(T)]


def rsvd_trials(a, cfg: SketchConfig, trials: int):
    """rsvd(A, cfg, Rng(cfg.seed + t)) for t < trials (the run_angles loop,
    drivers.hpp:400-408) with the passes over A shared by all trials."""
    import torch
    d = _Dev(a, "rsvd_trials")
    e = _eng(None if d.host else a)
    k, p, q, mode, seed, T = _trial_args(cfg, trials)
    l = max(k + p, 0)
    u, v = _empty(d.rows, l * T, d.host), _empty(d.cols, l * T, d.host)
    s = torch.empty(max(l * T, 1), dtype=torch.float64, device="cuda")
    _check(_load().rsvd_rsvd_trials_dev(e.handle, d.rows, d.cols, d.ptr, d.ld, k, p, q, mode, seed, T,
                                        u.data_ptr(), max(d.rows, 1), s.data_ptr(), v.data_ptr(),
                                        max(d.cols, 1)))
    u, v, s = _out(u, d.host), _out(v, d.host), _vec_out(s[:l * T], d.host)
    return [SvdApprox(u[:, t * l:(t + 1) * l], s[t * l:(t + 1) * l], v[:, t * l:(t + 1) * l])
            for t in range(T)]


def range_error_trials(a, cfg: SketchConfig, trials: int) -> np.ndarray:
    """computed_range_error(A, range_basis(A, cfg, Rng(cfg.seed + t))) for
    t < trials (the run_bounds loop, drivers.hpp:340-346)."""
    d = _Dev(a, "range_error_trials")
    e = _eng(None if d.host else a)
    k, p, q, mode, seed, T = _trial_args(cfg, trials)
    out = np.zeros(T)
    _check(_load().rsvd_range_error_trials_dev(e.handle, d.rows, d.cols, d.ptr, d.ld, k, p, q, mode,
                                               seed, T, out.ctypes.data_as(ctypes.c_void_p)))
    return out
