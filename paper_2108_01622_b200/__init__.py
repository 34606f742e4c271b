"""paper_2108_01622_b200 -- B200 (sm_100a) loop hafnians with repeated rows/columns.

Thin ctypes binding over the C-ABI of ``include/lhaf.h`` (liblhaf.so, built in-tree by
``paper_2108_01622_b200.build``).  Argument marshalling only: every step of the method runs
in the library's CUDA kernels.  There is no CPU fallback: if liblhaf.so is missing, importing
the binding raises, and without a CUDA device every compute call raises ``LhafError``.

Names follow the C-ABI: ``lhaf_rpt``, ``lhaf_rpt_batch``, ``lhaf_rpt_mixed``,
``lhaf_rpt_batch_dev``, ``lhaf_rpt_cutoff``, ``lhaf_gbs_matrices``, ``lhaf_gbs_prob``,
``lhaf_ips_prob``,
``lhaf_plan``, ``lhaf_decode``, the ``Job`` wrapper over
``lhaf_job_*``, and the rank calls ``lhaf_get_unique_id`` / ``lhaf_init_rank``.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# LHAF_LIB_PATH selects a diagnostic build of the same library (tools/phase_timing.py)
LIB_PATH = os.environ.get("LHAF_LIB_PATH") or os.path.join(_HERE, "liblhaf.so")

LHAF_MAX_PAIRS = 64
LHAF_OK = 0
_STATUS = {0: "LHAF_OK", 1: "LHAF_E_ARG", 2: "LHAF_E_NOT_SYMMETRIC", 3: "LHAF_E_TOO_LARGE",
           4: "LHAF_E_CUDA", 5: "LHAF_E_NCCL", 6: "LHAF_E_STATE", 7: "LHAF_E_INACCURATE"}


class LhafError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class PlanInfo(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int32), ("H", ctypes.c_int32), ("d", ctypes.c_int32),
                ("n", ctypes.c_int32), ("leftover", ctypes.c_int32), ("pad_", ctypes.c_int32),
                ("T", ctypes.c_uint64), ("T_eval", ctypes.c_uint64),
                ("p", ctypes.c_int32 * LHAF_MAX_PAIRS), ("q", ctypes.c_int32 * LHAF_MAX_PAIRS),
                ("eta", ctypes.c_int32 * LHAF_MAX_PAIRS)]

    def pairs(self):
        return [(self.p[h], self.q[h]) for h in range(self.H)]

    def etas(self):
        return [self.eta[h] for h in range(self.H)]


class JobInfo(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("d_max", ctypes.c_int32), ("n_max", ctypes.c_int32),
                ("kernel", ctypes.c_int32), ("units", ctypes.c_uint64), ("terms", ctypes.c_uint64),
                ("flops_per_term_model", ctypes.c_double), ("h2d_plan_bytes", ctypes.c_uint64),
                ("precision", ctypes.c_int32), ("pad_", ctypes.c_int32)]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2108_01622_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    dp = ctypes.POINTER(ctypes.c_double)
    ip = ctypes.POINTER(ctypes.c_int32)
    vp = ctypes.c_void_p
    u64 = ctypes.c_uint64
    sig = {
        "lhaf_plan": ([ip, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(PlanInfo)]),
        "lhaf_decode": ([ctypes.POINTER(PlanInfo), u64, ip, ip, ip, ctypes.POINTER(u64)]),
        "lhaf_rpt": ([dp, dp, ip, ctypes.c_int32, dp]),
        "lhaf_rpt_batch": ([dp, dp, ctypes.c_int64, ip, ctypes.c_int32, ctypes.c_int32, dp]),
        "lhaf_rpt_mixed": ([dp, dp, ip, ctypes.c_int32, dp]),
        "lhaf_rpt_cutoff": ([dp, dp, ip, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, dp]),
        "lhaf_rpt_cutoff_ex": ([dp, dp, ip, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                ctypes.c_double, dp, dp]),
        "lhaf_gbs_matrices": ([dp, dp, ctypes.c_int32, dp, dp, dp]),
        "lhaf_gbs_prob": ([dp, dp, ctypes.c_int32, ip, ctypes.c_int32, dp]),
        "lhaf_gbs_state": ([dp, dp, vp, vp, ctypes.c_int32, dp, dp]),
        "lhaf_gbs_prob_state": ([dp, dp, vp, vp, ctypes.c_int32, ip, dp]),
        "lhaf_ips_prob": ([dp, dp, ctypes.c_int32, ip, dp]),
        "lhaf_rpt_et": ([dp, dp, ip, ctypes.c_int32, dp]),
        "lhaf_rpt_multigamma": ([dp, dp, ctypes.c_int32, ip, ctypes.c_int32, dp]),
        "lhaf_rpt_batch_dev": ([vp, vp, ctypes.c_int64, ip, ctypes.c_int32, ctypes.c_int32,
                                ctypes.c_int32, vp, vp]),
        "lhaf_job_create": ([vp, vp, ctypes.c_int64, ip, ctypes.c_int32, ctypes.c_int32,
                             ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(vp)]),
        "lhaf_job_info_get": ([vp, ctypes.POINTER(JobInfo)]),
        "lhaf_job_plan": ([vp, ctypes.c_int32, ctypes.POINTER(PlanInfo)]),
        "lhaf_job_reset": ([vp, vp]),
        "lhaf_job_run": ([vp, u64, u64, vp]),
        "lhaf_job_allreduce": ([vp, vp]),
        "lhaf_job_reset_range": ([vp, u64, u64, vp]),
        "lhaf_job_allreduce_range": ([vp, u64, u64, vp]),
        "lhaf_job_finalize": ([vp, vp, ctypes.c_int32, vp]),
        "lhaf_job_abs_sum": ([vp, dp]),
        "lhaf_job_partials": ([vp, ctypes.POINTER(vp), ctypes.POINTER(ctypes.c_size_t)]),
        "lhaf_job_terms": ([vp, ctypes.POINTER(u64), ctypes.c_int32, dp]),
        "lhaf_set_device": ([ctypes.c_int32]),
        "lhaf_get_unique_id": ([vp]),
        "lhaf_init_rank": ([ctypes.c_int32, ctypes.c_int32, vp, ctypes.c_int32]),
        "lhaf_rank_info": ([ip, ip]),
        "lhaf_set_kernel": ([ctypes.c_int32]),
        "lhaf_set_precision": ([ctypes.c_int32]),
        "lhaf_shard_units": ([u64, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(u64),
                              ctypes.POINTER(u64)]),
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    lib.lhaf_job_destroy.argtypes = [vp]
    lib.lhaf_job_destroy.restype = None
    lib.lhaf_last_error.restype = ctypes.c_char_p
    lib.lhaf_version.restype = ctypes.c_char_p
    lib.lhaf_launch_count.restype = ctypes.c_uint64
    lib.lhaf_shutdown.restype = None
    lib.lhaf_get_precision.restype = ctypes.c_int32
    return lib


class _Missing:
    """Stands in for liblhaf.so when it could not be loaded (e.g. while `build` itself is being
    imported to rebuild it): every use raises the load error -- there is no CPU fallback."""

    def __init__(self, err: Exception):
        self._err = err

    def __getattr__(self, name):
        raise ImportError(f"liblhaf.so unavailable: {self._err}")


try:
    _lib = _load()
except (OSError, AttributeError, ImportError) as _e:  # stale or missing .so
    _lib = _Missing(_e)


def reload_library():
    """Re-load liblhaf.so after a rebuild (used by build())."""
    global _lib
    _lib = _load()
    return _lib

# every symbol include/lhaf.h declares (checked by tests/test_host.py::test_library_exports_every_declared_symbol)
EXPORTED = ["lhaf_plan", "lhaf_decode", "lhaf_rpt", "lhaf_rpt_batch", "lhaf_rpt_mixed", "lhaf_rpt_cutoff",
            "lhaf_rpt_cutoff_ex",
            "lhaf_gbs_matrices", "lhaf_gbs_prob", "lhaf_gbs_state", "lhaf_gbs_prob_state",
            "lhaf_ips_prob", "lhaf_rpt_et",
            "lhaf_rpt_multigamma",
            "lhaf_rpt_batch_dev", "lhaf_job_create", "lhaf_job_info_get", "lhaf_job_reset",
            "lhaf_job_run", "lhaf_job_allreduce", "lhaf_job_reset_range", "lhaf_job_allreduce_range",
            "lhaf_job_finalize", "lhaf_job_abs_sum", "lhaf_job_plan",
            "lhaf_job_partials", "lhaf_job_terms", "lhaf_job_destroy", "lhaf_set_device",
            "lhaf_get_unique_id", "lhaf_init_rank", "lhaf_rank_info", "lhaf_set_kernel",
            "lhaf_set_precision", "lhaf_get_precision",
            "lhaf_shard_units", "lhaf_last_error", "lhaf_version", "lhaf_launch_count",
            "lhaf_shutdown"]


def _check(status: int):
    if status != LHAF_OK:
        raise LhafError(status, _lib.lhaf_last_error().decode())


def _c128(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.complex128))


def _i32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def version() -> str:
    return _lib.lhaf_version().decode()


def lhaf_launch_count() -> int:
    """Kernel launches the library has issued in this process (bench.py's gpu_launches)."""
    return int(_lib.lhaf_launch_count())


def lhaf_plan(reps, mixed: int = 0) -> PlanInfo:
    reps = _i32(reps)
    info = PlanInfo()
    _check(_lib.lhaf_plan(_ip(reps), reps.shape[0], int(mixed), ctypes.byref(info)))
    return info


def lhaf_decode(info: PlanInfo, t: int):
    """(k digits, w, sign, weight) of term t -- integer work, bit-exact."""
    k = np.zeros(max(1, info.H), np.int32)
    w = np.zeros(max(1, info.H), np.int32)
    sign = ctypes.c_int32()
    weight = ctypes.c_uint64()
    _check(_lib.lhaf_decode(ctypes.byref(info), int(t), _ip(k), _ip(w), ctypes.byref(sign),
                            ctypes.byref(weight)))
    return k[:info.H].tolist(), w[:info.H].tolist(), sign.value, weight.value


def lhaf_rpt(A, gamma, reps) -> complex:
    A, gamma, reps = _c128(A), _c128(gamma), _i32(reps)
    out = np.zeros(2)
    _check(_lib.lhaf_rpt(_dp(A), _dp(gamma), _ip(reps), reps.shape[0], _dp(out)))
    return complex(out[0], out[1])


def lhaf_rpt_batch(A, gamma, reps_batch, gamma_per_pattern: bool = False) -> np.ndarray:
    A, gamma, reps = _c128(A), _c128(gamma), _i32(reps_batch)
    batch, k = reps.shape
    stride = gamma.shape[-1] if gamma_per_pattern else 0
    out = np.zeros(2 * batch)
    _check(_lib.lhaf_rpt_batch(_dp(A), _dp(gamma), stride, _ip(reps), k, batch, _dp(out)))
    return out[0::2] + 1j * out[1::2]


def lhaf_rpt_mixed(A2, gamma2, reps) -> complex:
    A2, gamma2, reps = _c128(A2), _c128(gamma2), _i32(reps)
    out = np.zeros(2)
    _check(_lib.lhaf_rpt_mixed(_dp(A2), _dp(gamma2), _ip(reps), reps.shape[0], _dp(out)))
    return complex(out[0], out[1])


def lhaf_gbs_matrices(sigma, alpha):
    """(A, gamma, prefactor) of a Gaussian state (App. A): A = X (I - sigma_Q^-1),
    gamma = alpha^dag sigma_Q^-1, prefactor exp(-alpha^dag sigma_Q^-1 alpha / 2) / sqrt(det sigma_Q)."""
    sigma, alpha = _c128(sigma), _c128(alpha)
    M = alpha.shape[0] // 2
    A = np.zeros((2 * M, 2 * M), np.complex128)
    g = np.zeros(2 * M, np.complex128)
    pref = np.zeros(2)
    _check(_lib.lhaf_gbs_matrices(_dp(sigma), _dp(alpha), M, _dp(A), _dp(g), _dp(pref)))
    return A, g, complex(pref[0], pref[1])


def lhaf_gbs_prob(sigma, alpha, n, pure: bool = False) -> complex:
    """P(n | sigma, alpha) (Eq. mixed_prob); pure=True uses |lhaf(B_n)|^2.
    Returns a complex number whose imaginary part is the rounding residue."""
    sigma, alpha, n = _c128(sigma), _c128(alpha), _i32(n)
    out = np.zeros(2)
    _check(_lib.lhaf_gbs_prob(_dp(sigma), _dp(alpha), n.shape[0], _ip(n), 1 if pure else 0, _dp(out)))
    return complex(out[0], out[1])


def _opt_ptr(x, dtype):
    if x is None:
        return None, None
    arr = np.ascontiguousarray(np.asarray(x, dtype=dtype))
    return arr, arr.ctypes.data


def lhaf_gbs_state(U, r, eta=None, beta=None):
    """(sigma, alpha) of squeezers r -> pure loss eta -> U -> displacement beta."""
    U = _c128(U)
    M = U.shape[0]
    r = np.ascontiguousarray(np.broadcast_to(np.asarray(r, float), (M,)))
    e_arr, e_ptr = _opt_ptr(None if eta is None else np.broadcast_to(np.asarray(eta, float), (M,)), np.float64)
    b_arr, b_ptr = _opt_ptr(beta, np.complex128)
    sig = np.zeros((2 * M, 2 * M), np.complex128)
    al = np.zeros(2 * M, np.complex128)
    _check(_lib.lhaf_gbs_state(_dp(U), _dp(r), e_ptr, b_ptr, M, _dp(sig), _dp(al)))
    return sig, al


def lhaf_gbs_prob_state(U, r, n, eta=None, beta=None) -> complex:
    """P(n) of the state of lhaf_gbs_state in one call."""
    U = _c128(U)
    M = U.shape[0]
    r = np.ascontiguousarray(np.broadcast_to(np.asarray(r, float), (M,)))
    e_arr, e_ptr = _opt_ptr(None if eta is None else np.broadcast_to(np.asarray(eta, float), (M,)), np.float64)
    b_arr, b_ptr = _opt_ptr(beta, np.complex128)
    nn = _i32(n)
    out = np.zeros(2)
    _check(_lib.lhaf_gbs_prob_state(_dp(U), _dp(r), e_ptr, b_ptr, M, _ip(nn), _dp(out)))
    return complex(out[0], out[1])


def lhaf_rpt_multigamma(A, gammas, reps) -> np.ndarray:
    """lhaf of one pattern under each row of gammas (one device job)."""
    A, gammas, reps = _c128(A), _c128(np.atleast_2d(gammas)), _i32(reps)
    out = np.zeros(2 * gammas.shape[0])
    _check(_lib.lhaf_rpt_multigamma(_dp(A), _dp(gammas), gammas.shape[0], _ip(reps), reps.shape[0], _dp(out)))
    return out[0::2] + 1j * out[1::2]


def lhaf_rpt_et(A, gamma, reps) -> complex:
    """lhaf by inclusion/exclusion over the pair copies (ET) on the device path."""
    A, gamma, reps = _c128(A), _c128(gamma), _i32(reps)
    out = np.zeros(2)
    _check(_lib.lhaf_rpt_et(_dp(A), _dp(gamma), _ip(reps), reps.shape[0], _dp(out)))
    return complex(out[0], out[1])


def lhaf_ips_prob(B, alpha, n) -> float:
    """MIS proposal probability Q(n | B, alpha)."""
    B, alpha, n = _c128(B), _c128(alpha), _i32(n)
    out = np.zeros(2)
    _check(_lib.lhaf_ips_prob(_dp(B), _dp(alpha), n.shape[0], _ip(n), _dp(out)))
    return float(out[0])


def lhaf_rpt_cutoff(A, gamma, reps_fixed, mode: int, n_cut: int) -> np.ndarray:
    """lhaf for the pattern reps_fixed with reps[mode] = 0 .. n_cut (App. B.5), one job."""
    A, gamma, reps = _c128(A), _c128(gamma), _i32(reps_fixed)
    out = np.zeros(2 * (n_cut + 1))
    _check(_lib.lhaf_rpt_cutoff(_dp(A), _dp(gamma), _ip(reps), reps.shape[0], mode, n_cut, _dp(out)))
    return out[0::2] + 1j * out[1::2]


def lhaf_rpt_cutoff_ex(A, gamma, reps_fixed, mode: int, n_cut: int, tol: float = 0.0):
    """lhaf_rpt_cutoff plus per-count error estimates kappa_j * 2^-46; with tol > 0 raises
    LhafError (status LHAF_E_INACCURATE) when an estimate exceeds tol.  Returns (values, err)."""
    A, gamma, reps = _c128(A), _c128(gamma), _i32(reps_fixed)
    out = np.zeros(2 * (n_cut + 1))
    err = np.zeros(n_cut + 1)
    _check(_lib.lhaf_rpt_cutoff_ex(_dp(A), _dp(gamma), _ip(reps), reps.shape[0], mode, n_cut,
                                   float(tol), _dp(out), _dp(err)))
    return out[0::2] + 1j * out[1::2], err


def lhaf_rpt_batch_dev(A_dev_ptr: int, gamma_dev_ptr: int, gamma_stride: int, reps_batch,
                       mixed: bool, out_dev_ptr: int, stream_ptr: int = 0):
    """Device-pointer entry (e.g. torch tensors' data_ptr() and current stream)."""
    reps = _i32(reps_batch)
    if reps.ndim == 1:
        reps = reps[None, :]
    batch, k = reps.shape
    _check(_lib.lhaf_rpt_batch_dev(ctypes.c_void_p(A_dev_ptr), ctypes.c_void_p(gamma_dev_ptr),
                                   gamma_stride, _ip(reps), k, batch, int(mixed),
                                   ctypes.c_void_p(out_dev_ptr), ctypes.c_void_p(stream_ptr)))


class Job:
    """A planned, device-resident evaluation (lhaf_job_*).  Inputs are copied to HBM at
    creation; ``run`` evaluates a work-unit range into the chunk-partial array."""

    def __init__(self, A, gamma, reps_batch, mixed: int = 0, gamma_per_pattern: bool = False):
        self._A, self._g, self._reps = _c128(A), _c128(gamma), _i32(reps_batch)
        if self._reps.ndim == 1:
            self._reps = self._reps[None, :]
        batch, k = self._reps.shape
        stride = self._g.shape[-1] if gamma_per_pattern else 0
        h = ctypes.c_void_p()
        _check(_lib.lhaf_job_create(self._A.ctypes.data,
                                    self._g.ctypes.data, stride, _ip(self._reps), k, batch,
                                    int(mixed), 0, ctypes.byref(h)))
        self._h = h
        self.info = JobInfo()
        _check(_lib.lhaf_job_info_get(self._h, ctypes.byref(self.info)))

    @property
    def units(self) -> int:
        return int(self.info.units)

    @property
    def terms(self) -> int:
        return int(self.info.terms)

    def plan(self, pattern: int = 0) -> PlanInfo:
        """The pattern's pairs / multiplicities in the job's evaluation order (lhaf_job_plan)."""
        info = PlanInfo()
        _check(_lib.lhaf_job_plan(self._h, pattern, ctypes.byref(info)))
        return info

    def reset(self, stream: int = 0):
        _check(_lib.lhaf_job_reset(self._h, ctypes.c_void_p(stream)))

    def run(self, unit_begin: int = 0, unit_end: int | None = None, stream: int = 0):
        ue = self.units if unit_end is None else unit_end
        _check(_lib.lhaf_job_run(self._h, unit_begin, ue, ctypes.c_void_p(stream)))

    def allreduce(self, stream: int = 0):
        _check(_lib.lhaf_job_allreduce(self._h, ctypes.c_void_p(stream)))

    def reset_range(self, unit_begin: int, unit_end: int, stream: int = 0):
        _check(_lib.lhaf_job_reset_range(self._h, unit_begin, unit_end, ctypes.c_void_p(stream)))

    def allreduce_range(self, unit_begin: int, unit_end: int, stream: int = 0):
        _check(_lib.lhaf_job_allreduce_range(self._h, unit_begin, unit_end, ctypes.c_void_p(stream)))

    def finalize(self, stream: int = 0) -> np.ndarray:
        out = np.zeros(2 * self.info.batch)
        _check(_lib.lhaf_job_finalize(self._h, out.ctypes.data, 0, ctypes.c_void_p(stream)))
        return out[0::2] + 1j * out[1::2]

    def finalize_dev(self, out_dev_ptr: int, stream: int = 0):
        _check(_lib.lhaf_job_finalize(self._h, ctypes.c_void_p(out_dev_ptr), 1,
                                      ctypes.c_void_p(stream)))

    def abs_sum(self) -> np.ndarray:
        out = np.zeros(self.info.batch)
        _check(_lib.lhaf_job_abs_sum(self._h, _dp(out)))
        return out

    def partials(self):
        p = ctypes.c_void_p()
        nbytes = ctypes.c_size_t()
        _check(_lib.lhaf_job_partials(self._h, ctypes.byref(p), ctypes.byref(nbytes)))
        return p.value, nbytes.value

    def terms_g(self, ts) -> np.ndarray:
        ts = np.ascontiguousarray(np.asarray(ts, dtype=np.uint64))
        out = np.zeros(2 * ts.shape[0])
        _check(_lib.lhaf_job_terms(self._h, ts.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                   ts.shape[0], _dp(out)))
        return out[0::2] + 1j * out[1::2]

    def close(self):
        if getattr(self, "_h", None):
            _lib.lhaf_job_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def lhaf_set_device(device: int):
    _check(_lib.lhaf_set_device(device))


def lhaf_set_kernel(variant: int):
    _check(_lib.lhaf_set_kernel(variant))


def lhaf_set_precision(mode: int):
    """0 = FP64 (default: the tree), 1 = precise per-term (double-double La Budde + series, v5)."""
    _check(_lib.lhaf_set_precision(mode))


def lhaf_get_precision() -> int:
    return int(_lib.lhaf_get_precision())


def lhaf_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.lhaf_get_unique_id(buf))
    return buf.raw


def lhaf_init_rank(rank: int, nranks: int, uid: bytes | None, device: int = -1):
    buf = ctypes.create_string_buffer(uid, 128) if uid is not None else None
    _check(_lib.lhaf_init_rank(rank, nranks, buf, device))


def lhaf_rank_info():
    r, n = ctypes.c_int32(), ctypes.c_int32()
    _check(_lib.lhaf_rank_info(ctypes.byref(r), ctypes.byref(n)))
    return r.value, n.value


def lhaf_shard_units(units: int, rank: int, nranks: int):
    b, e = ctypes.c_uint64(), ctypes.c_uint64()
    _check(_lib.lhaf_shard_units(units, rank, nranks, ctypes.byref(b), ctypes.byref(e)))
    return b.value, e.value


def lhaf_shutdown():
    _lib.lhaf_shutdown()
