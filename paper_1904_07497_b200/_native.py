"""ctypes bindings of the native libraries (C-ABI of include/respca_cu.h).

The CUDA engine is mandatory: there is no CPU fallback.  Loading fails loudly
when librespca_cu.so is missing (run ``python -m paper_1904_07497_b200.build``)
and ``Context()`` fails loudly when no sm_100 device is present.
"""
from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

LIB_DIR = Path(__file__).resolve().parent / "lib"

RESPCA_OK, RESPCA_EINVAL, RESPCA_ERUNTIME, RESPCA_ENOMEM, RESPCA_ECUDA, RESPCA_ENONFINITE, RESPCA_EIO = range(7)
F64, F32 = 0, 1
L1, L21 = 0, 1

u64 = C.c_uint64
dptr = C.POINTER(C.c_double)
u64ptr = C.POINTER(C.c_uint64)


class CConfig(C.Structure):
    """respca_cu_config — SolverConfig + KMeansConfig (solver.hpp:13-28, kmeans.hpp:11-17)."""

    _fields_ = [
        ("has_lambda", C.c_int), ("lambda_", C.c_double), ("rho0", C.c_double),
        ("kappa", C.c_double), ("tol", C.c_double), ("max_iter", u64), ("c", u64),
        ("sparse_norm", C.c_int), ("km_max_iters", u64), ("km_n_restarts", u64),
        ("km_seed", u64), ("km_tol", C.c_double), ("has_fixed_iters", C.c_int),
        ("fixed_iters", u64),
    ]


class CReport(C.Structure):
    """respca_cu_report — ConvergenceReport (solver.hpp:39-46) + timings."""

    _fields_ = [
        ("feas", dptr), ("delta_l", dptr), ("delta_s", dptr), ("objective", dptr),
        ("iters", u64), ("converged", C.c_int), ("lambda_", C.c_double),
        ("wall_time", C.c_double), ("init_ms", C.c_double), ("loop_ms", C.c_double),
        ("h2d_ms", C.c_double), ("d2h_ms", C.c_double), ("slow_iters", u64),
        ("hartigan_moves", u64), ("exact_fallbacks", u64), ("stop_resolves", u64),
    ]


class CMargins(C.Structure):
    """respca_cu_margins — decision margins of the last solve."""

    _fields_ = [("alm_stop", C.c_double), ("alm_stop_final", C.c_double), ("s_support", C.c_double),
                ("lloyd_stop", C.c_double), ("restart_gap", C.c_double), ("stop_resolves", u64)]


_lib = None
_lock = threading.RLock()

# every symbol include/respca_cu.h declares (checked by tests/test_boundary.py)
EXPORTS = [
    "respca_cu_default_config", "respca_cu_create", "respca_cu_destroy", "respca_cu_last_error",
    "respca_cu_kernel_launches", "respca_cu_solve", "respca_cu_l_update",
    "respca_cu_s_update_l1", "respca_cu_s_update_l21", "respca_cu_multiplier_update",
    "respca_cu_check_convergence", "respca_cu_kmeans", "respca_cu_kmeans_warm",
    "respca_cu_kmeans_pp_init", "respca_cu_lloyd_step", "respca_cu_group_scatter",
    "respca_cu_frob_norm", "respca_cu_elementwise_l1", "respca_cu_l21_norm",
    "respca_cu_column_l2_norms", "respca_cu_column_mean", "respca_cu_bench_prepare",
    "respca_cu_bench_steps", "respca_cu_debug_screen", "respca_cu_kmeans_pp_init_cb",
    "respca_cu_debug_screen_tc", "respca_cu_debug_guards", "respca_cu_last_margins", "respca_cu_binary_info", "respca_cu_solve_file",
    "respca_cu_outlier_scores", "respca_cu_synth_rpca", "respca_cu_synth_generate",
]


def lib() -> C.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            path = LIB_DIR / "librespca_cu.so"
            if not path.exists():
                raise RuntimeError(
                    f"{path} is missing: build the CUDA engine first "
                    "(python -m paper_1904_07497_b200.build); there is no CPU fallback")
            L = C.CDLL(str(path))
            vp = C.c_void_p
            L.respca_cu_default_config.argtypes = [C.POINTER(CConfig)]
            L.respca_cu_default_config.restype = None
            L.respca_cu_create.argtypes = [C.c_int, C.POINTER(vp)]
            L.respca_cu_destroy.argtypes = [vp]
            L.respca_cu_destroy.restype = None
            L.respca_cu_last_error.argtypes = [vp]
            L.respca_cu_last_error.restype = C.c_char_p
            L.respca_cu_kernel_launches.argtypes = [vp]
            L.respca_cu_kernel_launches.restype = u64
            L.respca_cu_solve.argtypes = [vp, vp, u64, u64, C.c_int, C.POINTER(CConfig), vp, vp,
                                          u64ptr, C.POINTER(CReport)]
            L.respca_cu_l_update.argtypes = [vp, dptr, u64, u64, u64ptr, u64, C.c_double,
                                             C.c_double, dptr]
            L.respca_cu_s_update_l1.argtypes = [vp, dptr, u64, u64, C.c_double, dptr]
            L.respca_cu_s_update_l21.argtypes = [vp, dptr, u64, u64, C.c_double, dptr]
            L.respca_cu_multiplier_update.argtypes = [vp, dptr, dptr, dptr, dptr, u64, u64, dptr,
                                                      C.c_double]
            L.respca_cu_check_convergence.argtypes = [vp, dptr, dptr, dptr, dptr, dptr, u64, u64,
                                                      C.c_double, C.POINTER(C.c_int), dptr, dptr,
                                                      dptr]
            L.respca_cu_kmeans.argtypes = [vp, dptr, u64, u64, u64, u64, u64, u64, C.c_double,
                                           u64ptr, dptr, dptr, u64ptr]
            L.respca_cu_kmeans_warm.argtypes = [vp, dptr, u64, u64, u64, u64, C.c_double, u64ptr,
                                                u64ptr, dptr, dptr, u64ptr]
            L.respca_cu_kmeans_pp_init.argtypes = [vp, dptr, u64, u64, u64, u64, dptr]
            L.respca_cu_lloyd_step.argtypes = [vp, dptr, u64, u64, dptr, u64, u64ptr, dptr]
            L.respca_cu_group_scatter.argtypes = [vp, dptr, u64, u64, u64ptr, u64, dptr]
            for nm in ("respca_cu_frob_norm", "respca_cu_elementwise_l1", "respca_cu_l21_norm",
                       "respca_cu_column_l2_norms"):
                getattr(L, nm).argtypes = [vp, dptr, u64, u64, dptr]
            L.respca_cu_column_mean.argtypes = [vp, dptr, u64, u64, u64ptr, u64, dptr]
            L.respca_cu_bench_prepare.argtypes = [vp, vp, u64, u64, C.c_int, C.POINTER(CConfig),
                                                  dptr]
            L.respca_cu_bench_steps.argtypes = [vp, u64, dptr, dptr, dptr, u64ptr]
            L.respca_cu_debug_screen.argtypes = [vp, dptr, u64, u64, dptr, u64, dptr, dptr]
            L.respca_cu_debug_screen_tc.argtypes = [vp, dptr, u64, u64, dptr, u64, dptr, dptr]
            L.respca_cu_debug_guards.argtypes = [C.c_char_p, u64]
            L.respca_cu_last_margins.argtypes = [vp, C.POINTER(CMargins)]
            L.respca_cu_binary_info.argtypes = [C.c_char_p, u64ptr, u64ptr, C.c_char_p, C.c_size_t]
            L.respca_cu_solve_file.argtypes = [vp, C.c_char_p, C.c_int, C.POINTER(CConfig),
                                               C.c_char_p, C.c_char_p, u64ptr, u64, C.POINTER(CReport)]
            L.respca_cu_outlier_scores.argtypes = [vp, dptr, u64, u64, C.c_double, dptr, u64ptr,
                                                   u64ptr]
            L.respca_cu_synth_rpca.argtypes = [vp, u64, u64, u64, C.c_double, C.c_double, C.c_double,
                                               C.c_double, u64, C.c_int, vp]
            L.respca_cu_synth_generate.argtypes = [vp, u64, u64, u64, C.c_double, C.c_double, C.c_double,
                                                   u64, vp, vp, vp, vp]
            _lib = L
        return _lib


class Context:
    """Owns one respca_cu_ctx (device buffers, streams, graphs) on one GPU."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        rc = lib().respca_cu_create(device, C.byref(self._h))
        if rc != RESPCA_OK:
            raise RuntimeError(
                f"respca_cu_create(device={device}) failed (status {rc}): no usable sm_100 "
                "CUDA device; this solver has no CPU fallback")

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def last_error(self) -> str:
        return lib().respca_cu_last_error(self._h).decode()

    def launches(self) -> int:
        return int(lib().respca_cu_kernel_launches(self._h))

    def close(self) -> None:
        if self._h:
            lib().respca_cu_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    with _lock:
        if _default_ctx is None:
            _default_ctx = Context(0)
        return _default_ctx


def check(ctx: Context, rc: int) -> None:
    """Map a status code onto the reference's exception classes."""
    if rc == RESPCA_OK:
        return
    msg = ctx.last_error()
    if rc == RESPCA_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if rc == RESPCA_ERUNTIME:
        raise RuntimeError(msg)  # std::runtime_error
    if rc == RESPCA_ENOMEM:
        raise MemoryError(msg)
    if rc == RESPCA_ENONFINITE:
        raise FloatingPointError(msg)
    if rc == RESPCA_EIO:
        raise IoError(msg)  # respca::io::IoError
    raise RuntimeError(f"CUDA error: {msg}")


class IoError(OSError):
    """respca::io::IoError family (io.hpp:13-33): open, magic, truncation."""
