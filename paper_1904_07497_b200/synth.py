"""Synthetic inputs for the BASELINE.json configurations (host generator,
csrc/synth.c, version "respca-synth-1").  The reference ships no benchmark data
and the paper's video datasets are absent, so seeded synthetic matrices with
BASELINE.json's shapes and distributions stand in."""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

LIB = Path(__file__).resolve().parent / "lib" / "libsynth.so"


class _Rpca(C.Structure):
    _fields_ = [("d", C.c_uint64), ("n", C.c_uint64), ("r", C.c_uint64), ("sigma", C.c_double),
                ("p", C.c_double), ("lo", C.c_double), ("hi", C.c_double), ("seed", C.c_uint64)]


class _Video(C.Structure):
    _fields_ = [("height", C.c_uint64), ("width", C.c_uint64), ("frames", C.c_uint64),
                ("block", C.c_uint64), ("blur_sigma", C.c_double), ("noise_sigma", C.c_double),
                ("seed", C.c_uint64)]


_lib = None
_lib_path = None


def use_library(path) -> None:
    """Load the generator from `path` instead of lib/libsynth.so — bench.py's
    reference arm uses the copy oracle/Makefile builds (oracle/libinput.so) so
    that arm loads no library of this package."""
    global _lib, _lib_path
    _lib, _lib_path = None, Path(path)


def _L():
    global _lib
    if _lib is None:
        path = _lib_path or LIB
        if _lib_path is None and not LIB.exists():
            from .build import build_synth
            build_synth()
        _lib = C.CDLL(str(path))
        _lib.synth_rpca.argtypes = [C.POINTER(_Rpca), C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.synth_video.argtypes = [C.POINTER(_Video), C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.synth_version.restype = C.c_char_p
    return _lib


def version() -> str:
    return _L().synth_version().decode()


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def rpca(d: int, n: int, r: int, sigma: float, p: float, lo: float = -50.0, hi: float = 50.0,
         seed: int = 42, with_truth: bool = False, out: np.ndarray | None = None):
    """X = U·Vᵀ + S0 (column-major (d, n) float64).  Returns X or (X, L0, S0).
    `out`: optional preallocated Fortran-ordered (d, n) float64 (e.g. pinned)."""
    if out is not None:
        assert out.shape == (d, n) and out.dtype == np.float64 and out.flags.f_contiguous
    X = out if out is not None else np.empty((d, n), order="F")
    L0 = np.empty((d, n), order="F") if with_truth else None
    S0 = np.empty((d, n), order="F") if with_truth else None
    spec = _Rpca(d, n, r, sigma, p, lo, hi, seed)
    if _L().synth_rpca(C.byref(spec), _ptr(X), _ptr(L0), _ptr(S0)) != 0:
        raise ValueError("synth_rpca: bad spec or out of memory")
    return (X, L0, S0) if with_truth else X


def rpca_device(d: int, n: int, r: int, sigma: float, p: float, lo: float = -50.0,
                hi: float = 50.0, seed: int = 42, dtype=np.float64, out: np.ndarray | None = None,
                ctx=None) -> np.ndarray:
    """rpca() with the O(d·n) assembly on the GPU (respca_cu_synth_rpca):
    byte-identical to the host generator, milliseconds instead of seconds at
    C3/C5 sizes.  `dtype` float32 gives the rounded copy synth_to_f32 makes."""
    from . import _native as N

    dt = np.dtype(dtype)
    if out is not None:
        assert out.shape == (d, n) and out.dtype == dt and out.flags.f_contiguous
    X = out if out is not None else np.empty((d, n), dtype=dt, order="F")
    ctx = ctx if ctx is not None else N.default_context()
    rc = N.lib().respca_cu_synth_rpca(ctx.handle, d, n, r, sigma, p, lo, hi, seed,
                                      N.F32 if dt == np.float32 else N.F64,
                                      X.ctypes.data_as(C.c_void_p))
    N.check(ctx, rc)
    return X


def video(frames: int = 1000, height: int = 240, width: int = 320, block: int = 40,
          blur_sigma: float = 24.0, noise_sigma: float = 0.01, seed: int = 42,
          with_truth: bool = False):
    d = height * width
    X = np.empty((d, frames), order="F")
    L0 = np.empty((d, frames), order="F") if with_truth else None
    S0 = np.empty((d, frames), order="F") if with_truth else None
    spec = _Video(height, width, frames, block, blur_sigma, noise_sigma, seed)
    if _L().synth_video(C.byref(spec), _ptr(X), _ptr(L0), _ptr(S0)) != 0:
        raise ValueError("synth_video: bad spec")
    return (X, L0, S0) if with_truth else X


@dataclass
class Workload:
    """One BASELINE.json configuration: generator + solver options."""

    name: str
    d: int
    n: int
    c: int
    tol: float
    dtype: str = "f64"
    kind: str = "rpca"
    r: int = 0
    sigma: float = 1.0
    p: float = 0.0
    lambda_: float | None = None
    seed: int = 42
    extra: dict = field(default_factory=dict)

    def make(self, with_truth: bool = False, out: np.ndarray | None = None):
        if self.kind == "video":
            v = video(frames=self.n, seed=self.seed, with_truth=with_truth)
            if out is not None and not with_truth:  # callers that pass `out` read it
                out[...] = v
                return out
            return v
        return rpca(self.d, self.n, self.r, self.sigma, self.p, seed=self.seed,
                    with_truth=with_truth, out=out)

    def make_device(self, out: np.ndarray | None = None, ctx=None):
        """make() with the O(d·n) assembly on the GPU when the generator has one
        (rpca); same bytes."""
        if self.kind != "rpca":
            return self.make(out=out)
        return rpca_device(self.d, self.n, self.r, self.sigma, self.p, seed=self.seed, out=out,
                           ctx=ctx)

    def solver_config(self, **over):
        from .respca import KMeansConfig, SolverConfig

        cfg = SolverConfig(lambda_=self.lambda_, tol=self.tol, c=self.c, kmeans=KMeansConfig())
        for k, v in over.items():
            setattr(cfg, k, v)
        return cfg


# BASELINE.json configs (App. C resolves the ambiguities:
# N(0, 1/sqrt(r)) is read as std 1/sqrt(r); "rank unknown" = c left at the
# library default 1; C4 tol 1e-5).
WORKLOADS = {
    "C1": Workload("C1", 500, 500, 25, 1e-7, r=25, sigma=1.0, p=0.05,
                   lambda_=1.0 / math.sqrt(500.0)),
    "C1-default-lambda": Workload("C1-default-lambda", 500, 500, 25, 1e-7, r=25, sigma=1.0,
                                  p=0.05),
    "C1-c1": Workload("C1-c1", 500, 500, 1, 1e-7, r=25, sigma=1.0, p=0.05),
    "C2": Workload("C2", 2000, 2000, 100, 1e-7, r=100, sigma=1.0, p=0.10),
    "C2-c1": Workload("C2-c1", 2000, 2000, 1, 1e-7, r=100, sigma=1.0, p=0.10),
    "C3": Workload("C3", 10000, 10000, 50, 1e-7, r=50, sigma=1.0 / math.sqrt(50.0), p=0.10),
    "C3-f32": Workload("C3-f32", 10000, 10000, 50, 1e-5, dtype="f32", r=50,
                       sigma=1.0 / math.sqrt(50.0), p=0.10),
    "C3-c1": Workload("C3-c1", 10000, 10000, 1, 1e-7, r=50, sigma=1.0 / math.sqrt(50.0), p=0.10),
    "C4": Workload("C4", 76800, 1000, 3, 1e-5, dtype="f32", kind="video"),
    "C5": Workload("C5", 40000, 40000, 1, 1e-6, r=20, sigma=1.0 / math.sqrt(20.0), p=0.05),
}
