"""Python host mirror of the reference's public API (proj/include/respca/*.hpp).

Same names, argument meaning and error behaviour as the C++ reference:
``std::invalid_argument`` → ``ValueError``, ``std::runtime_error`` →
``RuntimeError``.  Matrices are numpy arrays of shape (d, n) holding columns
as samples; they are passed to the device column-major (the reference's
DenseMatrix layout, matrix.hpp:26-31).  Every call runs on the GPU through the
C-ABI of include/respca_cu.h — there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as N


# --------------------------------------------------------------------------
# types (solver.hpp:13-62, kmeans.hpp:11-24)
# --------------------------------------------------------------------------
@dataclass
class KMeansConfig:
    c: int = 1
    max_iters: int = 100
    n_restarts: int = 1
    seed: int = 0
    tol: float = 1e-6


@dataclass
class SolverConfig:
    lambda_: Optional[float] = None  # unset → sqrt(max(d, n))  (solver.cpp:35-38)
    rho0: float = 1e-4
    kappa: float = 1.5
    tol: float = 1e-3
    max_iter: int = 500
    c: int = 1
    sparse_norm: str = "L1"  # "L1" | "L21"
    kmeans: KMeansConfig = field(default_factory=KMeansConfig)
    fixed_iters: Optional[int] = None

    def resolve_lambda(self, rows: int, cols: int) -> float:
        if self.lambda_ is not None:
            return float(self.lambda_)
        return float(np.sqrt(float(max(rows, cols))))

    def validate(self) -> None:  # solver.cpp:40-47
        if self.lambda_ is not None and self.lambda_ <= 0.0:
            raise ValueError("lambda must be > 0")
        if self.rho0 <= 0.0:
            raise ValueError("rho0 must be > 0")
        if self.kappa <= 1.0:
            raise ValueError("kappa must be > 1")
        if self.tol <= 0.0:
            raise ValueError("tol must be > 0")
        if self.c == 0:
            raise ValueError("c must be >= 1")
        if self.max_iter == 0:
            raise ValueError("max_iter must be >= 1")

    def to_c(self) -> N.CConfig:
        cc = N.CConfig()
        cc.has_lambda = 0 if self.lambda_ is None else 1
        cc.lambda_ = 0.0 if self.lambda_ is None else float(self.lambda_)
        cc.rho0, cc.kappa, cc.tol = float(self.rho0), float(self.kappa), float(self.tol)
        cc.max_iter, cc.c = int(self.max_iter), int(self.c)
        cc.sparse_norm = N.L21 if self.sparse_norm.upper() == "L21" else N.L1
        cc.km_max_iters, cc.km_n_restarts = int(self.kmeans.max_iters), int(self.kmeans.n_restarts)
        cc.km_seed, cc.km_tol = int(self.kmeans.seed), float(self.kmeans.tol)
        cc.has_fixed_iters = 0 if self.fixed_iters is None else 1
        cc.fixed_iters = 0 if self.fixed_iters is None else int(self.fixed_iters)
        return cc


@dataclass
class ConvergenceReport:
    feas: np.ndarray
    delta_l: np.ndarray
    delta_s: np.ndarray
    objective: np.ndarray
    converged: bool
    iters: int


@dataclass
class DecompositionResult:
    L: np.ndarray
    S: np.ndarray
    assignment: np.ndarray  # uint64 labels, length n
    report: ConvergenceReport
    wall_time: float
    lambda_: float
    init_ms: float = 0.0
    loop_ms: float = 0.0
    h2d_ms: float = 0.0
    d2h_ms: float = 0.0
    slow_iters: int = 0
    hartigan_moves: int = 0
    exact_fallbacks: int = 0
    stop_resolves: int = 0  # stop tests decided on the reference's sequential residual chains
    margins: Optional[dict] = None  # decision margins, see last_margins()


@dataclass
class KMeansResult:
    assignment: np.ndarray
    centroids: np.ndarray
    inertia: float
    iters_run: int


# --------------------------------------------------------------------------
# helpers
# --------------------------------------------------------------------------
def _ctx(ctx):
    return ctx if ctx is not None else N.default_context()


def _mat(a, dtype=np.float64) -> np.ndarray:
    a = np.asarray(a)
    if a.ndim != 2:
        raise ValueError("DenseMatrix: expected a 2-D (d, n) array")
    return np.asfortranarray(a, dtype=dtype)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(N.dptr)


def _labels(labels) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(labels), dtype=np.uint64)


def _up(a: np.ndarray):
    return a.ctypes.data_as(N.u64ptr)


# --------------------------------------------------------------------------
# solver (solver.hpp:67-88)
# --------------------------------------------------------------------------
def solve(x, cfg: Optional[SolverConfig] = None, precision: str = "f64",
          ctx: Optional[N.Context] = None, out=None) -> DecompositionResult:
    """respca::solve (solver.cpp:127-210) on the device.  precision "f32" is
    the API extension of the B200 build (fp32 storage, fp64 arithmetic).
    `out=(L, S)`: optional preallocated Fortran-ordered outputs (e.g. pinned)."""
    cfg = cfg or SolverConfig()
    ctx = _ctx(ctx)
    dt = np.float32 if precision == "f32" else np.float64
    xm = _mat(x, dt)
    d, n = xm.shape
    budget = cfg.fixed_iters if cfg.fixed_iters is not None else cfg.max_iter
    budget = max(int(budget), 1)  # allocation only: the solver writes rep.iters (0 for fixed_iters=0)
    if out is not None:
        L, S = out
        for a in (L, S):
            if a.shape != (d, n) or a.dtype != dt or not a.flags.f_contiguous:
                raise ValueError("solve: out arrays must be Fortran-ordered (d, n) of the dtype")
    else:
        L = np.empty((d, n), dtype=dt, order="F")
        S = np.empty((d, n), dtype=dt, order="F")
    lab = np.empty(n, dtype=np.uint64)
    arrs = [np.zeros(budget) for _ in range(4)]
    rep = N.CReport()
    rep.feas, rep.delta_l, rep.delta_s, rep.objective = (_dp(a) for a in arrs)
    cc = cfg.to_c()
    rc = N.lib().respca_cu_solve(ctx.handle, xm.ctypes.data_as(C.c_void_p), d, n,
                                 N.F32 if dt == np.float32 else N.F64, C.byref(cc),
                                 L.ctypes.data_as(C.c_void_p), S.ctypes.data_as(C.c_void_p),
                                 _up(lab), C.byref(rep))
    N.check(ctx, rc)
    it = int(rep.iters)
    report = ConvergenceReport(arrs[0][:it].copy(), arrs[1][:it].copy(), arrs[2][:it].copy(),
                               arrs[3][:it].copy(), bool(rep.converged), it)
    return DecompositionResult(L, S, lab, report, float(rep.wall_time), float(rep.lambda_),
                               float(rep.init_ms), float(rep.loop_ms), float(rep.h2d_ms),
                               float(rep.d2h_ms), int(rep.slow_iters), int(rep.hartigan_moves),
                               int(rep.exact_fallbacks), int(rep.stop_resolves), last_margins(ctx))


def last_margins(ctx=None) -> dict:
    """Decision margins of the context's last solve (respca_cu_margins,
    SURVEY.md Appendix A): relative distance of each discrete decision of the
    reference from its threshold; inf where the decision did not occur."""
    ctx = _ctx(ctx)
    m = N.CMargins()
    N.check(ctx, N.lib().respca_cu_last_margins(ctx.handle, C.byref(m)))
    return {k: (int(getattr(m, k)) if k == "stop_resolves" else float(getattr(m, k)))
            for k, _ in N.CMargins._fields_}


def _result(L, S, lab, arrs, rep) -> DecompositionResult:
    it = int(rep.iters)
    report = ConvergenceReport(arrs[0][:it].copy(), arrs[1][:it].copy(), arrs[2][:it].copy(),
                               arrs[3][:it].copy(), bool(rep.converged), it)
    return DecompositionResult(L, S, lab, report, float(rep.wall_time), float(rep.lambda_),
                               float(rep.init_ms), float(rep.loop_ms), float(rep.h2d_ms),
                               float(rep.d2h_ms), int(rep.slow_iters), int(rep.hartigan_moves),
                               int(rep.exact_fallbacks), int(rep.stop_resolves))


def binary_info(path) -> tuple[int, int]:
    """Rows and columns of a RESPCA1 file (io.hpp:66-69), validated like
    read_binary_matrix (io.cpp:138-153).  No GPU needed."""
    r, c = C.c_uint64(), C.c_uint64()
    err = C.create_string_buffer(512)
    rc = N.lib().respca_cu_binary_info(str(path).encode(), C.byref(r), C.byref(c), err, 512)
    if rc == N.RESPCA_EIO:
        raise N.IoError(err.value.decode())
    if rc != N.RESPCA_OK:
        raise ValueError(err.value.decode())
    return int(r.value), int(c.value)


def solve_file(x_path, cfg: Optional[SolverConfig] = None, l_path=None, s_path=None,
               precision: str = "f64", ctx: Optional[N.Context] = None) -> DecompositionResult:
    """solve() between RESPCA1 files, streamed disk → HBM → disk in pinned
    chunks.  The result carries no L/S arrays (None):
    they are in `l_path` / `s_path` when given."""
    cfg = cfg or SolverConfig()
    ctx = _ctx(ctx)
    d, n = binary_info(x_path)
    budget = cfg.fixed_iters if cfg.fixed_iters is not None else cfg.max_iter
    budget = max(int(budget), 1)  # allocation only: the solver writes rep.iters (0 for fixed_iters=0)
    lab = np.empty(n, dtype=np.uint64)
    arrs = [np.zeros(budget) for _ in range(4)]
    rep = N.CReport()
    rep.feas, rep.delta_l, rep.delta_s, rep.objective = (_dp(a) for a in arrs)
    cc = cfg.to_c()
    enc = (lambda p: None if p is None else str(p).encode())
    rc = N.lib().respca_cu_solve_file(ctx.handle, str(x_path).encode(),
                                      N.F32 if precision == "f32" else N.F64, C.byref(cc),
                                      enc(l_path), enc(s_path), _up(lab), n, C.byref(rep))
    N.check(ctx, rc)
    return _result(None, None, lab, arrs, rep)


class OutlierScores:
    """io::OutlierScores (io.hpp:100-103)."""

    def __init__(self, scores: np.ndarray, flagged: np.ndarray):
        self.scores = scores
        self.flagged = flagged


def outlier_scores(s, threshold: float, ctx=None) -> OutlierScores:
    """io::outlier_scores (io.cpp:296-306): column ℓ2 norms of S (the
    reference's sequential order) and the columns at or above `threshold`."""
    ctx = _ctx(ctx)
    sm = _mat(s)
    d, n = sm.shape
    sc = np.empty(n)
    fl = np.empty(n, dtype=np.uint64)
    nf = C.c_uint64()
    N.check(ctx, N.lib().respca_cu_outlier_scores(ctx.handle, _dp(sm), d, n, float(threshold),
                                                 _dp(sc), _up(fl), C.byref(nf)))
    return OutlierScores(sc, fl[: nf.value].copy())


@dataclass
class SynthData:
    """io.hpp SynthData: the generated problem and its ground truth."""
    x: np.ndarray
    l0: np.ndarray
    s0: np.ndarray
    assignment: np.ndarray


def synth_generate(d: int, n: int, c: int, sparsity: float = 0.05, magnitude: float = 1.0,
                   noise_sigma: float = 0.0, seed: int = 0, ctx=None) -> SynthData:
    """io::synth_generate (io.cpp:232-294): the reference's synthetic problem,
    byte-identical, with the d×n assembly on the device
    (respca_cu_synth_generate).  ValueError carries the reference's message."""
    ctx = _ctx(ctx)
    d, n, c = int(d), int(n), int(c)
    shape = (max(d, 0), max(n, 0))
    x, l0, s0 = (np.empty(shape, order="F") for _ in range(3))
    lab = np.empty(max(n, 0), dtype=np.uint64)
    rc = N.lib().respca_cu_synth_generate(ctx.handle, d, n, c, float(sparsity), float(magnitude),
                                          float(noise_sigma), int(seed), x.ctypes.data_as(C.c_void_p),
                                          l0.ctypes.data_as(C.c_void_p), s0.ctypes.data_as(C.c_void_p),
                                          lab.ctypes.data_as(C.c_void_p))
    N.check(ctx, rc)
    return SynthData(x, l0, s0, lab)


def write_binary_matrix(path, m) -> None:
    """RESPCA1 writer (io.cpp:156-164): magic, u64le rows, u64le cols, f64le
    column-major payload.  Host-side helper (tests, tools)."""
    a = np.asfortranarray(np.asarray(m, dtype=np.float64))
    with open(path, "wb") as f:
        f.write(b"RESPCA1\0")
        f.write(np.array(a.shape, dtype="<u8").tobytes())
        f.write(a.astype("<f8").tobytes(order="F"))


def read_binary_matrix(path) -> np.ndarray:
    """RESPCA1 reader with the reference's checks (io.cpp:138-153)."""
    d, n = binary_info(path)
    with open(path, "rb") as f:
        f.seek(24)
        a = np.fromfile(f, dtype="<f8", count=d * n)
    return np.asfortranarray(a.reshape((d, n), order="F"))


def l_update(D, labels, c: int, lambda_: float, rho: float, ctx=None) -> np.ndarray:
    ctx = _ctx(ctx)
    Dm = _mat(D)
    lab = _labels(labels)
    if lab.size != Dm.shape[1]:
        raise ValueError("l_update: assignment length != column count")
    out = np.empty_like(Dm, order="F")
    N.check(ctx, N.lib().respca_cu_l_update(ctx.handle, _dp(Dm), Dm.shape[0], Dm.shape[1],
                                             _up(lab), int(c), float(lambda_), float(rho),
                                             _dp(out)))
    return out


def s_update_l1(B, threshold: float, ctx=None) -> np.ndarray:
    ctx = _ctx(ctx)
    Bm = _mat(B)
    out = np.empty_like(Bm, order="F")
    N.check(ctx, N.lib().respca_cu_s_update_l1(ctx.handle, _dp(Bm), *Bm.shape, float(threshold),
                                                _dp(out)))
    return out


def s_update_l21(B, threshold: float, ctx=None) -> np.ndarray:
    ctx = _ctx(ctx)
    Bm = _mat(B)
    out = np.empty_like(Bm, order="F")
    N.check(ctx, N.lib().respca_cu_s_update_l21(ctx.handle, _dp(Bm), *Bm.shape, float(threshold),
                                                 _dp(out)))
    return out


def multiplier_update(theta, x, L, S, rho: float, kappa: float, ctx=None):
    """Θ += ρ(X − L − S); ρ = min(ρκ, 1e12).  Returns (Θ', ρ')."""
    ctx = _ctx(ctx)
    th = np.array(_mat(theta), order="F", copy=True)
    xm, lm, sm = _mat(x), _mat(L), _mat(S)
    r = C.c_double(float(rho))
    N.check(ctx, N.lib().respca_cu_multiplier_update(ctx.handle, _dp(th), _dp(xm), _dp(lm),
                                                      _dp(sm), *xm.shape, C.byref(r),
                                                      float(kappa)))
    return th, r.value


def check_convergence(x, l_prev, l, s_prev, s, tol: float, ctx=None):
    """Returns (converged, (feas, delta_l, delta_s))."""
    ctx = _ctx(ctx)
    ms = [_mat(a) for a in (x, l_prev, l, s_prev, s)]
    conv = C.c_int()
    f, dl, ds = C.c_double(), C.c_double(), C.c_double()
    N.check(ctx, N.lib().respca_cu_check_convergence(ctx.handle, *(_dp(a) for a in ms),
                                                      *ms[0].shape, float(tol), C.byref(conv),
                                                      C.byref(f), C.byref(dl), C.byref(ds)))
    return bool(conv.value), (f.value, dl.value, ds.value)


# --------------------------------------------------------------------------
# clustering (kmeans.hpp:28-43)
# --------------------------------------------------------------------------
def kmeans(m, cfg: KMeansConfig, ctx=None) -> KMeansResult:
    ctx = _ctx(ctx)
    mm = _mat(m)
    d, n = mm.shape
    c = int(cfg.c)
    lab = np.empty(n, dtype=np.uint64)
    cen = np.empty((d, max(c, 1)), order="F")
    inert, it = C.c_double(), C.c_uint64()
    N.check(ctx, N.lib().respca_cu_kmeans(ctx.handle, _dp(mm), d, n, c, int(cfg.max_iters),
                                           int(cfg.n_restarts), int(cfg.seed), float(cfg.tol),
                                           _up(lab), _dp(cen), C.byref(inert), C.byref(it)))
    return KMeansResult(lab, cen, inert.value, int(it.value))


def kmeans_warm(m, cfg: KMeansConfig, init_labels, ctx=None) -> KMeansResult:
    ctx = _ctx(ctx)
    mm = _mat(m)
    d, n = mm.shape
    init = _labels(init_labels)
    if init.size != n:
        raise ValueError("kmeans_warm: assignment does not match")
    c = int(cfg.c)
    lab = np.empty(n, dtype=np.uint64)
    cen = np.empty((d, max(c, 1)), order="F")
    inert, it = C.c_double(), C.c_uint64()
    N.check(ctx, N.lib().respca_cu_kmeans_warm(ctx.handle, _dp(mm), d, n, c, int(cfg.max_iters),
                                                float(cfg.tol), _up(init), _up(lab), _dp(cen),
                                                C.byref(inert), C.byref(it)))
    return KMeansResult(lab, cen, inert.value, int(it.value))


def kmeans_pp_init(m, c: int, seed: int, ctx=None) -> np.ndarray:
    ctx = _ctx(ctx)
    mm = _mat(m)
    d, n = mm.shape
    cen = np.empty((d, max(int(c), 1)), order="F")
    N.check(ctx, N.lib().respca_cu_kmeans_pp_init(ctx.handle, _dp(mm), d, n, int(c), int(seed),
                                                   _dp(cen)))
    return cen


def lloyd_step(m, centroids, ctx=None):
    ctx = _ctx(ctx)
    mm, cm = _mat(m), _mat(centroids)
    d, n = mm.shape
    if cm.shape[0] != d or cm.shape[1] == 0:
        raise ValueError("lloyd_step: bad centroid matrix")
    lab = np.empty(n, dtype=np.uint64)
    nxt = np.empty_like(cm, order="F")
    N.check(ctx, N.lib().respca_cu_lloyd_step(ctx.handle, _dp(mm), d, n, _dp(cm), cm.shape[1],
                                               _up(lab), _dp(nxt)))
    return lab, nxt


# --------------------------------------------------------------------------
# core (matrix.hpp:82-98)
# --------------------------------------------------------------------------
def group_scatter(m, labels, c: int, ctx=None) -> float:
    ctx = _ctx(ctx)
    mm = _mat(m)
    lab = _labels(labels)
    if lab.size != mm.shape[1]:
        raise ValueError("group_scatter: assignment length != column count")
    out = C.c_double()
    N.check(ctx, N.lib().respca_cu_group_scatter(ctx.handle, _dp(mm), *mm.shape, _up(lab), int(c),
                                                  C.byref(out)))
    return out.value


def _scalar(fn, m, ctx) -> float:
    ctx = _ctx(ctx)
    mm = _mat(m)
    out = C.c_double()
    N.check(ctx, getattr(N.lib(), fn)(ctx.handle, _dp(mm), *mm.shape, C.byref(out)))
    return out.value


def frob_norm(m, ctx=None) -> float:
    return _scalar("respca_cu_frob_norm", m, ctx)


def elementwise_l1(m, ctx=None) -> float:
    return _scalar("respca_cu_elementwise_l1", m, ctx)


def l21_norm(m, ctx=None) -> float:
    return _scalar("respca_cu_l21_norm", m, ctx)


def column_l2_norms(m, ctx=None) -> np.ndarray:
    ctx = _ctx(ctx)
    mm = _mat(m)
    out = np.empty(mm.shape[1])
    N.check(ctx, N.lib().respca_cu_column_l2_norms(ctx.handle, _dp(mm), *mm.shape, _dp(out)))
    return out


def column_mean(m, columns, ctx=None) -> np.ndarray:
    ctx = _ctx(ctx)
    mm = _mat(m)
    cols = _labels(columns)
    out = np.empty(mm.shape[0])
    N.check(ctx, N.lib().respca_cu_column_mean(ctx.handle, _dp(mm), *mm.shape, _up(cols),
                                                cols.size, _dp(out)))
    return out
