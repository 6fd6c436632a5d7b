"""TEST INFRASTRUCTURE — Python view of the CPU checkers (see oracle_abi.h).

    port()      -> the C restatement (oracle/liboracle.so)
    reference() -> the unmodified reference compiled from /root/reference
                   (oracle/_ref/librespca_ref.so; prebuilt copy on the GPU box)

Both expose the same methods, named like the reference API, so parity tests
read like the reference's own tests.  Only tests/, __graft_entry__.smoke() and
bench.py's CPU legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import math
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
u64 = C.c_uint64
dptr = C.POINTER(C.c_double)
u64ptr = C.POINTER(C.c_uint64)


class OrcConfig(C.Structure):
    _fields_ = [
        ("has_lambda", C.c_int), ("lambda_", C.c_double), ("rho0", C.c_double),
        ("kappa", C.c_double), ("tol", C.c_double), ("max_iter", u64), ("c", u64),
        ("sparse_norm", C.c_int), ("km_max_iters", u64), ("km_n_restarts", u64),
        ("km_seed", u64), ("km_tol", C.c_double), ("has_fixed_iters", C.c_int),
        ("fixed_iters", u64),
    ]


def make_config(cfg) -> OrcConfig:
    """From a paper_1904_07497_b200.respca.SolverConfig-like object."""
    o = OrcConfig()
    o.has_lambda = 0 if cfg.lambda_ is None else 1
    o.lambda_ = 0.0 if cfg.lambda_ is None else float(cfg.lambda_)
    o.rho0, o.kappa, o.tol = cfg.rho0, cfg.kappa, cfg.tol
    o.max_iter, o.c = cfg.max_iter, cfg.c
    o.sparse_norm = 1 if str(cfg.sparse_norm).upper() == "L21" else 0
    o.km_max_iters, o.km_n_restarts = cfg.kmeans.max_iters, cfg.kmeans.n_restarts
    o.km_seed, o.km_tol = cfg.kmeans.seed, cfg.kmeans.tol
    o.has_fixed_iters = 0 if cfg.fixed_iters is None else 1
    o.fixed_iters = 0 if cfg.fixed_iters is None else cfg.fixed_iters
    return o


@dataclass
class Result:
    L: np.ndarray
    S: np.ndarray
    labels: np.ndarray
    feas: np.ndarray
    delta_l: np.ndarray
    delta_s: np.ndarray
    objective: np.ndarray
    iters: int
    converged: bool
    lambda_: float
    wall_time: float


def _F(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _dp(a):
    return a.ctypes.data_as(dptr)


def _up(a):
    return a.ctypes.data_as(u64ptr)


class Checker:
    def __init__(self, path: Path, prefix: str):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(str(path))
        self.p = prefix
        self.name = prefix
        self._f("last_error").restype = C.c_char_p

    def _f(self, name):
        return getattr(self.lib, f"{self.p}_{name}")

    def _check(self, rc):
        if rc == 0:
            return
        msg = self._f("last_error")().decode()
        if rc == 1:
            raise ValueError(msg)
        if rc == 2:
            raise RuntimeError(msg)
        raise RuntimeError(f"oracle error {rc}: {msg}")

    # ---- solver --------------------------------------------------------
    def solve(self, x, cfg) -> Result:
        xm = _F(x)
        d, n = xm.shape
        budget = max(1, cfg.fixed_iters if cfg.fixed_iters is not None else cfg.max_iter)
        L = np.empty((d, n), order="F")
        S = np.empty((d, n), order="F")
        lab = np.empty(n, dtype=np.uint64)
        arr = [np.zeros(budget) for _ in range(4)]
        it, conv, lam, wall = C.c_uint64(), C.c_int(), C.c_double(), C.c_double()
        oc = make_config(cfg)
        self._check(self._f("solve")(_dp(xm), u64(d), u64(n), C.byref(oc), _dp(L), _dp(S),
                                     _up(lab), *(_dp(a) for a in arr), C.byref(it),
                                     C.byref(conv), C.byref(lam), C.byref(wall)))
        k = it.value
        return Result(L, S, lab, *(a[:k].copy() for a in arr), k, bool(conv.value), lam.value,
                      wall.value)

    def replay(self, x, cfg, init_labels, n_iters: int):
        """Reference-only loop replay from given labels (bench reference arm)."""
        xm = _F(x)
        d, n = xm.shape
        L = np.empty((d, n), order="F")
        S = np.empty((d, n), order="F")
        lab = np.empty(n, dtype=np.uint64)
        init = np.ascontiguousarray(init_labels, dtype=np.uint64)
        arr = [np.zeros(n_iters) for _ in range(5)]
        oc = make_config(cfg)
        f = self.lib.ref_replay
        self._check(f(_dp(xm), u64(d), u64(n), C.byref(oc), _up(init), u64(n_iters), _dp(L),
                      _dp(S), _up(lab), *(_dp(a) for a in arr)))
        return L, S, lab, arr[:4], arr[4]

    def l_update(self, D, labels, c, lambda_, rho):
        Dm = _F(D)
        lab = np.ascontiguousarray(labels, dtype=np.uint64)
        out = np.empty_like(Dm, order="F")
        self._check(self._f("l_update")(_dp(Dm), u64(Dm.shape[0]), u64(Dm.shape[1]), _up(lab),
                                        u64(c), C.c_double(lambda_), C.c_double(rho), _dp(out)))
        return out

    def s_update_l1(self, B, t):
        Bm = _F(B)
        out = np.empty_like(Bm, order="F")
        self._check(self._f("s_update_l1")(_dp(Bm), u64(Bm.shape[0]), u64(Bm.shape[1]),
                                           C.c_double(t), _dp(out)))
        return out

    def s_update_l21(self, B, t):
        Bm = _F(B)
        out = np.empty_like(Bm, order="F")
        self._check(self._f("s_update_l21")(_dp(Bm), u64(Bm.shape[0]), u64(Bm.shape[1]),
                                            C.c_double(t), _dp(out)))
        return out

    def multiplier_update(self, theta, x, L, S, rho, kappa):
        th = np.array(_F(theta), order="F", copy=True)
        xm, lm, sm = _F(x), _F(L), _F(S)
        r = C.c_double(rho)
        self._check(self._f("multiplier_update")(_dp(th), _dp(xm), _dp(lm), _dp(sm),
                                                 u64(xm.shape[0]), u64(xm.shape[1]),
                                                 C.byref(r), C.c_double(kappa)))
        return th, r.value

    def check_convergence(self, x, lp, l, sp, s, tol):
        ms = [_F(a) for a in (x, lp, l, sp, s)]
        conv = C.c_int()
        f, dl, ds = C.c_double(), C.c_double(), C.c_double()
        self._check(self._f("check_convergence")(*(_dp(a) for a in ms), u64(ms[0].shape[0]),
                                                 u64(ms[0].shape[1]), C.c_double(tol),
                                                 C.byref(conv), C.byref(f), C.byref(dl),
                                                 C.byref(ds)))
        return bool(conv.value), (f.value, dl.value, ds.value)

    # ---- clustering ----------------------------------------------------
    def kmeans(self, m, c, max_iters=100, n_restarts=1, seed=0, tol=1e-6):
        mm = _F(m)
        d, n = mm.shape
        lab = np.empty(n, dtype=np.uint64)
        cen = np.empty((d, max(c, 1)), order="F")
        inert, it = C.c_double(), C.c_uint64()
        self._check(self._f("kmeans")(_dp(mm), u64(d), u64(n), u64(c), u64(max_iters),
                                      u64(n_restarts), u64(seed), C.c_double(tol), _up(lab),
                                      _dp(cen), C.byref(inert), C.byref(it)))
        return lab, cen, inert.value, it.value

    def kmeans_warm(self, m, c, init, max_iters=100, tol=1e-6):
        mm = _F(m)
        d, n = mm.shape
        ini = np.ascontiguousarray(init, dtype=np.uint64)
        lab = np.empty(n, dtype=np.uint64)
        cen = np.empty((d, max(c, 1)), order="F")
        inert, it = C.c_double(), C.c_uint64()
        self._check(self._f("kmeans_warm")(_dp(mm), u64(d), u64(n), u64(c), u64(max_iters),
                                           C.c_double(tol), _up(ini), _up(lab), _dp(cen),
                                           C.byref(inert), C.byref(it)))
        return lab, cen, inert.value, it.value

    def kmeans_pp_init(self, m, c, seed):
        mm = _F(m)
        d, n = mm.shape
        cen = np.empty((d, max(c, 1)), order="F")
        self._check(self._f("kmeans_pp_init")(_dp(mm), u64(d), u64(n), u64(c), u64(seed),
                                              _dp(cen)))
        return cen

    def lloyd_step(self, m, C_):
        mm, cm = _F(m), _F(C_)
        d, n = mm.shape
        lab = np.empty(n, dtype=np.uint64)
        nxt = np.empty_like(cm, order="F")
        self._check(self._f("lloyd_step")(_dp(mm), u64(d), u64(n), _dp(cm), u64(cm.shape[1]),
                                          _up(lab), _dp(nxt)))
        return lab, nxt

    # ---- core ----------------------------------------------------------
    def group_scatter(self, m, labels, c):
        mm = _F(m)
        lab = np.ascontiguousarray(labels, dtype=np.uint64)
        out = C.c_double()
        self._check(self._f("group_scatter")(_dp(mm), u64(mm.shape[0]), u64(mm.shape[1]),
                                             _up(lab), u64(c), C.byref(out)))
        return out.value

    def _scalar(self, nm, m):
        mm = _F(m)
        out = C.c_double()
        self._check(self._f(nm)(_dp(mm), u64(mm.shape[0]), u64(mm.shape[1]), C.byref(out)))
        return out.value

    def frob_norm(self, m):
        return self._scalar("frob_norm", m)

    def elementwise_l1(self, m):
        return self._scalar("elementwise_l1", m)

    def l21_norm(self, m):
        return self._scalar("l21_norm", m)

    def column_l2_norms(self, m):
        mm = _F(m)
        out = np.empty(mm.shape[1])
        self._check(self._f("column_l2_norms")(_dp(mm), u64(mm.shape[0]), u64(mm.shape[1]),
                                               _dp(out)))
        return out

    def column_mean(self, m, cols):
        mm = _F(m)
        cl = np.ascontiguousarray(cols, dtype=np.uint64)
        out = np.empty(mm.shape[0])
        self._check(self._f("column_mean")(_dp(mm), u64(mm.shape[0]), u64(mm.shape[1]), _up(cl),
                                           u64(cl.size), _dp(out)))
        return out

    # ---- RNG (libstdc++ distributions) ---------------------------------
    def uniform_int(self, seed, lo, hi, count):
        out = np.empty(count, dtype=np.uint64)
        self._check(self._f("uniform_int")(u64(seed), u64(lo), u64(hi), u64(count), _up(out)))
        return out

    def uniform_real(self, seed, a, b, count):
        out = np.empty(count)
        self._check(self._f("uniform_real")(u64(seed), C.c_double(a), C.c_double(b), u64(count),
                                            _dp(out)))
        return out


_cache: dict[str, Checker] = {}


def ensure_built() -> None:
    if not (HERE / "liboracle.so").exists():
        subprocess.run(["make", "-s", "-C", str(HERE), "all"], check=True)


def port() -> Checker:
    if "orc" not in _cache:
        ensure_built()
        _cache["orc"] = Checker(HERE / "liboracle.so", "orc")
    return _cache["orc"]


def reference_available() -> bool:
    return (HERE / "_ref" / "librespca_ref.so").exists()


def reference() -> Checker:
    if "ref" not in _cache:
        if not reference_available():
            ensure_built()
        _cache["ref"] = Checker(HERE / "_ref" / "librespca_ref.so", "ref")
    return _cache["ref"]


class RefIO:
    """The unmodified reference's RESPCA1 reader/writer and outlier scores
    (io.cpp:138-164, 296-306) through oracle/ref_io_shim.cpp."""

    def __init__(self, path: Path):
        self.lib = C.CDLL(str(path))
        vp, cp = C.c_void_p, C.c_char_p
        self.lib.ref_write_binary.argtypes = [cp, vp, u64, u64, cp, C.c_size_t]
        self.lib.ref_read_binary.argtypes = [cp, vp, u64, C.POINTER(u64), C.POINTER(u64), cp,
                                             C.c_size_t]
        self.lib.ref_outlier_scores.argtypes = [vp, u64, u64, C.c_double, vp, vp, C.POINTER(u64),
                                                cp, C.c_size_t]

    @staticmethod
    def _raise(rc, err):
        msg = err.value.decode()
        if rc == 1:
            raise OSError(msg)  # io::IoError
        raise ValueError(msg)

    def write_binary(self, path, m):
        a = np.asfortranarray(np.asarray(m, dtype=np.float64))
        err = C.create_string_buffer(512)
        rc = self.lib.ref_write_binary(str(path).encode(), a.ctypes.data, a.shape[0], a.shape[1],
                                       err, 512)
        if rc:
            self._raise(rc, err)

    def read_binary(self, path, cap: int = 1 << 26):
        out = np.empty(cap)
        r, c = u64(), u64()
        err = C.create_string_buffer(512)
        rc = self.lib.ref_read_binary(str(path).encode(), out.ctypes.data, cap, C.byref(r),
                                      C.byref(c), err, 512)
        if rc:
            self._raise(rc, err)
        n = r.value * c.value
        return np.asfortranarray(out[:n].reshape((r.value, c.value), order="F"))

    def synth(self, d, n, c, sparsity=0.05, magnitude=1.0, sigma=0.0, seed=0):
        """io::synth_generate → (x, l0, s0, labels)."""
        f = self.lib.ref_synth
        f.argtypes = [u64, u64, u64, C.c_double, C.c_double, C.c_double, u64, C.c_void_p,
                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_char_p, C.c_size_t]
        x, l0, s0 = (np.empty((d, n), order="F") for _ in range(3))
        lab = np.empty(n, dtype=np.uint64)
        err = C.create_string_buffer(512)
        rc = f(d, n, c, sparsity, magnitude, sigma, seed, x.ctypes.data, l0.ctypes.data,
               s0.ctypes.data, lab.ctypes.data, err, 512)
        if rc:
            self._raise(rc, err)
        return x, l0, s0, lab

    def outlier_scores(self, s, threshold):
        a = np.asfortranarray(np.asarray(s, dtype=np.float64))
        d, n = a.shape
        sc, fl, nf = np.empty(n), np.empty(n, dtype=np.uint64), u64()
        err = C.create_string_buffer(512)
        rc = self.lib.ref_outlier_scores(a.ctypes.data, d, n, C.c_double(threshold), sc.ctypes.data,
                                         fl.ctypes.data, C.byref(nf), err, 512)
        if rc:
            self._raise(rc, err)
        return sc, fl[: nf.value].copy()


def reference_io_available() -> bool:
    return (HERE / "_ref" / "librespca_ref_io.so").exists()


def reference_io() -> RefIO:
    if "refio" not in _cache:
        _cache["refio"] = RefIO(HERE / "_ref" / "librespca_ref_io.so")
    return _cache["refio"]


def lambda_default(d: int, n: int) -> float:
    return math.sqrt(float(max(d, n)))
