"""GPU parity: the CUDA path through the C-ABI against the reference's own
outputs (golden fingerprints) and against the oracle on seeded inputs.

Bar (north_star): fp64 L and S bit-identical (relative Frobenius error 0 ≤ 1e-10),
same iteration count, same labels, same S support; report vectors within
1e-10 relative (they are tree-summed norms; the reference sums one chain).
"""
import numpy as np
import pytest

from helpers import (assert_matches_golden, bitwise, cfg_from, load, make_x, rel_fro,
                     small_cases, unpack_labels)

pytestmark = pytest.mark.gpu


def _solve(ctx, X, cfg, precision="f64"):
    from paper_1904_07497_b200 import respca

    return respca.solve(X, cfg, precision=precision, ctx=ctx)


@pytest.mark.parametrize("case", small_cases(), ids=lambda c: c["case"])
def test_small_solves_bitwise(ctx, case):
    X = make_x(case)
    res = _solve(ctx, X, cfg_from(case["config"]))
    assert_matches_golden(res, case)


@pytest.mark.parametrize("name", ["C1", "C1-default-lambda", "C1-c1"])
def test_c1_bitwise(ctx, name):
    case = load(f"solve_{name}.json")
    X = make_x(case)
    res = _solve(ctx, X, cfg_from(case["config"]))
    assert_matches_golden(res, case)
    assert int(np.count_nonzero(res.S)) == case["ref"]["S_nnz"]


@pytest.mark.parametrize("lanes", ["1", "5"])
def test_c1_bitwise_restart_lanes(ctx, monkeypatch, lanes):
    """solve()'s kmeans(X) with its 5 restarts forced in order (1 lane) or
    side by side (5 lanes): identical to the reference either way."""
    monkeypatch.setenv("RESPCA_KM_LANES", lanes)
    case = load("solve_C1.json")
    res = _solve(ctx, make_x(case), cfg_from(case["config"]))
    assert_matches_golden(res, case)


def test_solve_against_oracle_random(ctx, orc):
    """Fresh seeded inputs, no fixture: GPU vs the C restatement, bitwise."""
    from paper_1904_07497_b200 import synth
    from paper_1904_07497_b200.respca import KMeansConfig, SolverConfig

    rng = np.random.default_rng(5)
    for t in range(6):
        d, n = int(rng.integers(8, 90)), int(rng.integers(10, 140))
        c = int(rng.integers(1, min(9, n)))
        X = synth.rpca(d, n, int(rng.integers(1, 6)), 1.0, 0.07, seed=100 + t)
        lam = None if t % 2 else float(rng.uniform(0.05, 2.0))
        cfg = SolverConfig(lambda_=lam, c=c, tol=1e-6, kmeans=KMeansConfig(seed=t))
        a = _solve(ctx, X, cfg)
        b = orc.solve(X, cfg)
        assert a.report.iters == b.iters
        assert (a.assignment == b.labels).all()
        assert bitwise(a.L, b.L) and bitwise(a.S, b.S)


@pytest.mark.parametrize("d,n,c", [(200, 300, 10), (201, 300, 10), (202, 300, 10), (151, 120, 1), (152, 120, 1)])
def test_fp32_mode_tolerance(ctx, orc, d, n, c):
    """fp32 storage: ≤1e-4 relative Frobenius error of L and S against the
    fp64 reference on the same (f32-rounded) input (d % 4 = 0: the four-row FP32
    walk; d even: two rows per thread; odd d: one; c = 1 with d % 4 = 0: the
    stream kernel on fp32 storage, with odd d the one-row ring)."""
    from paper_1904_07497_b200 import synth
    from paper_1904_07497_b200.respca import SolverConfig

    X = synth.rpca(d, n, 10, 1.0 / np.sqrt(10), 0.1, seed=11).astype(np.float32)
    cfg = SolverConfig(c=c, tol=1e-5)
    a = _solve(ctx, X, cfg, precision="f32")
    b = orc.solve(X.astype(np.float64), cfg)
    assert rel_fro(a.L, b.L) <= 1e-4
    assert rel_fro(a.S, b.S) <= 1e-4
    assert a.L.dtype == np.float32


def test_validation_errors(ctx):
    from paper_1904_07497_b200.respca import SolverConfig

    x = np.random.default_rng(13).uniform(-1, 1, (3, 4))
    with pytest.raises(ValueError, match="c exceeds column count"):
        _solve(ctx, x, SolverConfig(c=5))
    bad = x.copy()
    bad[0, 0] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        _solve(ctx, bad, SolverConfig(c=1))
    with pytest.raises(ValueError, match="all-zero"):
        _solve(ctx, np.zeros((3, 4)), SolverConfig(c=1))
    with pytest.raises(ValueError, match="kappa"):
        _solve(ctx, x, SolverConfig(kappa=0.9))
    for kw, msg in ((dict(rho0=0.0), "rho0"), (dict(tol=0.0), "tol"), (dict(c=0), "c must"),
                    (dict(max_iter=0), "max_iter"), (dict(lambda_=-1.0), "lambda")):
        with pytest.raises(ValueError, match=msg):
            _solve(ctx, x, SolverConfig(**kw))


def test_fixed_iters_semantics(ctx):
    """fixed_iters runs exactly that many iterations, never 'converged'
    (solver.cpp:152, 197; test_solver.cpp:342-352)."""
    from paper_1904_07497_b200.respca import SolverConfig

    x = np.random.default_rng(14).uniform(0, 1, (5, 8))
    res = _solve(ctx, x, SolverConfig(c=2, fixed_iters=7))
    assert res.report.iters == 7 and len(res.report.feas) == 7
    assert not res.report.converged


def test_degenerate_shapes(ctx, orc):
    """1×n, d×1, c = n (singleton groups) — all bitwise against the oracle."""
    from paper_1904_07497_b200.respca import SolverConfig

    rng = np.random.default_rng(15)
    for d, n, c in ((1, 30, 3), (25, 1, 1), (6, 6, 6), (2, 50, 2), (33, 7, 1)):
        X = rng.uniform(-2, 2, (d, n))
        cfg = SolverConfig(c=c, tol=1e-6)
        a = _solve(ctx, X, cfg)
        b = orc.solve(X, cfg)
        assert a.report.iters == b.iters, (d, n, c)
        assert (a.assignment == b.labels).all(), (d, n, c)
        assert bitwise(a.L, b.L) and bitwise(a.S, b.S), (d, n, c)


def test_kernel_launch_accounting(ctx):
    from paper_1904_07497_b200 import synth
    from paper_1904_07497_b200.respca import SolverConfig

    before = ctx.launches()
    X = synth.rpca(64, 64, 3, 1.0, 0.05, seed=1)
    res = _solve(ctx, X, SolverConfig(c=3, tol=1e-6))
    assert ctx.launches() - before >= res.report.iters  # ≥ one kernel per iteration


@pytest.mark.parametrize("seed,d,n,c", [(1, 40, 60, 3), (2, 37, 91, 4), (3, 120, 80, 1), (4, 64, 200, 8)])
def test_l21_solve_bitwise(ctx, orc, seed, d, n, c):
    """sparse_norm = L21 (solver.cpp:90-102, 176-178, 191-193) on the device:
    bit-identical L, S, labels and iteration count vs the oracle."""
    from paper_1904_07497_b200 import synth
    from paper_1904_07497_b200.respca import SolverConfig

    X = synth.rpca(d, n, 3, 1.0, 0.05, seed=seed)
    for lam in (None, 0.3):
        cfg = SolverConfig(c=c, tol=1e-7, sparse_norm="L21", lambda_=lam)
        a = _solve(ctx, X, cfg)
        b = orc.solve(X, cfg)
        assert a.report.iters == b.iters
        assert (a.assignment == b.labels).all()
        assert bitwise(a.L, b.L) and bitwise(a.S, b.S)
        np.testing.assert_allclose(a.report.objective, b.objective, rtol=1e-9)
        np.testing.assert_allclose(a.report.feas, b.feas, rtol=1e-10)


@pytest.mark.parametrize("pdl", ["0", "1"])
def test_c1_bitwise_launch_modes(ctx, monkeypatch, pdl):
    """Programmatic dependent launch on (default) or off for the Pass A chain
    and k_finalize: every dependent kernel waits for its predecessor before
    its first read, so the bits are the reference's either way."""
    monkeypatch.setenv("RESPCA_PDL", pdl)
    for name in ("C1", "C2"):
        case = load(f"solve_{name}.json")
        res = _solve(ctx, make_x(case), cfg_from(case["config"]))
        assert_matches_golden(res, case)


@pytest.mark.parametrize("d,n,c,rb", [(200, 150, 1, "48"), (200, 150, 1, "16"), (96, 120, 4, "16"),
                                      (250, 90, 1, "8"), (64, 300, 3, "32")])
def test_stream_pass_f_bitwise(ctx, orc, monkeypatch, d, n, c, rb):
    """Pass F as row-block streams (k_pass_f_stream) forced with an explicit rows-
    per-stream: a partial last row block (d % rb != 0 — its chunks past d are
    skipped, not computed), several groups (member lists instead of consecutive
    columns) and the smallest block — L, S, labels and iterations as the oracle's."""
    from paper_1904_07497_b200 import synth
    from paper_1904_07497_b200.respca import SolverConfig

    monkeypatch.setenv("RESPCA_PASSF_STREAM", "1")
    monkeypatch.setenv("RESPCA_STREAM_RB", rb)
    X = synth.rpca(d, n, 3, 1.0, 0.08, seed=31 + d + c)
    cfg = SolverConfig(c=c, tol=1e-6)
    a = _solve(ctx, X, cfg)
    b = orc.solve(X, cfg)
    assert a.report.iters == b.iters
    assert (a.assignment == b.labels).all()
    assert bitwise(a.L, b.L) and bitwise(a.S, b.S)
