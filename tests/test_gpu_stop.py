"""The ALM stopping rule decided exactly as the reference decides it
(solver.cpp:197 on the sequential chains of solver.cpp:14-31 and
matrix.cpp:99-103), and the fixed_iters = 0 edge (solver.cpp:152, 157).

The device sums the residuals in a fixed-order tree; k_finalize decides on a
rigorous interval around the reference's chain value and sends the iteration
to Alm::resolve_stop (replay + k_exact_chains) when tol falls inside it.
These tests put tol exactly on (and one ulp below) the reference's own
residual value, where only the chains can decide, and force every stop test
through the chains on C1 and C2.
"""
import os

import numpy as np
import pytest

from helpers import assert_matches_golden, bitwise, cfg_from, load, make_x, unhex

pytestmark = pytest.mark.gpu


def _solve(ctx, X, cfg):
    from paper_1904_07497_b200 import respca

    return respca.solve(X, cfg, ctx=ctx)


@pytest.mark.parametrize("c", [1, 3])
def test_fixed_iters_zero(ctx, orc, c):
    """Zero iterations: L = X, S = 0, an empty report, iters = 0, not
    converged, labels = the initial kmeans(X) — bitwise against the oracle."""
    from paper_1904_07497_b200 import synth
    from paper_1904_07497_b200.respca import SolverConfig

    X = synth.rpca(40, 60, 3, 1.0, 0.05, seed=21)
    cfg = SolverConfig(c=c, fixed_iters=0)
    a = _solve(ctx, X, cfg)
    b = orc.solve(X, cfg)
    assert b.iters == 0 and a.report.iters == 0
    assert not a.report.converged and not b.converged
    assert len(a.report.feas) == 0 and len(a.report.objective) == 0
    assert bitwise(a.L, X) and bitwise(a.S, np.zeros_like(X))
    assert bitwise(a.L, b.L) and bitwise(a.S, b.S)
    assert (a.assignment == b.labels).all()
    # the context is reusable afterwards (no stale loop state)
    a2 = _solve(ctx, X, SolverConfig(c=c, fixed_iters=2))
    b2 = orc.solve(X, SolverConfig(c=c, fixed_iters=2))
    assert a2.report.iters == 2 and bitwise(a2.L, b2.L) and bitwise(a2.S, b2.S)


@pytest.mark.parametrize("name", ["C1", "C1-c1", "C2"])
def test_force_exact_stop_bitwise(ctx, monkeypatch, name):
    """RESPCA_ALM_STOP_FORCE_EXACT=1: every stop test goes through the replay
    and the reference-order chains — same bits, same iteration count, and the
    residual report equals the reference's own chain values bit for bit."""
    case = load(f"solve_{name}.json")
    monkeypatch.setenv("RESPCA_ALM_STOP_FORCE_EXACT", "1")
    from paper_1904_07497_b200 import _native as N

    fresh = N.Context(0)  # the switch is read when a solver is created
    res = _solve(fresh, make_x(case), cfg_from(case["config"]))
    assert_matches_golden(res, case)
    assert res.stop_resolves == res.report.iters
    g = case["ref"]
    for key, mine in (("feas", res.report.feas), ("delta_l", res.report.delta_l),
                      ("delta_s", res.report.delta_s)):
        assert bitwise(mine, unhex(g[key])), key


def _near_tol_cases():
    # (d, n, rank, sparse fraction, c, seed)
    return [(60, 80, 3, 0.05, 4, 3), (64, 90, 2, 0.08, 1, 8), (33, 47, 2, 0.1, 5, 12)]


@pytest.mark.parametrize("shape", _near_tol_cases(), ids=lambda s: "x".join(map(str, s[:2])) + f"c{s[4]}")
def test_stop_exactly_at_tol(ctx, orc, shape):
    """tol placed exactly on the reference's max residual of an iteration k
    (stop margin 0) and one ulp below it (margin 1 ulp ≈ 1e-16 relative): the
    iteration count, L, S and labels match the oracle (the restated
    reference) in both cases, and the undecidable test went to the chains."""
    from paper_1904_07497_b200 import synth
    from paper_1904_07497_b200.respca import SolverConfig

    d, n, r, p, c, seed = shape
    X = synth.rpca(d, n, r, 1.0, p, seed=seed)
    probe = orc.solve(X, SolverConfig(c=c, tol=1e-300, max_iter=60))
    mx = np.maximum(np.maximum(probe.feas, probe.delta_l), probe.delta_s)
    # an iteration whose max is a new running minimum (so the run reaches it)
    k = None
    for t in range(8, len(mx)):
        if mx[t] < mx[:t].min():
            k = t
            break
    assert k is not None
    for tol in (float(mx[k]), float(np.nextafter(mx[k], 0.0))):
        cfg = SolverConfig(c=c, tol=tol, max_iter=60)
        b = orc.solve(X, cfg)
        a = _solve(ctx, X, cfg)
        assert a.report.iters == b.iters, (tol, a.report.iters, b.iters)
        assert a.report.converged == b.converged
        assert (a.assignment == b.labels).all()
        assert bitwise(a.L, b.L) and bitwise(a.S, b.S)
        assert a.stop_resolves >= 1
        if tol == mx[k]:
            assert a.report.iters == k + 1 and a.report.converged
        # the resolved row k carries the reference's own chain values
        assert bitwise(a.report.feas[k], b.feas[k])
        assert bitwise(a.report.delta_l[k], b.delta_l[k])
        assert bitwise(a.report.delta_s[k], b.delta_s[k])


def test_stop_guard_is_quiet_on_c1(ctx):
    """Without the switch the interval test decides every C1 iteration itself
    (no replay) and still matches the reference."""
    assert os.environ.get("RESPCA_ALM_STOP_FORCE_EXACT") in (None, "", "0")
    case = load("solve_C1.json")
    res = _solve(ctx, make_x(case), cfg_from(case["config"]))
    assert_matches_golden(res, case)
    assert res.stop_resolves == 0


def test_screen_error_flag_routes_to_exact(ctx, monkeypatch):
    """A tcgen05 screen whose mbarrier wait failed (simulated with
    RESPCA_TC_FORCE_ERR=1) must not be trusted: every Pass A decision then
    comes from the exact chains and the solve is still bit-identical."""
    case = load("solve_C1.json")
    monkeypatch.setenv("RESPCA_TC_FORCE_ERR", "1")
    from paper_1904_07497_b200 import _native as N

    fresh = N.Context(0)
    X = make_x(case)
    res = _solve(fresh, X, cfg_from(case["config"]))
    assert_matches_golden(res, case)
    # every column of every fast-path iteration went to the chains
    assert res.exact_fallbacks >= (res.report.iters - 1) * X.shape[1]


def test_tiny_magnitudes_bitwise(ctx, orc):
    """Entries around 1e-30..1e-25: BF16/FP32 screen operands and products sit
    at or below the FP32 normal range (subnormal or flushed); the screens'
    absolute terms keep the intervals rigorous — bitwise against the oracle."""
    from paper_1904_07497_b200 import synth
    from paper_1904_07497_b200.respca import SolverConfig

    for scale in (1e-25, 1e-30):
        X = synth.rpca(96, 160, 3, 1.0, 0.05, seed=31) * scale
        cfg = SolverConfig(c=6, tol=1e-6, lambda_=0.5)
        a = _solve(ctx, X, cfg)
        b = orc.solve(X, cfg)
        assert a.report.iters == b.iters
        assert (a.assignment == b.labels).all()
        assert bitwise(a.L, b.L) and bitwise(a.S, b.S)


def _replay_support_margin(orc, X, c, lam, iters, tol=None):
    """The reference loop replayed with the oracle's building blocks
    (solver.cpp:157-201), returning min over iterations and entries of
    ||B| − 1/ρ|·ρ and the per-iteration max residuals."""
    d, n = X.shape
    labels = orc.kmeans(X, c, 100, 5, 0, 1e-6)[0]
    L = X.copy(order="F")
    S = np.zeros_like(X, order="F")
    Th = np.zeros_like(X, order="F")
    rho, best = 1e-4, np.inf
    for _ in range(iters):
        D = (X - S) + Th / rho
        L = orc.l_update(D, labels, c, lam, rho)
        labels = orc.kmeans_warm(L, c, labels)[0]
        B = (X - L) + Th / rho
        t = 1.0 / rho
        best = min(best, float(np.min(np.abs(np.abs(B) - t))) / t)
        S = orc.s_update_l1(B, t)
        Th, rho = orc.multiplier_update(Th, X, L, S, rho, 1.5)
    return best


def test_decision_margins(ctx, orc):
    """respca_cu_last_margins: the S-support margin equals
    the one a replay of the reference loop with the oracle's own building
    blocks measures, bit for bit; the ALM-stop margin is |max(report)/tol − 1|;
    the initial-clustering margins are reported."""
    from paper_1904_07497_b200 import synth
    from paper_1904_07497_b200.respca import SolverConfig

    X = synth.rpca(48, 72, 3, 1.0, 0.06, seed=9)
    lam = 0.7
    res = _solve(ctx, X, SolverConfig(c=4, lambda_=lam, fixed_iters=12))
    m = res.margins
    ref = _replay_support_margin(orc, X, 4, lam, 12)
    assert m["s_support"] == ref, (m["s_support"], ref)
    assert m["alm_stop"] == np.inf  # fixed_iters: no stop test
    assert 0.0 <= m["restart_gap"] < np.inf and 0.0 < m["lloyd_stop"] < np.inf
    case = load("solve_C1.json")
    res = _solve(ctx, make_x(case), cfg_from(case["config"]))
    m = res.margins
    mx = max(res.report.feas[-1], res.report.delta_l[-1], res.report.delta_s[-1])
    assert m["alm_stop_final"] == abs(mx / case["config"]["tol"] - 1.0)
    assert 1e-9 < m["alm_stop"] <= m["alm_stop_final"]
    assert 0.0 < m["s_support"] < 1.0 and m["stop_resolves"] == 0
    print("\nC1 margins:", m)
