"""CPU: pin the oracle (the C restatement, oracle/respca_oracle.c) to the
reference — the unmodified reference library compiled from its own sources
(oracle/_ref) where available, and the golden fingerprints the reference
produced (tests/golden/, made by tests/golden/make_golden.py) everywhere.
Also re-checks the reference's own unit-test properties against the oracle
(test_solver.cpp, test_kmeans.cpp, acceptance.cpp criteria 1, 2, 9)."""
import numpy as np
import pytest

from helpers import bitwise, cfg_from, load, make_x, sha, small_cases, unhex, unpack_labels

from oracle import oracle as O

HAVE_REF = O.reference_available()
need_ref = pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built (no /root/reference)")


def _same_result(a, b):
    assert a.iters == b.iters
    assert a.converged == b.converged
    assert (a.labels == b.labels).all()
    assert bitwise(a.L, b.L) and bitwise(a.S, b.S)
    for k in ("feas", "delta_l", "delta_s", "objective"):
        assert bitwise(getattr(a, k), getattr(b, k)), k


# ---------------------------------------------------------------- RNG pins
@need_ref
@pytest.mark.parametrize("seed", [0, 1, 42, 2**63 + 5])
def test_rng_matches_libstdcxx(orc, seed):
    ref = O.reference()
    for lo, hi in ((0, 0), (0, 1), (0, 9), (0, 499), (0, 9999), (7, 2**40), (0, 2**64 - 1)):
        assert (orc.uniform_int(seed, lo, hi, 3000) == ref.uniform_int(seed, lo, hi, 3000)).all()
    for a, b in ((0.0, 1.0), (0.0, 12345.678), (-3.0, 5.0), (0.0, 1e-300)):
        assert bitwise(orc.uniform_real(seed, a, b, 3000), ref.uniform_real(seed, a, b, 3000))


def test_mt19937_64_known_answer(orc):
    # The 10000th output of a default-seeded mt19937_64 is 9981545732273789042
    # (C++11 [rand.predef]); uniform_int over the full range returns raw draws.
    out = orc.uniform_int(5489, 0, 2**64 - 1, 10000)
    assert int(out[-1]) == 9981545732273789042


# ------------------------------------------------------ golden fingerprints
@pytest.mark.parametrize("case", small_cases(), ids=lambda c: c["case"])
def test_oracle_reproduces_small_goldens(orc, case):
    X = make_x(case)
    r = orc.solve(X, cfg_from(case["config"]))
    g = case["ref"]
    assert r.iters == g["iters"] and r.converged == g["converged"]
    assert sha(r.L) == g["L_sha256"] and sha(r.S) == g["S_sha256"]
    assert (r.labels == unpack_labels(g["labels"])).all()
    for k in ("feas", "delta_l", "delta_s", "objective"):
        assert bitwise(getattr(r, k), unhex(g[k])), k


@pytest.mark.parametrize("name", ["C1", "C1-default-lambda", "C1-c1", "C2-c1"])
def test_oracle_reproduces_workload_goldens(orc, name):
    case = load(f"solve_{name}.json")
    if case is None:
        pytest.skip("fixture not generated")
    X = make_x(case)
    r = orc.solve(X, cfg_from(case["config"]))
    g = case["ref"]
    assert r.iters == g["iters"]
    assert sha(r.L) == g["L_sha256"] and sha(r.S) == g["S_sha256"]
    assert (r.labels == unpack_labels(g["labels"])).all()


# ------------------------------------------- port vs compiled reference
@need_ref
def test_port_vs_reference_random_solves(orc):
    from paper_1904_07497_b200 import synth
    from paper_1904_07497_b200.respca import KMeansConfig, SolverConfig

    ref = O.reference()
    rng = np.random.default_rng(0)
    for t in range(12):
        d, n = int(rng.integers(1, 70)), int(rng.integers(2, 120))
        c = int(rng.integers(1, min(10, n) + 1))
        X = synth.rpca(d, n, int(rng.integers(1, 5)), 1.0, 0.06, seed=500 + t)
        cfg = SolverConfig(lambda_=None if t % 3 else float(rng.uniform(0.01, 3)), c=c,
                           tol=float(10.0 ** -rng.integers(3, 9)),
                           fixed_iters=None if t % 4 else int(rng.integers(1, 20)),
                           sparse_norm="L21" if t % 5 == 4 else "L1",
                           kmeans=KMeansConfig(seed=t, n_restarts=int(rng.integers(1, 7))))
        _same_result(orc.solve(X, cfg), ref.solve(X, cfg))


@need_ref
def test_port_vs_reference_stop_edges(orc):
    """The edges tests/test_gpu_stop.py checks the device against: fixed_iters
    = 0 (solver.cpp:152, 157) and tol exactly on / one ulp below the
    reference's own max residual (solver.cpp:197, `<=`)."""
    from paper_1904_07497_b200 import synth
    from paper_1904_07497_b200.respca import SolverConfig

    ref = O.reference()
    X = synth.rpca(40, 60, 3, 1.0, 0.05, seed=21)
    for c in (1, 3):
        a = orc.solve(X, SolverConfig(c=c, fixed_iters=0))
        _same_result(a, ref.solve(X, SolverConfig(c=c, fixed_iters=0)))
        assert a.iters == 0 and bitwise(a.L, X) and not a.S.any()
    X = synth.rpca(60, 80, 3, 1.0, 0.05, seed=3)
    probe = ref.solve(X, SolverConfig(c=4, tol=1e-300, max_iter=30))
    mx = np.maximum(np.maximum(probe.feas, probe.delta_l), probe.delta_s)
    k = next(t for t in range(8, len(mx)) if mx[t] < mx[:t].min())
    for tol, stops_at_k in ((float(mx[k]), True), (float(np.nextafter(mx[k], 0.0)), False)):
        cfg = SolverConfig(c=4, tol=tol, max_iter=30)
        r = ref.solve(X, cfg)
        _same_result(orc.solve(X, cfg), r)
        assert (r.iters == k + 1) == stops_at_k


@need_ref
def test_port_vs_reference_building_blocks(orc):
    ref = O.reference()
    rng = np.random.default_rng(1)
    for t in range(10):
        d, n = int(rng.integers(1, 40)), int(rng.integers(3, 90))
        c = int(rng.integers(1, min(8, n) + 1))
        m = rng.normal(size=(d, n))
        lab = np.concatenate([np.arange(c), rng.integers(0, c, n - c)]).astype(np.uint64)
        rng.shuffle(lab)
        lam, rho = float(rng.uniform(0, 4)), float(rng.uniform(0.01, 3))
        assert bitwise(orc.l_update(m, lab, c, lam, rho), ref.l_update(m, lab, c, lam, rho))
        assert bitwise(orc.s_update_l1(m, 0.3), ref.s_update_l1(m, 0.3))
        assert bitwise(orc.s_update_l21(m, 0.9), ref.s_update_l21(m, 0.9))
        assert orc.group_scatter(m, lab, c) == ref.group_scatter(m, lab, c)
        assert orc.frob_norm(m) == ref.frob_norm(m) and orc.l21_norm(m) == ref.l21_norm(m)
        assert orc.elementwise_l1(m) == ref.elementwise_l1(m)
        assert bitwise(orc.column_l2_norms(m), ref.column_l2_norms(m))
        a = orc.kmeans(m, c, 100, 3, t, 1e-6)
        b = ref.kmeans(m, c, 100, 3, t, 1e-6)
        assert (a[0] == b[0]).all() and bitwise(a[1], b[1]) and a[2] == b[2] and a[3] == b[3]
        assert bitwise(orc.kmeans_pp_init(m, c, t), ref.kmeans_pp_init(m, c, t))
        a = orc.kmeans_warm(m, c, lab)
        b = ref.kmeans_warm(m, c, lab)
        assert (a[0] == b[0]).all() and bitwise(a[1], b[1]) and a[2] == b[2] and a[3] == b[3]
        th, x, L, S = (rng.normal(size=(d, n)) for _ in range(4))
        ta, ra = orc.multiplier_update(th, x, L, S, rho, 1.5)
        tb, rb = ref.multiplier_update(th, x, L, S, rho, 1.5)
        assert bitwise(ta, tb) and ra == rb
        assert orc.check_convergence(x, L, S, th, m, 1e-3) == ref.check_convergence(x, L, S, th, m, 1e-3)


@need_ref
def test_error_messages_match_reference(orc):
    from paper_1904_07497_b200.respca import SolverConfig

    ref = O.reference()
    x = np.random.default_rng(13).uniform(-1, 1, (3, 4))
    cases = [(x, SolverConfig(c=5)), (np.zeros((3, 4)), SolverConfig()),
             (x, SolverConfig(kappa=0.9)), (x, SolverConfig(rho0=-1.0)),
             (x, SolverConfig(tol=0.0)), (x, SolverConfig(max_iter=0)),
             (x, SolverConfig(lambda_=-2.0))]
    bad = x.copy()
    bad[1, 1] = np.inf
    cases.append((bad, SolverConfig()))
    for X, cfg in cases:
        with pytest.raises(ValueError) as ea:
            orc.solve(X, cfg)
        with pytest.raises(ValueError) as eb:
            ref.solve(X, cfg)
        assert str(ea.value) == str(eb.value)


# ------------------------- the reference's own properties, on the oracle
def _dense_l_update(D, labels, c, lam, rho):
    """Explicit per-group solve of P(L)(2λM + ρI) = ρP(D) (test_util.hpp:61-83)."""
    L = np.zeros_like(D)
    for g in range(c):
        idx = np.where(labels == g)[0]
        k = len(idx)
        M = np.eye(k) - np.full((k, k), 1.0 / k)
        A = 2 * lam * M + rho * np.eye(k)
        L[:, idx] = np.linalg.solve(A.T, (rho * D[:, idx]).T).T
    return L


def test_l_update_matches_dense_inverse(orc):
    """acceptance.cpp criterion 1: 200 random instances, group sizes 1..20, 1e-10."""
    rng = np.random.default_rng(100)
    worst = 0.0
    for _ in range(200):
        c = int(rng.integers(1, 5))
        labels = np.concatenate([np.full(int(rng.integers(1, 21)), g) for g in range(c)])
        rng.shuffle(labels)
        D = rng.uniform(-1, 1, (6, labels.size))
        lam, rho = rng.uniform(0.05, 10), rng.uniform(0.01, 5)
        a = orc.l_update(D, labels.astype(np.uint64), c, lam, rho)
        b = _dense_l_update(D, labels, c, lam, rho)
        worst = max(worst, np.linalg.norm(a - b) / np.linalg.norm(b))
    assert worst < 1e-10


def test_prox_operators_grid_oracle(orc):
    """test_solver.cpp:81-96, 131-151 / acceptance criterion 9."""
    rng = np.random.default_rng(900)
    t = 0.37
    grid = np.arange(-2.5, 2.5, 0.005)
    for bij in rng.uniform(-2, 2, 300):
        s = orc.s_update_l1(np.array([[bij]]), t)[0, 0]
        f_opt = t * abs(s) + 0.5 * (s - bij) ** 2
        f = t * np.abs(grid) + 0.5 * (grid - bij) ** 2
        assert f_opt <= f.min() + 1e-8
    b = rng.uniform(0.1, 1.0, (5, 1))
    s = orc.s_update_l21(b, 0.3)
    f_opt = 0.3 * np.linalg.norm(s) + 0.5 * np.sum((s - b) ** 2)
    scales = np.arange(0.0, 1.2, 1e-4)
    f = 0.3 * scales * np.linalg.norm(b) + 0.5 * ((scales - 1.0) ** 2) * np.sum(b * b)
    assert f_opt <= f.min() + 1e-8


def test_scatter_identities(orc):
    """acceptance criterion 2: pairwise and trace-form scatter identities."""
    rng = np.random.default_rng(200)
    for trial in range(40):
        n = 4 + trial % 12
        m = rng.uniform(-1, 1, (5, n))
        lab = np.concatenate([np.arange(2), rng.integers(0, 2, n - 2)]).astype(np.uint64)
        sc = orc.group_scatter(m, lab, 2)
        pair = 0.0
        for g in range(2):
            cols = m[:, lab == g]
            dd = ((cols[:, :, None] - cols[:, None, :]) ** 2).sum()
            pair += dd / (2.0 * cols.shape[1])
        assert abs(pair - sc) <= 1e-10 * max(1.0, sc)


def test_rho_growth_and_cap(orc):
    x = np.random.default_rng(8).uniform(-1, 1, (2, 3))
    th = np.zeros((2, 3))
    rho = 1e-4
    for k in range(1, 41):
        th, rho = orc.multiplier_update(th, x, x, np.zeros((2, 3)), rho, 1.5)
        assert rho == pytest.approx(1e-4 * 1.5 ** k, rel=1e-13)
    _, r = orc.multiplier_update(th, x, x, np.zeros((2, 3)), 9e11, 1.5)
    assert r == 1e12


def test_kmeans_near_optimal_tiny(orc):
    """test_kmeans.cpp:148-166 / acceptance criterion 7."""
    for seed in range(10):
        m = np.random.default_rng(seed + 700).uniform(-1, 1, (3, 10 + seed % 3))
        n = m.shape[1]
        best = np.inf
        for mask in range(1, (1 << n) - 1):
            lab = np.array([(mask >> j) & 1 for j in range(n)], dtype=np.uint64)
            best = min(best, orc.group_scatter(m, lab, 2))
        _, _, inertia, _ = orc.kmeans(m, 2, 100, 5, seed, 1e-6)
        assert inertia <= best * 1.05 + 1e-12
