"""GPU building blocks (solver.hpp:67-84, kmeans.hpp:28-43, matrix.hpp:82-98)
against the oracle, bitwise where the reference's op order is reproduced,
plus the reference's own unit-test properties (test_solver.cpp,
test_kmeans.cpp)."""
import numpy as np
import pytest

from helpers import bitwise

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    from paper_1904_07497_b200 import respca

    return respca


def rand(rng, d, n, lo=-1.0, hi=1.0):
    return rng.uniform(lo, hi, (d, n))


def rand_labels(rng, n, c):
    lab = np.concatenate([np.arange(c), rng.integers(0, c, n - c)])
    rng.shuffle(lab)
    return lab.astype(np.uint64)


def test_l_update_bitwise(ctx, orc, R):
    rng = np.random.default_rng(1)
    for d, n, c in ((5, 9, 2), (40, 100, 7), (37, 61, 3), (256, 300, 12), (1, 20, 4)):
        D = rand(rng, d, n)
        lab = rand_labels(rng, n, c)
        lam, rho = float(rng.uniform(0.05, 10)), float(rng.uniform(0.01, 5))
        assert bitwise(R.l_update(D, lab, c, lam, rho, ctx=ctx), orc.l_update(D, lab, c, lam, rho))


def test_l_update_limits_and_errors(ctx, R):
    rng = np.random.default_rng(2)
    D = rand(rng, 4, 7)
    lab = rand_labels(rng, 7, 2)
    np.testing.assert_allclose(R.l_update(D, lab, 2, 0.0, 0.7, ctx=ctx), D, rtol=1e-14)
    L = R.l_update(D, lab, 2, 1.0, 1e12, ctx=ctx)
    assert np.linalg.norm(L - D) / np.linalg.norm(D) < 1e-9
    for rho in (0.0, -1.0):
        with pytest.raises(ValueError, match="rho must be > 0"):
            R.l_update(D, lab, 2, 1.0, rho, ctx=ctx)
    with pytest.raises(ValueError, match="empty group"):
        R.l_update(D, np.zeros(7, dtype=np.uint64), 2, 1.0, 1.0, ctx=ctx)


def test_s_update_bitwise_and_cases(ctx, orc, R):
    rng = np.random.default_rng(3)
    B = rand(rng, 33, 47, -3, 3)
    for t in (0.0, 0.37, 1.2):
        assert bitwise(R.s_update_l1(B, t, ctx=ctx), orc.s_update_l1(B, t))
        assert bitwise(R.s_update_l21(B, 3 * t, ctx=ctx), orc.s_update_l21(B, 3 * t))
    s = R.s_update_l1(np.array([[2.0, -0.3]]), 0.5, ctx=ctx)
    assert s[0, 0] == 1.5 and s[0, 1] == 0.0
    with pytest.raises(ValueError, match="negative threshold"):
        R.s_update_l1(B, -0.1, ctx=ctx)
    b = np.array([[3.0, 0.1], [4.0, 0.1]])
    assert np.linalg.norm(R.s_update_l21(b, 10.0, ctx=ctx)) == 0.0
    s = R.s_update_l21(b, 1.0, ctx=ctx)
    np.testing.assert_allclose(s[:, 0], [2.4, 3.2])
    with pytest.raises(ValueError, match="negative threshold"):
        R.s_update_l21(B, -1.0, ctx=ctx)


def test_multiplier_update(ctx, orc, R):
    rng = np.random.default_rng(7)
    x, L, S, th = (rand(rng, 13, 17) for _ in range(4))
    a, ra = R.multiplier_update(th, x, L, S, 1e-4, 1.5, ctx=ctx)
    b, rb = orc.multiplier_update(th, x, L, S, 1e-4, 1.5)
    assert bitwise(a, b) and ra == rb
    rho = 1e-4
    for k in range(1, 41):  # exact geometric growth, test_solver.cpp:185-197
        _, rho = R.multiplier_update(th, x, L, S, rho, 1.5, ctx=ctx)
        assert rho == pytest.approx(1e-4 * 1.5 ** k, rel=1e-13)
    _, r = R.multiplier_update(th, x, L, S, 9e11, 1.5, ctx=ctx)
    assert r == 1e12  # kRhoCap
    with pytest.raises(ValueError, match="kappa"):
        R.multiplier_update(th, x, L, S, 1.0, 1.0, ctx=ctx)


def test_check_convergence(ctx, orc, R):
    rng = np.random.default_rng(9)
    x = rand(rng, 3, 4)
    s = np.zeros((3, 4))
    ok, r = R.check_convergence(x, x, x, s, s, 1e-3, ctx=ctx)
    assert ok and r == (0.0, 0.0, 0.0)
    ms = [rand(rng, 30, 40) for _ in range(5)]
    a = R.check_convergence(*ms, 1e-3, ctx=ctx)
    b = orc.check_convergence(*ms, 1e-3)
    assert a[0] == b[0]
    np.testing.assert_allclose(a[1], b[1], rtol=1e-12)
    with pytest.raises(ValueError, match="all-zero"):
        z = np.zeros((3, 4))
        R.check_convergence(z, z, z, z, z, 1e-3, ctx=ctx)


def test_kmeans_pp_init_bitwise(ctx, orc, R):
    rng = np.random.default_rng(11)
    for d, n, c, seed in ((3, 6, 6, 1), (4, 20, 2, 5), (30, 200, 9, 42), (7, 50, 1, 3)):
        m = rand(rng, d, n)
        assert bitwise(R.kmeans_pp_init(m, c, seed, ctx=ctx), orc.kmeans_pp_init(m, c, seed))
    with pytest.raises(ValueError, match="exceeds column count"):
        R.kmeans_pp_init(rand(rng, 3, 6), 7, 0, ctx=ctx)


def test_lloyd_step_bitwise(ctx, orc, R):
    rng = np.random.default_rng(12)
    lab, nxt = R.lloyd_step(np.array([[0.0, 1.0, 10.0, 11.0]]), np.array([[0.5, 10.5]]), ctx=ctx)
    assert list(lab) == [0, 0, 1, 1] and nxt[0, 0] == 0.5 and nxt[0, 1] == 10.5
    for d, n, c in ((3, 30, 3), (25, 120, 8), (60, 300, 20)):
        m = rand(rng, d, n)
        C0 = orc.kmeans_pp_init(m, c, 3)
        a = R.lloyd_step(m, C0, ctx=ctx)
        b = orc.lloyd_step(m, C0)
        assert (a[0] == b[0]).all() and bitwise(a[1], b[1])


def test_lloyd_step_repairs_empty_cluster(ctx, orc, R):
    """A far-away centroid gets no points → repair_empty steals the farthest
    point (kmeans.cpp:40-64)."""
    rng = np.random.default_rng(13)
    m = rand(rng, 4, 40)
    C0 = np.concatenate([m[:, :3], np.full((4, 2), 1e3)], axis=1)
    a = R.lloyd_step(m, C0, ctx=ctx)
    b = orc.lloyd_step(m, C0)
    assert (a[0] == b[0]).all() and bitwise(a[1], b[1])


def test_repair_impossible_raises(ctx, R):
    m = np.zeros((2, 3))
    m[:, 1] = 1.0
    C0 = np.array([[0.0, 50.0, 60.0, 70.0], [0.0, 50.0, 60.0, 70.0]])
    # 3 columns, 4 centroids cannot all be non-empty; kmeans.cpp:58
    with pytest.raises((RuntimeError, ValueError)):
        R.lloyd_step(m, C0, ctx=ctx)


def test_kmeans_bitwise(ctx, orc, R):
    from paper_1904_07497_b200.respca import KMeansConfig

    rng = np.random.default_rng(14)
    for d, n, c, seed, restarts in ((3, 15, 4, 0, 1), (4, 24, 2, 3, 5), (20, 200, 6, 7, 5),
                                    (50, 400, 16, 1, 2), (2, 10, 2, 9, 5)):
        m = rand(rng, d, n)
        a = R.kmeans(m, KMeansConfig(c=c, seed=seed, n_restarts=restarts), ctx=ctx)
        lab, cen, inertia, it = orc.kmeans(m, c, 100, restarts, seed, 1e-6)
        assert (a.assignment == lab).all()
        assert bitwise(a.centroids, cen)
        assert a.inertia == inertia and a.iters_run == it
    with pytest.raises(ValueError):
        R.kmeans(rand(rng, 2, 5), KMeansConfig(c=6), ctx=ctx)
    with pytest.raises(ValueError):
        R.kmeans(rand(rng, 2, 5), KMeansConfig(c=0), ctx=ctx)


@pytest.mark.parametrize("lanes", ["2", "3", "5"])
def test_kmeans_restart_lanes_bitwise(ctx, orc, R, monkeypatch, lanes):
    """Restarts run side by side (one stream + host thread per lane, seeding
    in turn): same winner, labels, centroids, inertia as the reference's
    sequential loop (kmeans.cpp:237-250)."""
    from paper_1904_07497_b200.respca import KMeansConfig

    monkeypatch.setenv("RESPCA_KM_LANES", lanes)
    rng = np.random.default_rng(24)
    for d, n, c, seed, restarts in ((4, 24, 2, 3, 5), (20, 200, 6, 7, 5), (64, 300, 12, 2, 7),
                                    (2, 10, 2, 9, 4)):
        m = rand(rng, d, n)
        a = R.kmeans(m, KMeansConfig(c=c, seed=seed, n_restarts=restarts), ctx=ctx)
        lab, cen, inertia, it = orc.kmeans(m, c, 100, restarts, seed, 1e-6)
        assert (a.assignment == lab).all()
        assert bitwise(a.centroids, cen)
        assert a.inertia == inertia and a.iters_run == it
    # duplicate columns: a seeding runs out of positive d² mass and skips its
    # draws, so the next restarts' speculated engine states are wrong and are
    # redone from the true ones
    base = np.random.default_rng(3).uniform(-1, 1, (6, 3))
    m = np.asfortranarray(np.array([base[:, i % 3] for i in range(30)]).T)
    m[:, 5] += 1e-3
    a = R.kmeans(m, KMeansConfig(c=5, seed=11, n_restarts=5), ctx=ctx)
    lab, cen, inertia, it = orc.kmeans(m, 5, 100, 5, 11, 1e-6)
    assert (a.assignment == lab).all() and bitwise(a.centroids, cen)
    assert a.inertia == inertia and a.iters_run == it


def test_kmeans_warm_bitwise(ctx, orc, R):
    from paper_1904_07497_b200.respca import KMeansConfig

    rng = np.random.default_rng(15)
    for d, n, c in ((3, 16, 2), (10, 80, 5), (40, 250, 12)):
        m = rand(rng, d, n)
        init = (np.arange(n) % c).astype(np.uint64)
        a = R.kmeans_warm(m, KMeansConfig(c=c), init, ctx=ctx)
        lab, cen, inertia, it = orc.kmeans_warm(m, c, init)
        assert (a.assignment == lab).all() and bitwise(a.centroids, cen)
        assert a.inertia == inertia and a.iters_run == it


def test_core_norms(ctx, orc, R):
    rng = np.random.default_rng(16)
    m = rand(rng, 37, 53)
    np.testing.assert_allclose(R.frob_norm(m, ctx=ctx), orc.frob_norm(m), rtol=1e-13)
    np.testing.assert_allclose(R.elementwise_l1(m, ctx=ctx), orc.elementwise_l1(m), rtol=1e-13)
    assert bitwise(R.column_l2_norms(m, ctx=ctx), orc.column_l2_norms(m))  # exact chains
    assert R.l21_norm(m, ctx=ctx) == orc.l21_norm(m)
    cols = np.array([5, 2, 9, 2], dtype=np.uint64)
    assert bitwise(R.column_mean(m, cols, ctx=ctx), orc.column_mean(m, cols))
    lab = rand_labels(rng, 53, 4)
    np.testing.assert_allclose(R.group_scatter(m, lab, 4, ctx=ctx), orc.group_scatter(m, lab, 4),
                               rtol=1e-12)
    with pytest.raises(ValueError, match="empty column set"):
        R.column_mean(m, np.array([], dtype=np.uint64), ctx=ctx)


def test_screen_bound_is_rigorous(ctx, orc):
    """The screened distance interval always contains the reference's exact
    sequential sq_dist (kmeans.cpp:12-19), across shapes, scales and dtypes of
    the split-K DMMA kernel; decisions are only ever taken inside it."""
    import ctypes as C

    from paper_1904_07497_b200 import _native as N

    rng = np.random.default_rng(21)
    for d, n, c, scale in ((3, 40, 5, 1.0), (37, 130, 9, 1e3), (1000, 300, 50, 1e-3),
                           (4096, 200, 64, 50.0), (333, 257, 17, 1.0), (64, 500, 100, 1.0)):
        m = np.asfortranarray(rng.normal(0, scale, (d, n)))
        Cm = np.asfortranarray(m[:, rng.choice(n, c, replace=False)] + rng.normal(0, scale * 1e-3, (d, c)))
        a = np.empty(n * c)
        e = np.empty(n * c)
        N.check(ctx, N.lib().respca_cu_debug_screen(ctx.handle, m.ctypes.data_as(N.dptr), d, n,
                                                    Cm.ctypes.data_as(N.dptr), c,
                                                    a.ctypes.data_as(N.dptr),
                                                    e.ctypes.data_as(N.dptr)))
        a, e = a.reshape(n, c), e.reshape(n, c)
        # exact sequential chains, the reference's order (numpy cumsum is sequential)
        diff = m[:, :, None] - Cm[:, None, :]
        exact = np.cumsum(diff * diff, axis=0)[-1]
        assert (np.abs(exact - a) <= e).all(), (d, n, c, float(np.max(np.abs(exact - a) / e)))
        assert (e <= 1e-9 * (np.abs(exact) + scale * scale * d)).all()


def test_tc_screen_bound_is_rigorous(ctx):
    """The tcgen05 BF16 screen (ALM fast path): its interval always contains the
    reference's exact sequential sq_dist."""
    from paper_1904_07497_b200 import _native as N

    rng = np.random.default_rng(22)
    for d, n, c, scale in ((3, 40, 5, 1.0), (130, 300, 50, 1e2), (1000, 257, 64, 1e-3),
                           (4096, 200, 17, 5.0), (64, 129, 1, 1.0), (10000, 160, 50, 0.14)):
        m = np.asfortranarray(rng.normal(0, scale, (d, n)))
        Cm = np.asfortranarray(m[:, rng.choice(n, c, replace=False)] * 0.5 +
                               rng.normal(0, scale, (d, c)))
        a = np.empty(n * c)
        e = np.empty(n * c)
        N.check(ctx, N.lib().respca_cu_debug_screen_tc(ctx.handle, m.ctypes.data_as(N.dptr), d, n,
                                                       Cm.ctypes.data_as(N.dptr), c,
                                                       a.ctypes.data_as(N.dptr),
                                                       e.ctypes.data_as(N.dptr)))
        a, e = a.reshape(n, c), e.reshape(n, c)
        diff = m[:, :, None] - Cm[:, None, :]
        exact = np.cumsum(diff * diff, axis=0)[-1]
        err = np.abs(exact - a)
        assert (err <= e).all(), (d, n, c, float(np.max(err / e)))
        # the screen is informative: its error is far below the distances
        assert np.median(err / np.maximum(exact, 1e-300)) < 1e-2
