"""§8(f): solve() between RESPCA1 files streamed disk → HBM → disk, and
io::outlier_scores on the device — against the reference's own outputs."""
import numpy as np
import pytest

from helpers import cfg_from, load, make_x, sha, unpack_labels
from oracle import oracle as O
from paper_1904_07497_b200 import _native as N
from paper_1904_07497_b200 import respca

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_solve_file_bitwise(ctx, tmp_path, name):
    case = load(f"solve_{name}.json")
    X = make_x(case)
    xp, lp, sp = tmp_path / "x.bin", tmp_path / "l.bin", tmp_path / "s.bin"
    respca.write_binary_matrix(xp, X)
    res = respca.solve_file(xp, cfg_from(case["config"]), lp, sp, ctx=ctx)
    g = case["ref"]
    assert res.report.iters == g["iters"]
    assert (res.assignment == unpack_labels(g["labels"])).all()
    L, S = respca.read_binary_matrix(lp), respca.read_binary_matrix(sp)
    assert sha(L) == g["L_sha256"] and sha(S) == g["S_sha256"]


def test_solve_file_matches_in_memory_fp32(ctx, tmp_path):
    from paper_1904_07497_b200 import synth
    from paper_1904_07497_b200.respca import SolverConfig

    X = synth.rpca(300, 500, 10, 1.0, 0.05, seed=4)
    xp, lp = tmp_path / "x.bin", tmp_path / "l.bin"
    respca.write_binary_matrix(xp, X)
    cfg = SolverConfig(c=5, tol=1e-6)
    a = respca.solve_file(xp, cfg, lp, None, precision="f32", ctx=ctx)
    b = respca.solve(X.astype(np.float32), cfg, precision="f32", ctx=ctx)
    assert a.report.iters == b.report.iters
    assert np.array_equal(respca.read_binary_matrix(lp), b.L.astype(np.float64))


def test_solve_file_errors(ctx, tmp_path):
    with pytest.raises(N.IoError, match="cannot open"):
        respca.solve_file(tmp_path / "missing.bin", ctx=ctx)
    p = tmp_path / "bad.bin"
    p.write_bytes(b"NOTRESPC" + bytes(16))
    with pytest.raises(N.IoError, match="bad magic"):
        respca.solve_file(p, ctx=ctx)


@pytest.mark.skipif(not O.reference_io_available(), reason="reference I/O not built")
def test_outlier_scores_match_reference(ctx):
    ref = O.reference_io()
    rng = np.random.default_rng(9)
    S = np.where(rng.uniform(size=(200, 300)) < 0.02, rng.uniform(-50, 50, (200, 300)), 0.0)
    for thr in (0.0, 10.0, 60.0):
        a = respca.outlier_scores(S, thr, ctx=ctx)
        sc, fl = ref.outlier_scores(S, thr)
        assert np.array_equal(a.scores.view(np.uint64), sc.view(np.uint64))
        assert np.array_equal(a.flagged, fl)
    with pytest.raises(ValueError, match="negative threshold"):
        respca.outlier_scores(S, -1.0, ctx=ctx)
