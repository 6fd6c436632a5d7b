"""GPU parity at BASELINE.json scale against the reference's own outputs.

fp64 workloads (C2 c=100, C2 c=1, C3 c=50, C3 c=1): L, S, labels and the
iteration count bit-identical to the unmodified reference (golden SHA-256
fingerprints made by tests/golden/make_golden.py; the reference took 128 s,
9 s, 2,277 s and 277 s on one core).  fp32 workloads (C3-f32, C4): their
input solved in fp64 is bit-identical to the reference's fp64 solve of it
(2,159 s and 234 s on one core), and the fp32-storage solve is within 1e-4
relative Frobenius error of that (the true error) with the S-support mismatch
counted.  C5 (d=n=40,000, 12.8 GB per matrix, c=1): the resident solve, pinned
bitwise by reference solves of row slices (c=1 rows are independent).
"""
import numpy as np
import pytest

from helpers import bitwise, cfg_from, load, make_x, rel_fro, sha, unhex, unpack_labels

pytestmark = pytest.mark.gpu


def _solve(ctx, X, cfg, precision="f64"):
    from paper_1904_07497_b200 import respca

    return respca.solve(X, cfg, precision=precision, ctx=ctx)


@pytest.mark.parametrize("name", ["C2", "C2-c1", "C3", "C3-c1"])
def test_workload_bitwise(ctx, name):
    case = load(f"solve_{name}.json")
    assert case is not None, f"golden fixture solve_{name}.json missing"
    X = make_x(case)
    res = _solve(ctx, X, cfg_from(case["config"]))
    g = case["ref"]
    assert res.report.iters == g["iters"]
    assert res.report.converged == g["converged"]
    assert (res.assignment == unpack_labels(g["labels"])).all()
    assert sha(res.L) == g["L_sha256"], "L not bit-identical to the reference"
    assert sha(res.S) == g["S_sha256"], "S not bit-identical to the reference"
    assert int(np.count_nonzero(res.S)) == g["S_nnz"]
    np.testing.assert_allclose(res.report.feas, unhex(g["feas"]), rtol=1e-10)


@pytest.mark.parametrize("name", ["C3-f32", "C4"])
def test_fp32_workload_true_error(ctx, name):
    """The fp32-storage workloads, judged as north_star states it.

    1. Their (f32-rounded) input solved in fp64 is bit-identical to the
       reference's own fp64 solve of it (tests/golden/solve_{name}.json: 37 and
       43 iterations; C4 runs the tight-cluster FP64 DMMA screen at d = 76,800).
    2. The fp32-storage solve of the same input is within 1e-4 relative
       Frobenius error of that fp64 solve for L and S (the true error, not a
       sketch), with the S-support mismatch count reported and bounded."""
    from paper_1904_07497_b200 import synth

    case = load(f"solve_{name}.json")
    w = synth.WORKLOADS[name]
    X64 = make_x(case)  # f32-rounded values in fp64
    g = case["ref"]
    r64 = _solve(ctx, X64, cfg_from(case["config"]))
    assert r64.report.iters == g["iters"] and r64.report.converged == g["converged"]
    assert (r64.assignment == unpack_labels(g["labels"])).all()
    assert sha(r64.L) == g["L_sha256"], "fp64 L not bit-identical to the reference"
    assert sha(r64.S) == g["S_sha256"], "fp64 S not bit-identical to the reference"
    assert int(np.count_nonzero(r64.S)) == g["S_nnz"]
    X32 = np.asfortranarray(X64.astype(np.float32))
    del X64
    r32 = _solve(ctx, X32, w.solver_config(), precision="f32")
    assert r32.L.dtype == np.float32
    eL = rel_fro(r32.L, r64.L)
    eS = rel_fro(r32.S, r64.S)
    nz32, nz64 = r32.S != 0, r64.S != 0
    mismatch = int(np.count_nonzero(nz32 != nz64))
    print(f"\n[{name}] fp32 vs fp64 (= reference): rel Frobenius L {eL:.3e}, S {eS:.3e}; "
          f"S support mismatch {mismatch} of {int(nz64.sum())} nonzeros "
          f"(iters fp32 {r32.report.iters}, fp64 {r64.report.iters})")
    assert eL <= 1e-4, eL
    assert eS <= 1e-4, eS
    # fp32 storage flips entries whose |B| sits within float rounding of 1/ρ
    assert mismatch <= 1e-3 * max(1, int(nz64.sum())), mismatch


def test_c5_resident_solve(ctx, orc):
    """C5: 40,000² fp64, rank 20, 5 % corruption, tol 1e-6, c = 1 — X, L, S, Θ
    (51.2 GB) resident in HBM for the whole solve — and pinned bitwise by row
    slices: with one group every row evolves independently for a given
    iteration count (l_update sums per row, solver.cpp:51-77; everything else
    is elementwise; ρ depends only on t), so the reference solving a slice of
    rows with λ passed explicitly (solver.cpp:35-38) and fixed_iters = the
    device's count must reproduce exactly those rows of L and S."""
    from oracle import oracle as O
    from paper_1904_07497_b200 import synth
    from paper_1904_07497_b200.respca import SolverConfig

    w = synth.WORKLOADS["C5"]
    X = w.make()
    res = _solve(ctx, X, w.solver_config())
    assert res.report.converged
    assert 30 <= res.report.iters <= 80
    assert max(res.report.feas[-1], res.report.delta_l[-1], res.report.delta_s[-1]) <= w.tol
    assert (res.assignment == 0).all()
    chk = O.reference() if O.reference_available() else orc
    base = w.solver_config()
    cfg = SolverConfig(lambda_=res.lambda_, rho0=base.rho0, kappa=base.kappa, tol=base.tol,
                       max_iter=base.max_iter, c=1, fixed_iters=res.report.iters)
    d = X.shape[0]
    for r0, r1 in ((0, 96), (19_968, 20_032), (d - 96, d)):
        ref = chk.solve(np.asfortranarray(X[r0:r1]), cfg)
        assert ref.iters == res.report.iters
        assert bitwise(res.L[r0:r1], ref.L), (r0, r1)
        assert bitwise(res.S[r0:r1], ref.S), (r0, r1)
    del X
