"""CPU: the seeded generator is deterministic (thread-count independent) and
reproduces the inputs the golden fixtures were made from."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from helpers import GOLDEN, load, sha, small_cases

ROOT = Path(__file__).resolve().parents[1]


def test_generator_thread_invariant():
    code = ("import sys; sys.path.insert(0, %r); from paper_1904_07497_b200 import synth; "
            "import hashlib; X = synth.rpca(300, 257, 7, 0.5, 0.1, seed=9); "
            "print(hashlib.sha256(X.tobytes(order='F')).hexdigest())") % str(ROOT)
    outs = set()
    for threads in ("1", "3", "8"):
        env = dict(os.environ, OMP_NUM_THREADS=threads)
        outs.add(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                                text=True, check=True).stdout.strip())
    assert len(outs) == 1


@pytest.mark.parametrize("case", small_cases(), ids=lambda c: c["case"])
def test_small_golden_inputs(case):
    from helpers import make_x

    make_x(case)  # asserts the sha


@pytest.mark.parametrize("name", ["C1", "C1-default-lambda", "C1-c1", "C2", "C2-c1", "C3-c1"])
def test_workload_golden_inputs(name):
    case = load(f"solve_{name}.json")
    if case is None:
        pytest.skip("fixture not generated")
    from helpers import make_x

    make_x(case)


def test_rpca_statistics():
    from paper_1904_07497_b200 import synth

    X, L0, S0 = synth.rpca(400, 300, 10, 1.0 / np.sqrt(10), 0.1, seed=1, with_truth=True)
    assert np.array_equal(X, L0 + S0)
    frac = np.count_nonzero(S0) / S0.size
    assert abs(frac - 0.1) < 0.01
    nz = S0[S0 != 0]
    assert nz.min() >= -50 and nz.max() <= 50
    assert np.linalg.matrix_rank(L0) == 10


def test_video_statistics():
    from paper_1904_07497_b200 import synth

    X, L0, S0 = synth.video(frames=40, height=48, width=64, block=8, blur_sigma=6.0,
                            seed=3, with_truth=True)
    assert X.shape == (48 * 64, 40)
    assert X.min() >= 0.0 and X.max() <= 1.0
    assert np.linalg.matrix_rank(L0, tol=1e-9) == 3
    frac = np.count_nonzero(np.abs(S0) > 0) / S0.size
    assert 0.005 < frac < 0.03  # one 8×8 block per 48×64 frame ≈ 2 %
