"""Device memory checking without compute-sanitizer (closed on the GPU pool):
RESPCA_GUARD=1 poisons every device allocation with 0xFF bytes (NaN in any
floating-point buffer, −1 in an index buffer) and puts a 4 KiB guard after
it.  Every path below must stay bit-identical to the oracle — a read of
memory no kernel wrote would carry the poison into L, S or the labels — and
leave every guard intact (no write past the end of a buffer).

Runs in a subprocess so the switch is read at start-up."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

CODE = r'''
import ctypes as C, sys
import numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from helpers import bitwise, cfg_from, load, make_x, sha
from oracle import oracle as O
from paper_1904_07497_b200 import _native as N, respca, synth
from paper_1904_07497_b200.respca import KMeansConfig, SolverConfig
orc = O.port()
ctx = N.Context(0)
def same(X, cfg, prec="f64"):
    a = respca.solve(X, cfg, ctx=ctx, precision=prec)
    if prec == "f32":
        return
    b = orc.solve(X, cfg)
    assert a.report.iters == b.iters, (a.report.iters, b.iters)
    assert (a.assignment == b.labels).all()
    assert bitwise(a.L, b.L) and bitwise(a.S, b.S)
X = synth.rpca(96, 130, 4, 1.0, 0.05, seed=7)
same(X, SolverConfig(c=4, tol=1e-6))                       # TMA/tcgen05 screen, ring Pass F
same(X, SolverConfig(c=1, tol=1e-6))                       # stream Pass F
same(X, SolverConfig(c=5, tol=1e-6, sparse_norm="L21"))    # l2,1 passes
same(X, SolverConfig(c=3, fixed_iters=0))
same(np.asfortranarray(X[:95]), SolverConfig(c=3, tol=1e-6))  # odd d
respca.solve(X.astype(np.float32), SolverConfig(c=4, tol=1e-5), precision="f32", ctx=ctx)
case = load("solve_C1.json")
r = respca.solve(make_x(case), cfg_from(case["config"]), ctx=ctx)
assert sha(r.L) == case["ref"]["L_sha256"] and sha(r.S) == case["ref"]["S_sha256"]
m = np.random.default_rng(3).uniform(-1, 1, (64, 900))
a = respca.kmeans(m, KMeansConfig(c=9, seed=2, n_restarts=3), ctx=ctx)  # Gram Hartigan clusters
lab, cen, inertia, it = orc.kmeans(m, 9, 100, 3, 2, 1e-6)
assert (a.assignment == lab).all() and bitwise(a.centroids, cen)
msg = C.create_string_buffer(2048)
bad = N.lib().respca_cu_debug_guards(msg, 2048)
assert bad == 0, (bad, msg.value.decode())
print("guards ok")
'''


def test_poisoned_guarded_allocations():
    env = dict(os.environ, RESPCA_GUARD="1")
    p = subprocess.run([sys.executable, "-c", CODE], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=900)
    assert p.returncode == 0 and "guards ok" in p.stdout, (p.stdout[-2000:], p.stderr[-3000:])
