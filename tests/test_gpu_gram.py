"""The Gram-matrix Hartigan refinement (csrc/hart_gram.cuh) against the oracle's
kmeans (kmeans.cpp:96-139, 237-250): labels, centroids, inertia and Lloyd
iterations bit-identical, on data built to stress it —

* integer-valued columns (exact distance ties),
* duplicate columns, tiny and large magnitudes,
* clusters of 1, 2, 4, 8 and 16 CTAs (RESPCA_GRAM_CL; 16 is the default at every n,
  also where most CTAs of the cluster own no column), the per-pass path
  (RESPCA_HART_GRAM=0) on the same inputs, and every move forced through the
  exact fallback (RESPCA_GRAM_FORCE_EXACT=1: the logged moves are replayed
  onto the reference's centroids and the reference's own chain decides).

Each configuration runs in a subprocess: the switches are read once per
process.  RESPCA_TRACE=1 makes the engine report which refinement ran and how
many exact fallbacks it took."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
from oracle import oracle as O
from paper_1904_07497_b200 import respca as R
from paper_1904_07497_b200.respca import KMeansConfig
from helpers import bitwise
orc = O.port()
rng = np.random.default_rng(7)
cases = []
# integer grid: many exact ties
cases.append(("ints", rng.integers(-2, 3, (8, 600)).astype(float), 6, 3, 3))
cases.append(("ints-wide", rng.integers(-1, 2, (5, 1500)).astype(float), 12, 1, 2))
# duplicates + a perturbed copy
base = rng.uniform(-1, 1, (16, 40))
dup = np.asfortranarray(np.concatenate([base] * 6, axis=1))
dup[:, 3] += 1e-9
cases.append(("dups", dup, 7, 5, 2))
# magnitudes far from 1
cases.append(("tiny", rng.normal(0, 1e-150, (24, 700)), 9, 2, 2))
cases.append(("large", rng.normal(0, 1e150, (24, 700)), 9, 4, 2))
# mixture with a sparse heavy part (the RPCA shape)
X = rng.normal(0, 1, (64, 2500)) + (rng.random((64, 2500)) < 0.1) * rng.uniform(-50, 50, (64, 2500))
cases.append(("rpca", X, 20, 11, 2))
bad = 0
for name, m, c, seed, restarts in cases:
    m = np.asfortranarray(m)
    a = R.kmeans(m, KMeansConfig(c=c, seed=seed, n_restarts=restarts))
    lab, cen, inertia, it = orc.kmeans(m, c, 100, restarts, seed, 1e-6)
    ok = (a.assignment == lab).all() and bitwise(a.centroids, cen) and a.inertia == inertia and a.iters_run == it
    print("CASE", name, "OK" if ok else "BAD", int((a.assignment != lab).sum()), flush=True)
    bad += not ok
sys.exit(1 if bad else 0)
"""


def run(env_extra):
    env = dict(os.environ, RESPCA_TRACE="1", **env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    return r


@pytest.mark.parametrize("cl", ["1", "2", "4", "8", "16"])
def test_gram_refinement_bitwise(cl):
    r = run({"RESPCA_GRAM_CL": cl})
    assert r.returncode == 0, r.stdout + r.stderr[-4000:]
    assert r.stdout.count(" OK ") == 6, r.stdout
    # the Gram refinement ran, with the requested cluster size
    runs = [ln for ln in r.stderr.splitlines() if "hartigan(gram, CL=" in ln]
    assert runs and all(f"CL={cl})" in ln for ln in runs), r.stderr[-2000:]


def fallbacks(stderr):
    return sum(int(ln.split(" fallbacks")[0].split()[-1]) for ln in stderr.splitlines()
               if "hartigan(gram, CL=" in ln)


@pytest.mark.parametrize("cl", ["1", "4", "16"])
def test_gram_exact_fallback_bitwise(cl):
    """Every provable move routed through the exact fallback (log replay onto
    the reference's centroids + the reference's chain): same results."""
    r = run({"RESPCA_GRAM_CL": cl, "RESPCA_GRAM_FORCE_EXACT": "1"})
    assert r.returncode == 0, r.stdout + r.stderr[-4000:]
    assert r.stdout.count(" OK ") == 6, r.stdout
    assert fallbacks(r.stderr) > 100, r.stderr[-2000:]


@pytest.mark.parametrize("env", [{"RESPCA_LLOYD_INCR": "0"}, {"RESPCA_PP_JOINT": "0", "RESPCA_KM_LANES": "3"},
                                 {"RESPCA_KM_LANES": "3"}])
def test_init_switches_bitwise(env):
    """Full Lloyd steps instead of incremental ones, restarts seeded one by
    one, and restarts side by side (lanes): the same results."""
    r = run(env)
    assert r.returncode == 0, r.stdout + r.stderr[-4000:]
    assert r.stdout.count(" OK ") == 6, r.stdout


@pytest.mark.parametrize("env,exact", [({"RESPCA_KM_LANES": "3"}, None),
                                       ({"RESPCA_KM_LANES": "3", "RESPCA_PP_GRAM_FORCE_AMB": "2"}, 1),
                                       ({"RESPCA_KM_LANES": "2", "RESPCA_PP_GRAM": "0"}, -1)])
def test_seeding_on_gram_bitwise(env, exact):
    """k-means++ d² from the Gram matrix (k_pp_gram) with its rigorous bound:
    the same picks as the reference's chains on tie-heavy, duplicate, tiny and
    large inputs; a restart forced to the exact chains (and the switch off)
    gives the same results."""
    r = run(env)
    assert r.returncode == 0, r.stdout + r.stderr[-4000:]
    assert r.stdout.count(" OK ") == 6, r.stdout
    lines = [ln for ln in r.stderr.splitlines() if "k-means++ on G:" in ln and "restarts," in ln]
    if exact == -1:
        assert not lines
    else:
        assert len(lines) >= 6, r.stderr[-2000:]
        if exact:
            assert all(int(ln.split(",")[-1].split()[0]) >= 1 for ln in lines), lines


def test_per_pass_refinement_bitwise():
    r = run({"RESPCA_HART_GRAM": "0"})
    assert r.returncode == 0, r.stdout + r.stderr[-4000:]
    assert r.stdout.count(" OK ") == 6, r.stdout
    assert "hartigan(gram" not in r.stderr


SHAPES = r"""
import sys, numpy as np
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
from oracle import oracle as O
from paper_1904_07497_b200 import respca as R
from paper_1904_07497_b200.respca import KMeansConfig
from helpers import bitwise
orc = O.port()
rng = np.random.default_rng(11)
bad = 0
# odd d / n (scalar copies, partial tiles), every KPL width (c ≤ 32, 64, 128, 256)
for d, n, c, seed in ((37, 517, 7, 1), (300, 1025, 33, 2), (64, 900, 70, 3), (21, 1300, 129, 4),
                      (16, 1500, 256, 5), (3, 40, 2, 6)):
    m = np.asfortranarray(rng.normal(0, 1, (d, n)) + (rng.random((d, n)) < 0.1) * rng.uniform(-20, 20, (d, n)))
    a = R.kmeans(m, KMeansConfig(c=c, seed=seed, n_restarts=2))
    lab, cen, inertia, it = orc.kmeans(m, c, 100, 2, seed, 1e-6)
    ok = (a.assignment == lab).all() and bitwise(a.centroids, cen) and a.inertia == inertia and a.iters_run == it
    print("SHAPE", d, n, c, "OK" if ok else "BAD", flush=True)
    bad += not ok
sys.exit(1 if bad else 0)
"""


@pytest.mark.parametrize("cl", ["1", "8", "16"])
def test_gram_shapes_bitwise(cl):
    """Odd row/column counts, partial Gram tiles and every lanes-per-centroid
    width of the refinement kernel (c up to its 256 limit)."""
    env = dict(os.environ, RESPCA_TRACE="1", RESPCA_GRAM_CL=cl)
    r = subprocess.run([sys.executable, "-c", SHAPES], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr[-4000:]
    assert r.stdout.count(" OK") == 6, r.stdout
    assert r.stderr.count("hartigan(gram, CL=") >= 6, r.stderr[-2000:]
