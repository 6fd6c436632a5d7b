"""respca_b200 — the reference CLI (proj/tools/respca_cli.cpp) on the B200
engine; cases follow the reference's own proj/tests/test_cli.cpp.  CPU cases
(usage, synth) run anywhere; solves are marked gpu."""
import json
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from paper_1904_07497_b200 import respca

CLI = str(respca.__file__).rsplit("/", 1)[0] + "/lib/respca_b200"


def run(*args):
    p = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=600)
    return p.returncode, p.stdout, p.stderr


def test_help_and_usage_exit_codes(tmp_path):
    assert run("--help")[0] == 0
    assert run()[0] == 2
    assert run("nosuch")[0] == 2
    assert run("decompose", "--groups", "1")[0] == 2  # missing --input
    rc, _, err = run("decompose", "--input", tmp_path / "missing.csv", "--groups", "1")
    assert rc == 2 and "does not exist" in err
    assert run("decompose", "--input", tmp_path / "x.csv", "--bogus", "1")[0] == 2
    assert run("frames", "--frames", tmp_path, "--groups", "1")[0] == 2


def test_synth_rejects_c_above_n():
    assert run("synth", "--c", 5, "--n", 3, "--d", 4)[0] == 2  # test_cli.cpp:82-84


def test_synth_reloadable(tmp_path):  # test_cli.cpp:61-80
    x, l0, s0 = tmp_path / "x.bin", tmp_path / "l0.bin", tmp_path / "s0.bin"
    assert run("synth", "--d", 50, "--n", 120, "--c", 3, "--sparsity", 0.05, "--seed", 7,
               "--out-x", x, "--out-l0", l0, "--out-s0", s0)[0] == 0
    mx, ml, ms = (respca.read_binary_matrix(p) for p in (x, l0, s0))
    assert int(np.count_nonzero(ms)) == 300
    assert np.array_equal(mx, ml + ms)


@pytest.mark.skipif(not O.reference_io_available(), reason="reference I/O not built")
@pytest.mark.parametrize("args", [(50, 120, 3, 0.05, 1.0, 0.0, 7), (13, 40, 40, 0.3, 5.0, 0.1, 2),
                                  (7, 9, 1, 0.0, 1.0, 0.5, 0)])
def test_synth_bytes_match_reference(tmp_path, args):
    """The restated io::synth_generate produces the reference's exact bytes."""
    d, n, c, sp, mag, sig, seed = args
    paths = [tmp_path / f"{k}.bin" for k in ("x", "l0", "s0")]
    lab = tmp_path / "labels.csv"
    assert run("synth", "--d", d, "--n", n, "--c", c, "--sparsity", sp, "--magnitude", mag,
               "--noise-sigma", sig, "--seed", seed, "--out-x", paths[0], "--out-l0", paths[1],
               "--out-s0", paths[2], "--out-labels", lab)[0] == 0
    ref = O.reference_io().synth(d, n, c, sp, mag, sig, seed)
    for p, r in zip(paths, ref[:3]):
        assert np.array_equal(respca.read_binary_matrix(p).view(np.uint64), r.view(np.uint64))
    assert np.array_equal(np.loadtxt(lab, dtype=np.uint64, ndmin=1), ref[3])


@pytest.mark.gpu
def test_decompose_end_to_end(tmp_path):  # test_cli.cpp:86-115
    x = tmp_path / "x.bin"
    assert run("synth", "--d", 60, "--n", 150, "--c", 3, "--sparsity", 0.05, "--seed", 3,
               "--out-x", x)[0] == 0
    lo, so, rep = tmp_path / "l.bin", tmp_path / "s.bin", tmp_path / "report.jsonl"
    rc, out, err = run("decompose", "--input", x, "--groups", 3, "--out-l", lo, "--out-s", so,
                       "--report", rep)
    assert rc == 0, err
    lines = [json.loads(s) for s in rep.read_text().splitlines() if s]
    summary = lines[-1]
    assert summary["converged"] is True and 23 <= summary["iters"] <= 28
    assert len(lines) == summary["iters"] + 1 and lines[0]["iter"] == 1
    mx, ml, ms = (respca.read_binary_matrix(p) for p in (x, lo, so))
    assert np.linalg.norm(mx - ml - ms) / np.linalg.norm(mx) <= 2e-3
    assert out.startswith("converged=true iters=")


@pytest.mark.gpu
def test_decompose_csv_auto_lambda(tmp_path):  # test_cli.cpp:126-138
    rng = np.random.default_rng(5)
    x = tmp_path / "x.csv"
    np.savetxt(x, rng.uniform(0, 1, (100, 200)), delimiter=",", fmt="%.17g")
    rep = tmp_path / "r.jsonl"
    rc, _, err = run("decompose", "--input", x, "--groups", 2, "--lambda", "auto", "--max-iter", 5,
                     "--report", rep)
    assert rc == 0, err
    s = json.loads(rep.read_text().splitlines()[-1])
    assert abs(s["lambda"] - np.sqrt(200.0)) <= 1e-4 * np.sqrt(200.0)
    assert run("decompose", "--input", x, "--groups", 0)[0] == 2


@pytest.mark.gpu
def test_outliers_flags_corrupted_columns(tmp_path):  # test_cli.cpp:140-
    rng = np.random.default_rng(6)
    base = rng.uniform(0, 1, 40)
    X = np.tile(base[:, None], (1, 30))
    X[:, 7] += rng.uniform(5, 6, 40)
    X[:, 21] -= rng.uniform(5, 6, 40)
    x = tmp_path / "x.bin"
    respca.write_binary_matrix(x, X)
    rc, out, err = run("outliers", "--input", x, "--groups", 1, "--threshold", 10)
    assert rc == 0, err
    flagged = sorted(int(s.split()[0]) for s in out.splitlines() if s.endswith("FLAGGED"))
    assert flagged == [7, 21]


@pytest.mark.gpu
def test_outliers_reference_scenario(tmp_path):  # test_cli.cpp:136-165 (CSV input)
    rng = np.random.default_rng(6)
    base = rng.uniform(0, 1, 30)
    m = np.tile(base[:, None], (1, 30))
    m[:, 10] = 10.0 * rng.uniform(0, 1, 30)
    m[:, 20] = 10.0 * rng.uniform(0, 1, 30)
    x = tmp_path / "x.csv"
    np.savetxt(x, m, delimiter=",", fmt="%.17g")
    rc, out, err = run("outliers", "--input", x, "--groups", 1, "--threshold", 5)
    assert rc == 0, err
    assert "# threshold=5" in out and out.count("FLAGGED") == 2
