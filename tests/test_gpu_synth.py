"""§8(f) item 2: the respca-synth-1 generator with its O(d·n) assembly on the
device is byte-identical to the host generator (csrc/synth.c)."""
import numpy as np
import pytest

from paper_1904_07497_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("args", [(500, 500, 25, 1.0, 0.05, 42), (2000, 2000, 100, 1.0, 0.1, 42),
                                  (301, 77, 3, 0.3, 0.5, 9), (1, 5, 1, 2.0, 0.0, 1)])
def test_device_generator_bytes(ctx, args):
    d, n, r, sigma, p, seed = args
    host = synth.rpca(d, n, r, sigma, p, seed=seed)
    dev = synth.rpca_device(d, n, r, sigma, p, seed=seed, ctx=ctx)
    assert np.array_equal(host.view(np.uint64), dev.view(np.uint64))
    dev32 = synth.rpca_device(d, n, r, sigma, p, seed=seed, dtype=np.float32, ctx=ctx)
    assert np.array_equal(dev32, host.astype(np.float32))


def test_device_generator_c3_matches_workload(ctx):
    w = synth.WORKLOADS["C3"]
    a = w.make()
    b = w.make_device(ctx=ctx)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


# io::synth_generate (io.cpp:232-294) with the d×n assembly on the device
SPECS = [(50, 120, 3, 0.05, 1.0, 0.0, 7), (64, 64, 64, 0.3, 2.5, 0.0, 1), (33, 101, 7, 0.0, 1.0, 0.0, 2),
         (20, 30, 4, 0.999, 5.0, 0.0, 3), (40, 90, 5, 0.1, 1.0, 0.25, 4), (1, 1, 1, 0.5, 1.0, 0.0, 5),
         (700, 900, 11, 0.07, 3.0, 0.01, 11)]


@pytest.mark.parametrize("spec", SPECS)
def test_synth_generate_device_bytes(ctx, spec):
    """respca_cu_synth_generate against the unmodified reference's
    io::synth_generate: X, L0, S0 and the labels byte-identical (uniform
    prototypes, partial Fisher-Yates positions, signs, magnitudes, noise)."""
    from oracle import oracle as O
    from paper_1904_07497_b200 import respca as R

    d, n, c, sp, mag, sig, seed = spec
    x, l0, s0, lab = O.reference_io().synth(d, n, c, sp, mag, sig, seed)
    got = R.synth_generate(d, n, c, sp, mag, sig, seed, ctx=ctx)
    for a, b in ((x, got.x), (l0, got.l0), (s0, got.s0)):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    assert np.array_equal(lab, got.assignment)
    assert int((got.s0 != 0).sum()) == int(np.floor(sp * d * n + 0.5))  # llround


@pytest.mark.parametrize("bad", [(0, 5, 1, 0.1), (5, 0, 1, 0.1), (4, 3, 5, 0.1), (4, 3, 0, 0.1), (4, 3, 2, 1.0),
                                 (4, 3, 2, -0.1)])
def test_synth_generate_device_rejects(ctx, bad):
    """The reference's argument checks (io.cpp:233-241), same messages."""
    from oracle import oracle as O
    from paper_1904_07497_b200 import respca as R

    d, n, c, sp = bad
    with pytest.raises(ValueError) as ours:
        R.synth_generate(d, n, c, sp, ctx=ctx)
    with pytest.raises(Exception) as ref:
        O.reference_io().synth(d, n, c, sp)
    assert str(ref.value).split(": ", 1)[-1] in str(ours.value) or str(ours.value) in str(ref.value)


def test_cli_synth_on_device(tmp_path):
    """`respca_b200 synth --device 0` writes the reference's bytes."""
    import subprocess
    from pathlib import Path

    from oracle import oracle as O
    from paper_1904_07497_b200 import respca as R

    exe = Path(__file__).resolve().parents[1] / "paper_1904_07497_b200" / "lib" / "respca_b200"
    d, n, c, sp, mag, sig, seed = 60, 150, 3, 0.05, 1.5, 0.0, 3
    r = subprocess.run([str(exe), "synth", "--d", str(d), "--n", str(n), "--c", str(c), "--sparsity", str(sp),
                        "--magnitude", str(mag), "--seed", str(seed), "--device", "0", "--out-x",
                        str(tmp_path / "x.bin"), "--out-s0", str(tmp_path / "s0.bin")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    x, l0, s0, lab = O.reference_io().synth(d, n, c, sp, mag, sig, seed)
    assert np.array_equal(R.read_binary_matrix(tmp_path / "x.bin").view(np.uint64), x.view(np.uint64))
    assert np.array_equal(R.read_binary_matrix(tmp_path / "s0.bin").view(np.uint64), s0.view(np.uint64))
