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
