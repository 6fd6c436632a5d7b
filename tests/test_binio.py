"""RESPCA1 binary matrices (io.hpp:66-69, io.cpp:138-164) — host side of the
§8(f) disk → HBM streaming, pinned against the unmodified reference reader /
writer (oracle/_ref/librespca_ref_io.so).  No GPU needed."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1904_07497_b200 import _native as N
from paper_1904_07497_b200 import respca

needs_ref = pytest.mark.skipif(not O.reference_io_available(), reason="reference I/O not built")


@needs_ref
def test_roundtrip_both_ways(tmp_path):
    ref = O.reference_io()
    rng = np.random.default_rng(1)
    for shape in ((1, 1), (7, 3), (40, 65)):
        m = rng.standard_normal(shape)
        m.flat[0] = -0.0
        p1, p2 = tmp_path / "ref.bin", tmp_path / "ours.bin"
        ref.write_binary(p1, m)
        respca.write_binary_matrix(p2, m)
        assert p1.read_bytes() == p2.read_bytes()  # byte-identical files
        assert respca.binary_info(p1) == shape
        a = respca.read_binary_matrix(p1)
        b = ref.read_binary(p2)
        assert np.array_equal(a.view(np.uint64), np.asfortranarray(m).view(np.uint64))
        assert np.array_equal(b.view(np.uint64), np.asfortranarray(m).view(np.uint64))


@needs_ref
@pytest.mark.parametrize("kind", ["missing", "short", "magic", "header", "payload"])
def test_errors_match_reference(tmp_path, kind):
    ref = O.reference_io()
    p = tmp_path / "bad.bin"
    good = np.arange(12.0).reshape(3, 4)
    respca.write_binary_matrix(p, good)
    raw = p.read_bytes()
    if kind == "missing":
        p = tmp_path / "none.bin"
    elif kind == "short":
        p.write_bytes(b"RESP")
    elif kind == "magic":
        p.write_bytes(b"RESPCA2\0" + raw[8:])
    elif kind == "header":
        p.write_bytes(raw[:12])
    else:
        p.write_bytes(raw[:-8])
    with pytest.raises(OSError) as ours:
        respca.binary_info(p)
    with pytest.raises(OSError) as theirs:
        ref.read_binary(p)
    assert str(ours.value) == str(theirs.value)
    assert isinstance(ours.value, N.IoError)


def test_c_abi_exports_io_symbols():
    lib = N.lib()
    for sym in ("respca_cu_binary_info", "respca_cu_solve_file", "respca_cu_outlier_scores"):
        assert hasattr(lib, sym)
