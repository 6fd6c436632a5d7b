"""CPU: the drop-in boundary — the C-ABI library loads, exports every symbol
include/*.h declares, and fails loudly (no CPU fallback) without a GPU."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared(header: Path, prefix: str) -> set[str]:
    text = header.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(rf"\b({prefix}\w+)\s*\(", text))


def test_engine_exports_every_declared_symbol():
    from paper_1904_07497_b200 import _native as N

    lib = N.lib()
    names = declared(ROOT / "include" / "respca_cu.h", "respca_cu_")
    assert len(names) >= 20
    missing = [nm for nm in sorted(names) if not hasattr(lib, nm)]
    assert not missing, missing
    assert names == set(N.EXPORTS), "python binding list drifted from the header"


def test_engine_is_sm100a_code():
    import subprocess

    so = ROOT / "paper_1904_07497_b200" / "lib" / "librespca_cu.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_no_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1904_07497_b200 import _native as N
    from paper_1904_07497_b200 import respca
    import numpy as np

    with pytest.raises(RuntimeError, match="no CPU fallback|no usable sm_100"):
        N.Context(0)
    with pytest.raises(RuntimeError):
        respca.solve(np.ones((3, 4)), respca.SolverConfig())


def test_default_config_matches_reference_defaults():
    """solver.hpp:15-24, kmeans.hpp:12-16."""
    from paper_1904_07497_b200 import _native as N
    from paper_1904_07497_b200.respca import SolverConfig

    cc = N.CConfig()
    N.lib().respca_cu_default_config(C.byref(cc))
    py = SolverConfig().to_c()
    for f, _ in N.CConfig._fields_:
        assert getattr(cc, f) == getattr(py, f), f
    assert (cc.rho0, cc.kappa, cc.tol, cc.max_iter, cc.c) == (1e-4, 1.5, 1e-3, 500, 1)
    assert (cc.km_max_iters, cc.km_n_restarts, cc.km_seed, cc.km_tol) == (100, 1, 0, 1e-6)


def test_config_struct_layout_matches_header():
    """ctypes mirror of respca_cu_config / respca_cu_report has the C layout."""
    import subprocess
    import tempfile

    from paper_1904_07497_b200 import _native as N

    src = r'''
#include <stddef.h>
#include <stdio.h>
#include "respca_cu.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu\n", sizeof(respca_cu_config), offsetof(respca_cu_config, fixed_iters),
         sizeof(respca_cu_report), offsetof(respca_cu_report, stop_resolves),
         offsetof(respca_cu_config, km_tol));
  return 0;
}'''
    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "l.c"
        p.write_text(src)
        exe = Path(td) / "l"
        subprocess.run(["gcc", f"-I{ROOT / 'include'}", str(p), "-o", str(exe)], check=True)
        out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    got = [C.sizeof(N.CConfig), N.CConfig.fixed_iters.offset, C.sizeof(N.CReport),
           N.CReport.stop_resolves.offset, N.CConfig.km_tol.offset]
    assert [int(v) for v in out] == got


def test_dropin_header_compiles_and_links():
    """The C++ drop-in facade (include/respca_b200/respca.hpp) builds against
    the C-ABI library: a user program that calls respca::solve links."""
    import subprocess
    import tempfile

    lib = ROOT / "paper_1904_07497_b200" / "lib"
    if not (lib / "librespca_b200.so").exists():
        pytest.skip("drop-in not built")
    src = r'''
#include "respca_b200/respca.hpp"
int main() {
  respca::SolverConfig cfg; cfg.c = 2; cfg.validate();
  respca::DenseMatrix x(3, 4);
  return cfg.resolve_lambda(3, 4) > 1.9 ? 0 : 1;
}'''
    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "u.cpp"
        p.write_text(src)
        exe = Path(td) / "u"
        subprocess.run(["g++", "-std=c++20", f"-I{ROOT / 'include'}", str(p), "-o", str(exe),
                        f"-L{lib}", "-lrespca_b200", "-lrespca_cu", f"-Wl,-rpath,{lib}"],
                       check=True)
        assert subprocess.run([str(exe)]).returncode == 0
