"""Build recipe for the native libraries (in-tree, sm_100a).

    python -m paper_1904_07497_b200.build      # or __graft_entry__.build()

Outputs (git-ignored, shipped to the GPU box with the snapshot):
    paper_1904_07497_b200/lib/librespca_cu.so   CUDA engine + C-ABI (include/respca_cu.h)
    paper_1904_07497_b200/lib/librespca_b200.so C++ drop-in (include/respca_b200/respca.hpp)
    paper_1904_07497_b200/lib/libsynth.so       host synthetic-input generator
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "lib"
INC = ROOT / "include"

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# --fmad=false: reference arithmetic (no FMA contraction); explicit __fma_rn only
NVFLAGS = ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
           "-Xptxas", "-v", "--expt-relaxed-constexpr", "-w"]


def _run(cmd: list[str], log: Path | None = None) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        log.write_text(res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:4])} ...")


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(p.stat().st_mtime > t for p in deps)


def build_cuda(force: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    out = LIB / "librespca_cu.so"
    deps = (list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [INC / "respca_cu.h", CSRC / "synth.c",
            CSRC / "synth.h"])
    if force or _stale(out, deps):
        # synth.c rides along for the device generator's host factors (U, V)
        _run([NVCC, *ARCH, *NVFLAGS, f"-I{INC}", f"-I{CSRC}", "-shared",
              str(CSRC / "engine.cu"), str(CSRC / "synth.c"), "-o", str(out), "-lcudart",
              "-Xcompiler", "-pthread,-ffp-contract=off"],
             log=LIB / "ptxas_engine.log")
    return out


def build_synth(force: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    out = LIB / "libsynth.so"
    deps = [CSRC / "synth.c", CSRC / "synth.h"]
    if force or _stale(out, deps):
        cc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"  # /opt/gcc lacks libgomp.spec
        _run([cc, "-std=c11", "-O3", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
              "-fno-fast-math", str(CSRC / "synth.c"), "-o", str(out), "-lm"])
    return out


def build_dropin(force: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    out = LIB / "librespca_b200.so"
    src = CSRC / "dropin.cpp"
    if not src.exists():
        return out
    deps = [src, INC / "respca_b200" / "respca.hpp", INC / "respca_cu.h"]
    if force or _stale(out, deps):
        cxx = os.environ.get("CXX", "g++")
        _run([cxx, "-std=gnu++20", "-O2", "-fPIC", "-shared", f"-I{INC}", str(src),
              "-o", str(out), f"-L{LIB}", "-lrespca_cu", "-Wl,-rpath,$ORIGIN"])
    return out


def build_cli(force: bool = False) -> Path:
    """respca_b200: the reference command-line tool on the C-ABI."""
    LIB.mkdir(exist_ok=True)
    out = LIB / "respca_b200"
    src = ROOT / "paper_1904_07497_b200" / "tools" / "respca_cli.cpp"
    deps = [src, INC / "respca_cu.h", LIB / "librespca_cu.so"]
    if force or _stale(out, deps):
        cxx = os.environ.get("CXX", "g++")
        _run([cxx, "-std=gnu++20", "-O2", f"-I{INC}", str(src), "-o", str(out), f"-L{LIB}",
              "-lrespca_cu", "-Wl,-rpath,$ORIGIN"])
    return out


def build_oracle() -> None:
    """CPU checkers (test infrastructure): oracle/liboracle.so always; the
    reference library oracle/_ref/ only where /root/reference exists."""
    _run(["make", "-s", "-C", str(ROOT / "oracle"), "all"])
    if Path("/root/reference/proj/tests/acceptance.cpp").exists():
        _run(["make", "-s", "-C", str(ROOT / "oracle"), "acceptance"])


def build_all(force: bool = False) -> None:
    build_synth(force)
    build_cuda(force)
    build_dropin(force)
    build_cli(force)
    build_oracle()


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print("built:", *sorted(p.name for p in LIB.glob("*.so")))
