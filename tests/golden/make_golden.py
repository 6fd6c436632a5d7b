"""Generate the golden fixtures from the UNMODIFIED reference (oracle/_ref).

    python tests/golden/make_golden.py small            # seconds: unit + small solves
    python tests/golden/make_golden.py C1 C2 C2-c1 ...  # BASELINE workloads (C3: ~40 min)

The reference ships no golden vectors; these fixtures are
its outputs on seeded inputs, stored as exact fingerprints: SHA-256 of the
raw little-endian bytes of L and S, the labels (zlib+base64), and the report
vectors as exact hex floats.  X itself is regenerated from the seeded
generator (paper_1904_07497_b200/csrc/synth.c), whose bytes are pinned by
x_sha256.  Needs /root/reference (this container), never the GPU box.
"""
from __future__ import annotations

import base64
import hashlib
import json
import sys
import time
import zlib
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_1904_07497_b200 import synth  # noqa: E402
from paper_1904_07497_b200.respca import KMeansConfig, SolverConfig  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.asfortranarray(a).tobytes(order="F")).hexdigest()


def pack_labels(lab: np.ndarray) -> str:
    return base64.b64encode(zlib.compress(np.asarray(lab, dtype=np.uint32).tobytes(), 9)).decode()


def unpack_labels(s: str) -> np.ndarray:
    return np.frombuffer(zlib.decompress(base64.b64decode(s)), dtype=np.uint32).astype(np.uint64)


def hexs(v) -> list[str]:
    return [float(x).hex() for x in np.asarray(v, dtype=np.float64)]


def cfg_dict(cfg: SolverConfig) -> dict:
    return {"lambda_": cfg.lambda_, "rho0": cfg.rho0, "kappa": cfg.kappa, "tol": cfg.tol,
            "max_iter": cfg.max_iter, "c": cfg.c, "sparse_norm": cfg.sparse_norm,
            "kmeans": vars(cfg.kmeans), "fixed_iters": cfg.fixed_iters}


def cfg_from(d: dict) -> SolverConfig:
    km = KMeansConfig(**d["kmeans"])
    return SolverConfig(lambda_=d["lambda_"], rho0=d["rho0"], kappa=d["kappa"], tol=d["tol"],
                        max_iter=d["max_iter"], c=d["c"], sparse_norm=d["sparse_norm"],
                        kmeans=km, fixed_iters=d["fixed_iters"])


def solve_case(name: str, gen: dict, X: np.ndarray, cfg: SolverConfig) -> dict:
    ref = O.reference()
    t = time.time()
    r = ref.solve(X, cfg)
    el = time.time() - t
    return {
        "case": name, "generator": gen, "x_sha256": sha(X), "config": cfg_dict(cfg),
        "ref": {
            "iters": r.iters, "converged": r.converged, "lambda": float(r.lambda_).hex(),
            "L_sha256": sha(r.L), "S_sha256": sha(r.S), "labels": pack_labels(r.labels),
            "feas": hexs(r.feas), "delta_l": hexs(r.delta_l), "delta_s": hexs(r.delta_s),
            "objective": hexs(r.objective), "S_nnz": int(np.count_nonzero(r.S)),
            "L_fro": float(np.linalg.norm(r.L)), "S_fro": float(np.linalg.norm(r.S)),
            "wall_time_s": r.wall_time, "elapsed_s": el,
        },
    }


def sketch_mats(d: int, n: int, k: int = 16, seed: int = 7):
    """Seeded ±1 sketch matrices Ψ (d×k), Ω (n×k); relative Frobenius errors
    are estimated as ‖Ψᵀ(A − B)Ω‖_F / ‖ΨᵀBΩ‖_F (JL-style, k² samples)."""
    rng = np.random.default_rng(seed)
    return (rng.integers(0, 2, (d, k)) * 2.0 - 1.0, rng.integers(0, 2, (n, k)) * 2.0 - 1.0)


def sketch(a: np.ndarray, psi: np.ndarray, omega: np.ndarray) -> np.ndarray:
    return psi.T @ (np.asarray(a, dtype=np.float64) @ omega)


def workload_sketch(name: str) -> dict:
    """Reference solve of a workload with tolerance fingerprints (for fp32 runs
    that are compared within 1e-4 instead of bitwise)."""
    w = synth.WORKLOADS[name]
    X = w.make()
    X = X.astype(np.float32).astype(np.float64)
    r = O.reference().solve(X, w.solver_config())
    psi, om = sketch_mats(*X.shape)
    return {"case": name, "x_sha256": sha(X), "iters": r.iters,
            "L_fro": float(np.linalg.norm(r.L)), "S_fro": float(np.linalg.norm(r.S)),
            "L_sketch": sketch(r.L, psi, om).ravel().tolist(),
            "S_sketch": sketch(r.S, psi, om).ravel().tolist(),
            "S_nnz": int(np.count_nonzero(r.S)),
            "S_support_hash": hashlib.sha256(np.packbits(np.asfortranarray(r.S) != 0).tobytes()).hexdigest()}


def workload_case(name: str) -> dict:
    w = synth.WORKLOADS[name]
    X = w.make()
    if w.dtype == "f32":  # the fp32 workloads are solved from the same f32-rounded input
        X = X.astype(np.float32).astype(np.float64)
    gen = {"workload": name, "version": synth.version()}
    return solve_case(name, gen, X, w.solver_config())


SMALL = [
    # (name, d, n, r, sigma, p, seed, solver overrides)
    ("tiny-c3", 40, 60, 3, 1.0, 0.05, 1, dict(c=3, tol=1e-7)),
    ("tiny-c1", 30, 50, 2, 1.0, 0.05, 2, dict(c=1, tol=1e-7)),
    ("small-c5-smalllam", 80, 120, 5, 1.0, 0.05, 3, dict(c=5, tol=1e-7, lambda_=0.05)),
    ("small-c8-fixed", 64, 96, 4, 1.0, 0.08, 4, dict(c=8, fixed_iters=12)),
    ("odd-d-c4", 37, 91, 4, 1.0, 0.05, 5, dict(c=4, tol=1e-6)),
    ("tall-c2", 300, 40, 2, 1.0, 0.05, 6, dict(c=2, tol=1e-7)),
    ("wide-c10", 20, 400, 6, 1.0, 0.05, 7, dict(c=10, tol=1e-7, lambda_=0.3)),
    ("maxiter-cap", 50, 70, 4, 1.0, 0.1, 8, dict(c=3, tol=1e-12, max_iter=15)),
    ("c-equals-n", 12, 9, 3, 1.0, 0.1, 9, dict(c=9, tol=1e-6)),
    ("seed7-restarts", 48, 150, 6, 1.0, 0.05, 10, dict(c=6, tol=1e-7)),
]


def small_cases() -> list[dict]:
    out = []
    for name, d, n, r, sig, p, seed, over in SMALL:
        X = synth.rpca(d, n, r, sig, p, seed=seed)
        cfg = SolverConfig(**{k: v for k, v in over.items()})
        if name == "seed7-restarts":
            cfg.kmeans = KMeansConfig(seed=7, n_restarts=7)
        gen = {"rpca": dict(d=d, n=n, r=r, sigma=sig, p=p, seed=seed), "version": synth.version()}
        out.append(solve_case(name, gen, X, cfg))
    return out


def main(argv: list[str]) -> None:
    if not O.reference_available():
        O.ensure_built()
    for arg in argv:
        if arg == "small":
            cases = small_cases()
            (OUT / "small_solves.json").write_text(json.dumps(cases, indent=1))
            print("wrote small_solves.json", len(cases))
        elif arg.startswith("sketch-"):
            name = arg[len("sketch-"):]
            rec = workload_sketch(name)
            (OUT / f"sketch_{name}.json").write_text(json.dumps(rec))
            print("wrote sketch", name)
        elif arg.startswith("init-"):
            # the reference's one-time kmeans(X) labels (solver.cpp:145-148):
            # the bench's reference arm replays the ALM loop from them
            name = arg[len("init-"):]
            w = synth.WORKLOADS[name]
            X = w.make()
            t = time.time()
            lab, _, inertia, it = O.reference().kmeans(X, w.c, 100, 5, 0, 1e-6)
            rec = {"case": name, "x_sha256": sha(X), "labels": pack_labels(lab),
                   "inertia": float(inertia).hex(), "iters_run": int(it),
                   "elapsed_s": time.time() - t}
            (OUT / f"init_{name}.json").write_text(json.dumps(rec, indent=1))
            print("wrote init", name, rec["elapsed_s"])
        else:
            case = workload_case(arg)
            (OUT / f"solve_{arg}.json").write_text(json.dumps(case, indent=1))
            print("wrote", arg, case["ref"]["iters"], case["ref"]["elapsed_s"])


if __name__ == "__main__":
    main(sys.argv[1:] or ["small"])
