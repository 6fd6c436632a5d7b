#!/usr/bin/env python
"""Benchmark: RES-PCA ALM iterations/sec + time-to-converge on one B200
(BASELINE.json metric), workload C3 = d=n=10000, rank 50, c=50, fp64, tol 1e-7.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload C3] [--no-cpu-baseline] [--no-e2e]

One "step" = one ALM iteration of respca::solve (solver.cpp:157-201) over the
whole d×n matrix.  Arms:
  ours       value  = K / device time of K resident iterations (X, L, S, Θ in HBM)
             e2e    = iterations / wall time of a complete respca_cu_solve() from
                      pinned host X to host L, S, labels (H2D, one-time kmeans(X),
                      the loop, D2H all inside) — the drop-in call a user makes.
  reference  the UNMODIFIED reference (oracle/_ref, compiled from the reference
             sources) replaying the same ALM iterations on the host CPU from the
             reference's own initial kmeans(X) labels (tests/golden/init_C3.json).
Multi-GPU: the path does not shard (every config fits one B200): --gpus N runs
N independent replicas (one process per GPU, torchrun), value = total
iterations / max-over-ranks device time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "RES-PCA iters/sec + time-to-converge (1 B200) & HBM GB/s as % of 8 TB/s roofline"


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "src": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "src": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML in a
    background thread every 5 ms (nvidia-smi's 50 ms floor is longer than a
    short timed region); falls back to `nvidia-smi -lms 50`."""

    REASONS = {  # nvmlClocksEventReason* bits
        0x0000000000000004: "sw_power_cap",
        0x0000000000000008: "hw_slowdown",
        0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000080: "hw_power_brake_slowdown",
    }

    def __init__(self, device: int):
        self.device = device
        self.samples: list[tuple[float, float, int]] = []
        self.stop = threading.Event()
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def run():
                while not self.stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((float(sm), float(mx), int(rs)))
                    except Exception:  # noqa: BLE001
                        pass
                    time.sleep(0.005)

            self.t = threading.Thread(target=run, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            try:
                q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                     "clocks_event_reasons.hw_thermal_slowdown,"
                     "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
                self.proc = subprocess.Popen(
                    ["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms",
                     "50", "-i", str(self.device)], stdout=subprocess.PIPE,
                    stderr=subprocess.DEVNULL, text=True)
                self.t = threading.Thread(target=lambda: [self.lines.append(x) for x in self.proc.stdout],
                                          daemon=True)
                self.t.start()
            except FileNotFoundError:
                pass
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        for s_, m_, rs in self.samples:
            sm.append(s_)
            mx = max(mx, m_)
            for bit, nm in self.REASONS.items():
                if rs & bit:
                    reasons.add(nm)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic(workload):
    """DRAM bytes per Pass-F launch from the committed ncu capture
    (profiles/ncu_traffic.json), or None when this workload was not captured."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f).get(workload)
        return None if t is None else t["read_bytes"] + t["write_bytes"]
    except (OSError, ValueError, KeyError):
        return None


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch.distributed as dist

        backend = "nccl" if args.impl == "ours" else "gloo"
        if backend == "nccl":
            import torch

            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
        pg = dist
    return world, rank, local, pg


def barrier(pg, local):
    if pg is None:
        return
    import torch

    if torch.cuda.is_available():
        torch.cuda.synchronize(local)
    pg.barrier()


def allmax(pg, value: float, local: int) -> float:
    if pg is None:
        return value
    import torch

    dev = torch.device("cuda", local) if torch.cuda.is_available() else torch.device("cpu")
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


class _Pinned(np.ndarray):
    pass


def pinned(d: int, n: int, dtype=np.float64) -> np.ndarray:
    import torch

    tdt = torch.float64 if dtype == np.float64 else torch.float32
    t = torch.empty((n, d), dtype=tdt, pin_memory=True)
    a = t.numpy().T.view(_Pinned)
    a.keep = t
    return a


def cpu_reference_sample(w, X: np.ndarray, iters: int) -> dict:
    """The unmodified reference (oracle/_ref) replaying `iters` ALM iterations
    of this workload on one host core, from its own kmeans(X) labels."""
    from oracle import oracle as O

    sys.path.insert(0, str(ROOT / "tests"))
    from helpers import load, unpack_labels

    init = load(f"init_{w.name}.json")
    if init is not None:
        labels = unpack_labels(init["labels"])
        src = "reference kmeans(X) labels (tests/golden)"
    else:
        labels = (np.arange(w.n) % w.c).astype(np.uint64)
        src = "round-robin labels (init fixture missing)"
    ref = O.reference()
    cfg = w.solver_config()
    cfg.fixed_iters = iters
    t0 = time.time()
    _, _, _, _, secs = ref.replay(X, cfg, labels, iters)
    wall = time.time() - t0
    per = float(np.mean(secs))
    return {"iter_seconds": [float(s) for s in secs], "mean_s": per, "wall_s": wall,
            "labels_src": src}


def run_reference(args, w, rank) -> None:
    if rank != 0:
        return
    from paper_1904_07497_b200 import synth

    # the input comes from the checker side's own build of the seeded generator
    # (oracle/libinput.so, same bytes as the ours arm): this arm loads only
    # libraries under oracle/ — the reference itself is oracle/_ref/librespca_ref.so
    synth.use_library(ROOT / "oracle" / "libinput.so")
    X = w.make()
    if w.dtype == "f32":
        X = X.astype(np.float32).astype(np.float64)
    # the driver's step counts, unless they would run past the arm's time budget
    # (≈8.6 s per C3 iteration on one core): then capped, and the line says why
    per_iter_est = 8.7 * (w.d * w.n) / 1e8
    budget_s = args.ref_budget_s
    warm, steps = args.warmup, args.steps
    cap = None
    if (warm + steps) * per_iter_est > budget_s:
        warm = min(warm, 1)
        steps = max(1, min(steps, int(budget_s / per_iter_est) - warm))
        cap = (f"capped from --steps {args.steps} --warmup {args.warmup}: one reference iteration "
               f"takes ≈{per_iter_est:.1f} s on one core, the arm's budget is {budget_s:.0f} s")
    s = cpu_reference_sample(w, X, warm + steps)
    timed = s["iter_seconds"][warm:]
    total = float(sum(timed))
    value = len(timed) / total
    ncpu = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "iters/s",
        "n_gpus": args.gpus, "steps": len(timed), "warmup": warm,
        "ms_per_step": 1e3 * total / len(timed), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, respca-synth-1)",
        "config": {**workload_config(w), "parallelism": f"replicas x{args.gpus}"},
        "cpu_baseline": {"value": value, "unit": "iters/s", "cores": 1, "kind": "reference",
                         "sample": f"{len(timed)} full ALM iterations of {w.name} replayed "
                                   f"through the reference's public building blocks "
                                   f"(solver.cpp:157-201 statement order) from "
                                   f"{s['labels_src']}; single-threaded reference, 1 of "
                                   f"{ncpu} host cores"},
        "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    if cap:
        line["steps_capped"] = cap
    print(json.dumps(line), flush=True)


def workload_config(w) -> dict:
    return {"workload": f"{w.name}: d={w.d} n={w.n} rank={w.r} c={w.c} {w.dtype} tol={w.tol}"
                        f" lambda={'sqrt(max(d,n))' if w.lambda_ is None else w.lambda_}",
            "d": w.d, "n": w.n, "c": w.c, "rank": w.r, "tol": w.tol,
            "l2_policy": "inputs larger than L2 (X, L, S, Θ = 3.2 GB at C3; 126 MB L2)",
            "generator": "respca-synth-1 seed 42"}


def run_ours(args, w, world, rank, local, pg) -> None:
    import ctypes as C

    from paper_1904_07497_b200 import _native as N
    from paper_1904_07497_b200 import respca

    ctx = N.Context(local)
    L = N.lib()
    dt = np.float32 if w.dtype == "f32" else np.float64
    Xp = pinned(w.d, w.n, np.float64)
    w.make_device(out=Xp, ctx=ctx)  # respca-synth-1, O(d·n) part assembled on the GPU
    if dt == np.float64:
        Xh = Xp
    else:  # fp32 storage: the caller's input is an f32 matrix in pinned memory
        Xh = pinned(w.d, w.n, np.float32)
        Xh[...] = Xp
    cfg = w.solver_config()
    cc = cfg.to_c()
    esize = 8 if dt == np.float64 else 4
    N_el = w.d * w.n

    # ---------------- end to end through the C-ABI ("e2e") ----------------
    # runs first, so its first call is the cold one (kernel modules, device
    # allocations, graph capture, tensor maps of this context all happen in it)
    e2e = None
    ttc = None
    if not args.no_e2e:
        Lh, Sh = pinned(w.d, w.n, dt), pinned(w.d, w.n, dt)
        runs = []
        cold = None
        for rep in range(1 + args.e2e_runs):  # first run: cold, reported apart
            barrier(pg, local)
            t0 = time.perf_counter()
            res = respca.solve(Xh, cfg, precision=w.dtype, ctx=ctx, out=(Lh, Sh))
            el = time.perf_counter() - t0
            if rep:
                runs.append((el, res))
            else:
                cold = el
            if os.environ.get("RESPCA_BENCH_VERBOSE"):
                print(f"e2e run {rep}: wall {el:.3f}s init {res.init_ms:.0f}ms loop {res.loop_ms:.0f}ms "
                      f"h2d {res.h2d_ms:.0f}ms d2h {res.d2h_ms:.0f}ms c-abi {res.wall_time:.3f}s",
                      file=sys.stderr, flush=True)
        el = allmax(pg, statistics.median(r[0] for r in runs), local)  # median run; all in runs_s
        cold = allmax(pg, cold, local)
        res = runs[-1][1]
        e2e = {"value": world * res.report.iters / el, "unit": "iters/s",
               "h2d_bytes_per_step": int(N_el * esize),
               "d2h_bytes_per_step": int(2 * N_el * esize + 8 * w.n + 32 * res.report.iters),
               "step": "one complete respca_cu_solve (pinned host X → host L, S, labels)",
               "iters": res.report.iters, "converged": res.report.converged,
               "wall_s": el, "runs_s": [round(r[0], 4) for r in runs],
               "cold_first_call_s": round(cold, 4),
               "cold_value": world * res.report.iters / cold}
        ttc = {"seconds": el, "device_init_ms": res.init_ms, "device_loop_ms": res.loop_ms,
               "h2d_ms": res.h2d_ms, "d2h_ms": res.d2h_ms, "iters": res.report.iters,
               "hartigan_moves": res.hartigan_moves, "exact_fallbacks": res.exact_fallbacks,
               "slow_iters": res.slow_iters, "stop_resolves": res.stop_resolves}
        # parity against the reference's golden fingerprint when one exists
        try:
            sys.path.insert(0, str(ROOT / "tests"))
            from helpers import load, sha, unpack_labels

            g = load(f"solve_{w.name}.json")
            if g is not None and w.dtype == "f64":
                ttc["parity_vs_reference"] = {
                    "iters_equal": res.report.iters == g["ref"]["iters"],
                    "labels_equal": bool((res.assignment == unpack_labels(g["ref"]["labels"])).all()),
                    "L_bitwise": sha(np.asarray(Lh)) == g["ref"]["L_sha256"],
                    "S_bitwise": sha(np.asarray(Sh)) == g["ref"]["S_sha256"],
                    "reference_solve_s": g["ref"]["elapsed_s"]}
        except Exception as exc:  # noqa: BLE001
            ttc["parity_vs_reference"] = f"unavailable: {exc}"

    # ---------------- device-resident throughput ("value") ----------------
    init_ms = C.c_double()
    N.check(ctx, L.respca_cu_bench_prepare(ctx.handle, Xh.ctypes.data_as(C.c_void_p), w.d, w.n,
                                           N.F64 if dt == np.float64 else N.F32, C.byref(cc),
                                           C.byref(init_ms)))
    ms, pf, pa, slow = C.c_double(), C.c_double(), C.c_double(), C.c_uint64()
    N.check(ctx, L.respca_cu_bench_steps(ctx.handle, args.warmup, C.byref(ms), C.byref(pf),
                                         C.byref(pa), C.byref(slow)))
    barrier(pg, local)
    l0 = ctx.launches()
    with ClockSampler(local) as clk:
        N.check(ctx, L.respca_cu_bench_steps(ctx.handle, args.steps, C.byref(ms), C.byref(pf),
                                             C.byref(pa), C.byref(slow)))
    launches = ctx.launches() - l0
    barrier(pg, local)
    t_ms = allmax(pg, ms.value, local)
    value = world * args.steps / (t_ms / 1e3)
    pf_avg = pf.value / args.steps
    pa_avg = pa.value / args.steps
    pk = peaks()
    alg_bytes = 7 * N_el * esize  # ALG_BYTES_PER_ITER = 7·d·n·s
    achieved = alg_bytes / (pf_avg / 1e3) / 1e9
    # Pass F also writes L′ as BF16 (2 B/element) for the TMA-fed tcgen05 screen
    # whenever 1 < c ≤ 64 (ℓ1): a design choice of this build, reported apart
    lb_side = 1 < w.c <= 64 and os.environ.get("RESPCA_TC_SCREEN", "") not in ("0", "1")
    side_bytes = 2 * N_el if lb_side else 0
    # whole-iteration roofline: same algorithmic bytes over the full step
    iter_gbs = alg_bytes / (t_ms / args.steps / 1e3) / 1e9

    # ---------------- CPU baseline (rank 0, N=1) ----------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            Xc = np.asarray(Xp)
            s = cpu_reference_sample(w, Xc if dt == np.float64 else Xc.astype(np.float32).astype(np.float64),
                                     args.cpu_iters)
            cpu = {"value": 1.0 / s["mean_s"], "unit": "iters/s", "cores": 1,
                   "kind": "reference",
                   "sample": f"{args.cpu_iters} full ALM iteration(s) of {w.name} by the "
                             f"unmodified reference (oracle/_ref) through its public building "
                             f"blocks from {s['labels_src']}; 1 of {os.cpu_count()} host cores",
                   "seconds_per_iter": s["mean_s"]}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "iters/s", "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": w.dtype, "data": "synthetic (seeded, respca-synth-1)",
            "config": {**workload_config(w), "parallelism": f"replicas x{world}"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"],
                         "unit": "GB/s", "frac": achieved / pk["hbm_gbs"], "traffic": ncu_traffic(args.workload),
                         "kernel": ("k_pass_f_stream" if (w.c == 1 and w.d <= 75776 and w.d % (2 if w.dtype == "f64" else 4) == 0)
                                    else "k_pass_f_ring") + " (Pass F: fused L/S/Θ update + group sums + residuals)",
                         "alg_bytes_per_launch": alg_bytes,
                         "alg_bytes_note": "7·N·s (X,S,Θ,L in; L,S,Θ out), SURVEY.md §8(d)",
                         "side_output_bytes_per_launch": side_bytes,
                         "side_output_note": ("BF16 copy of L′ (2·N bytes) for the TMA-fed tcgen05 screen: "
                                              "written by the kernel, not counted in achieved/frac")
                                             if side_bytes else None,
                         "kernel_bytes_frac": (alg_bytes + side_bytes) / (pf_avg / 1e3) / 1e9 / pk["hbm_gbs"],
                         "avg_launch_ms": pf_avg,
                         "peak_src": pk["src"],
                         "iteration_gbs": iter_gbs, "iteration_frac": iter_gbs / pk["hbm_gbs"],
                         "pass_a_ms": pa_avg},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "time_to_converge": ttc,
            "init_ms": init_ms.value,
            "slow_iters_in_timed_region": int(slow.value),
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-runs", type=int, default=5)
    ap.add_argument("--cpu-iters", type=int, default=1)
    ap.add_argument("--ref-budget-s", type=float, default=300.0,
                    help="reference arm: cap warm-up + timed iterations to about this many seconds")
    args = ap.parse_args()
    from paper_1904_07497_b200 import synth

    w = synth.WORKLOADS[args.workload]
    world, rank, local, pg = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, w, rank)
    else:
        run_ours(args, w, world, rank, local, pg)
    if pg is not None:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
