"""Benchmark: MGRIT time-to-solution on BASELINE config 2 (127^2 DOF x 4096 steps, multilevel V, m=8).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg2] [--nt NT]

One "step" = one complete MGRIT solve (G setup, V-cycles to residual < 1e-8,
finalisation) of the canonical seeded cfg2 problem.  Prints ONE JSON line.

Arms
  ours       the B200 path.  ``value`` = ndof*Nt / time-to-solution with the
             problem resident on the device (CUDA events, max over ranks);
             ``e2e`` = same metric through the public API ``solve(spec, opts)``
             returning the host numpy array (H2D of inputs, D2H of U inside the
             timed region).
  reference  the reference's CPU implementation of the path (the oracle port,
             oracle/riesz_oracle.py, numpy/OpenBLAS on all host cores): each step
             times a bounded sample of real propagations at every level's dt and
             extrapolates to the full solve with the reference-equivalent counts
             (profiles/cfg2_reference_counts.json: identical control flow).
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

os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count() or 1))

import numpy as np  # noqa: E402

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)
from paper_1805_06688_b200.flops import FP16_MMA_SYNC_PEAK_TFLOPS, fmv, fmv_split16, fpc, fpc_dense  # noqa: E402

PROFILES = os.path.join(REPO, "profiles")
METRIC = "MGRIT fine-step space-time DOF/s (ndof*Nt / time-to-solution to 1e-8 residual)"
UNIT = "DOF/s"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    return ws, int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


def load_case(args):
    """The bench workload.  Strong scaling (default): the BASELINE config 2 problem split over the ranks.
    Weak scaling (option): 4096 fine steps PER GPU over a horizon T = N at the same step -- a different
    problem whose MGRIT iteration count grows with T (measured 21 / 30 / 90 for T = 1 / 2 / 8)."""
    from paper_1805_06688_b200.configs import make_case

    ws = dist_env()[0]
    if args.nt is None and ws > 1 and args.scaling == "weak":
        return make_case(args.config, Nt=make_case(args.config).tmesh.n_intervals * ws, T=float(ws))
    return make_case(args.config, Nt=args.nt)


def case_options(case, args):
    from paper_1805_06688_b200.mgrit import MgritOptions

    return MgritOptions(m=case.m, max_levels=case.max_levels, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol,
                        cg_preconditioner=args.precond)


def workload(case):
    T = float(case.tmesh.points[-1])
    per = f" (weak scaling: {int(round(T))} x the BASELINE horizon, T = {T:g}, same step)" if T != 1.0 else ""
    return {"workload": f"BASELINE configs[1] ({case.name}){per}: Riesz SFDE, {case.grid.nx}x{case.grid.ny} DOF, "
                        f"Nt={case.tmesh.n_intervals} uniform, beta={case.beta}, gamma={case.gamma}, "
                        f"Kx={case.kx}, Ky={case.ky}, multilevel MGRIT V-cycle m={case.m} FCF, CG tol "
                        f"{case.cg_rel_tol:g}, halt {case.halt_tol:g}",
            "ndof": case.grid.ndof, "nt": case.tmesh.n_intervals, "m": case.m,
            "l2": "inputs larger than L2: U, G and the residual copy are 528 MB each (no flush needed)"}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for name, flag in zip(names, parts[4:8]):
                if flag.lower() == "active":
                    reasons.add(name)
        load = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU reference leg
def reference_counts(case):
    """Reference-equivalent solve / CG counts of cfg2 (Nt = 4096); for the weak-scaled Nt = 4096 k the
    counts are scaled by k (solve counts grow linearly with Nt at a fixed MGRIT iteration count; the
    extra coarse level is not charged) and labelled as such."""
    path = os.path.join(PROFILES, f"{case.name}_reference_counts.json")
    n = case.tmesh.n_intervals
    if case.name != "cfg2" or n % 4096 or not os.path.exists(path):
        return None
    with open(path) as f:
        counts = json.load(f)
    k = n // 4096
    if k > 1:
        scale = lambda d: {key: v * k for key, v in d.items()}  # noqa: E731
        counts = dict(counts, setup=scale(counts["setup"]), levels=[scale(d) for d in counts["levels"]],
                      source=counts["source"] + f"; scaled x{k} for Nt = {n} (weak scaling)")
    return counts


def cpu_sample(case, counts, budget_s: float = 12.0):
    """Time real oracle propagations at each level's dt; extrapolate to one full solve.

    Returns (estimated time-to-solution in s, sample description, threads used).
    """
    from oracle import riesz_oracle as O

    prob = O.Problem(O.Grid(case.grid.mx, case.grid.my), case.tmesh.points, case.kx, case.ky, case.beta,
                     case.gamma, case.source, case.initial)
    levels = O.level_points(case.tmesh.points, case.m, case.max_levels)
    rng = np.random.default_rng(1)
    est = 0.0
    desc = []
    per_level_budget = budget_s / (len(levels) + 1)
    for li, pts in enumerate(levels):
        st = O.Stepper(O.Problem(prob.grid, pts, prob.kx, prob.ky, prob.beta, prob.gamma, prob.source,
                                 prob.initial), rel_tol=case.cg_rel_tol)
        dt = pts[1] - pts[0]
        t0 = time.perf_counter()
        nprop = 0
        applies = 0
        while time.perf_counter() - t0 < per_level_budget or nprop < 2:
            its0 = st.cg_its
            st.propagate(dt, rng.random(prob.grid.ndof))
            applies += (st.cg_its - its0) + 3  # explicit + initial residual + CG iterations + true residual
            nprop += 1
        t_apply = (time.perf_counter() - t0) / applies
        if li >= len(counts["levels"]):
            break  # weak-scaled runs have one more (tiny) coarse level than the counted cfg2 run
        c = counts["levels"][li]
        est += t_apply * (c["cg_iterations"] + 3 * c["solves"])
        if li == 0:
            est += t_apply * (counts["setup"]["cg_iterations"] + 2 * counts["setup"]["solves"])
        desc.append(f"L{li}: {nprop} propagations ({applies} applies, {t_apply * 1e3:.3f} ms/apply)")
    try:
        from threadpoolctl import threadpool_info

        threads = max((i.get("num_threads", 1) for i in threadpool_info() if i.get("internal_api") == "openblas"),
                      default=1)
    except Exception:
        threads = int(os.environ.get("OPENBLAS_NUM_THREADS", "1"))
    sample = ("oracle port (numpy/OpenBLAS) propagations at every level's dt: " + "; ".join(desc)
              + f"; extrapolated with reference-equivalent counts ({counts['source']})")
    return est, sample, threads


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    case = load_case(args)
    counts = reference_counts(case)
    if counts is None:
        print(json.dumps({"impl": "reference", "unavailable": "no reference-equivalent counts for this config"}))
        return 0
    work = case.grid.ndof * case.tmesh.n_intervals
    for _ in range(args.warmup):
        cpu_sample(case, counts, budget_s=2.0)
    vals = []
    t_run = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        est, sample, threads = cpu_sample(case, counts, budget_s=args.cpu_budget)
        t_run.append(time.perf_counter() - t0)
        vals.append(work / est)
    value = statistics.median(vals)
    tts = work / value
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tts * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic (canonical seeded recipe)",
        "config": workload(case),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                         "sample_wall_s": statistics.median(t_run), "extrapolated_tts_s": tts},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- GPU arm
def measure_fp64_peak():
    """cuBLAS DGEMM (torch.matmul float64, 8192^3) as the FP64 tensor roofline denominator."""
    import torch

    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b)
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2.0 * n**3 / (best * 1e-3) / 1e12


def ncu_traffic():
    path = os.path.join(PROFILES, "ncu_chain_summary.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d.get("launch")
    return None, None


def run_ours(args):
    import torch

    from paper_1805_06688_b200.engine import Engine
    from paper_1805_06688_b200.mgrit import solve
    from paper_1805_06688_b200.stepper import ProblemSpec

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    case = load_case(args)
    spec = ProblemSpec(**case.problem_kwargs())
    opts = case_options(case, args)
    work = case.grid.ndof * case.tmesh.n_intervals
    peak = measure_fp64_peak()
    eng = Engine.for_problem(case.grid, case.beta, case.gamma, case.kx, case.ky)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    iters = None
    for _ in range(args.warmup):
        _, tr = solve(spec, opts, device_result=True, engine=eng)
        iters = tr.iterations
    barrier()
    launches0 = eng.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        e0.record()
        for _ in range(args.steps):
            U, tr = solve(spec, opts, device_result=True, engine=eng)
        e1.record()
        barrier()
    launches = eng.launches - launches0
    ms = e0.elapsed_time(e1) / args.steps
    # one more (untimed) solve with per-launch CUDA events and counter snapshots: the chain kernel's
    # share of the step and its algorithmic FLOPs (roofline)
    eng.start_trace()
    solve(spec, opts, device_result=True, engine=eng)
    barrier()
    trace = eng.stop_trace()
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = work / (ms * 1e-3)  # whole job: one cfg2 problem, time axis sharded over the ranks

    # dominant kernel: the chain kernel (all rm_sweep_run launches)
    k_ms = sum(a.elapsed_time(b) for _, a, b, *_ in trace)
    mvs = sum(int((after - before)[2].item()) for _, _, _, before, after, _ in trace)
    pcs = sum(int((after - before)[3].item()) for _, _, _, before, after, _ in trace)
    mvs16 = sum(int((after - before)[4].item()) for _, _, _, before, after, _ in trace)
    # Algorithmic FLOPs: F_mv per operator apply -- whether it ran on FP64 DMMA or as a
    # split-FP16 product inside the PCG iteration -- and F_pc per tau application.  The roofline is the
    # FP64 tensor peak (the arithmetic the path is specified in); the chain kernel executes part of that
    # work on FP16 tensor cores, which the auxiliary "executed" fields account for separately: its
    # executed-FLOP time bound is F64/P64 + F16/P16 (mixed_bound_frac = bound / measured time).
    nx_, ny_ = case.grid.nx, case.grid.ny
    alg = (mvs + mvs16) * fmv(nx_, ny_, eng.flags) + pcs * fpc(nx_, ny_)
    achieved = alg / (k_ms * 1e-3) / 1e12
    lp = args.precond in ("tau", "tau16") and nx_ == ny_  # FP16 DST stages: square grids
    f64 = mvs * fmv(nx_, ny_, eng.flags) + (0.0 if lp else pcs * fpc(nx_, ny_))
    f16 = (pcs * fpc_dense(nx_, ny_) if lp else 0.0) + mvs16 * fmv_split16(nx_, ny_)
    t_bound = f64 / (peak * 1e12) + f16 / (FP16_MMA_SYNC_PEAK_TFLOPS * 1e12)
    traffic, traffic_launch = ncu_traffic()

    # end to end through the public API (host inputs, host result)
    # (one untimed call first: the public API's engine cache and the page-locked result block are
    # built once per process; each result is released before the next call, as a caller looping over
    # solves would)
    e2e_ms = []
    Uh, tr_h = solve(spec, opts)
    for _ in range(args.steps):
        Uh = None
        barrier()
        t0 = time.perf_counter()
        Uh, tr_h = solve(spec, opts)
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e = statistics.median(e2e_ms)
    if dist is not None:
        t = torch.tensor([e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = float(t.item())
    nlev = len(tr_h.residual_norms)
    ndof, N = case.grid.ndof, case.tmesh.n_intervals
    h2d = 8 * (2 * ndof + 2 * (N + 1) + 8 * (case.grid.nx + case.grid.ny))
    d2h = 8 * ((N + 1) * ndof + nlev * (N + 1))

    if rank == 0:
        cpu = None
        counts = reference_counts(case)
        if counts is not None and not args.no_cpu:
            est, sample, threads = cpu_sample(case, counts, budget_s=args.cpu_budget)
            cpu = {"value": work / est, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                   "extrapolated_tts_s": est}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (canonical seeded recipe, SURVEY.md §8d)",
            "config": dict(workload(case), mgrit_iterations=iters, cg_preconditioner=args.precond,
                           parallelism=(f"time slabs x{ws} (contiguous coarse intervals per rank, NCCL C-point "
                                        f"exchange, pipelined coarsest level)" if ws > 1 else "single GPU")),
            "e2e": {"value": work / (e2e * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches // args.steps,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "chain_kernel (fused PCG: FP64 DMMA block-Toeplitz applies for right-hand "
                                   "sides and true residuals, split-FP16 HMMA applies inside the iteration, tau "
                                   "DST stages on FP16 HMMA)",
                         "achieved_counts": "algorithmic FP64-equivalent FLOPs: F_mv per operator apply (FP64 or "
                                            "split-FP16), F_pc per tau application (flops.py)",
                         "peak_source": "cuBLAS DGEMM 8192^3 measured in this run (FP64 is not in "
                                        "MEASURED_PEAKS.json)",
                         "executed_fp64_flops_per_step": f64, "executed_fp16_flops_per_step": f16,
                         "fp16_peak": FP16_MMA_SYNC_PEAK_TFLOPS,
                         "fp16_peak_source": "legacy mma.sync FP16 (tools/lowp_peak.cu, profiles/r01_lowp_peak.txt)",
                         "mixed_bound_frac": t_bound / (k_ms * 1e-3),
                         "traffic_launch": traffic_launch,
                         "flops_per_apply": fmv(case.grid.nx, case.grid.ny, eng.flags), "fp64_applies_per_step": mvs,
                         "flops_per_precond": fpc(case.grid.nx, case.grid.ny),
                         "precond_applies_per_step": pcs,
                         "split_fp16_applies_per_step": mvs16,
                         "executed_flops_per_split_fp16_apply": fmv_split16(case.grid.nx, case.grid.ny),
                         "kernel_ms_per_step": k_ms},
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--scaling", choices=["weak", "strong"], default="strong",
                    help="N > 1: strong = the cfg2 problem split over the GPUs (default); weak = one cfg2-sized "
                         "slab of 4096 fine steps per GPU over a horizon T = N (a different, harder problem)")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--nt", type=int, default=None)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--precond", choices=["tau", "tau16", "tau64", "none"], default="tau",
                    help="inner CG: tau-preconditioned (default) or the reference's plain CG")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
