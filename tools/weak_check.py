import sys, time, torch
sys.path.insert(0, '.')
from paper_1805_06688_b200.configs import make_case
from paper_1805_06688_b200.mgrit import MgritOptions, solve
from paper_1805_06688_b200.stepper import ProblemSpec
for k in (2, 8):
    case = make_case("cfg2", Nt=4096 * k, T=float(k) if len(sys.argv) > 1 else 1.0)
    spec = ProblemSpec(**case.problem_kwargs())
    opts = MgritOptions(m=case.m, max_levels=case.max_levels, halt_tol=case.halt_tol, cg_rel_tol=case.cg_rel_tol)
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        U, tr = solve(spec, opts, device_result=True)
        torch.cuda.synchronize(); t = time.perf_counter() - t0
    print(f"Nt={4096*k} T={k}: iters={tr.iterations} TTS={t:.3f}s per-4096-block={t/k:.3f}s res={tr.residual_norms[-1]:.2e}", flush=True)
