import sys, time, torch
sys.path.insert(0,'/root/repo')
from paper_1805_06688_b200.configs import make_case
from paper_1805_06688_b200.mgrit import MgritOptions, solve
from paper_1805_06688_b200.stepper import ProblemSpec
case = make_case("cfg3"); spec = ProblemSpec(**case.problem_kwargs())
for tol in (1e-12, 1e-13, 1e-12, 1e-13):
    opts = MgritOptions(m=case.m, halt_tol=case.halt_tol, cg_rel_tol=tol)
    torch.cuda.synchronize(); t=time.perf_counter()
    U, tr = solve(spec, opts, device_result=True)
    torch.cuda.synchronize(); print(tol, tr.iterations, time.perf_counter()-t, tr.cg_iterations[-1], flush=True)
