import sys, numpy as np, torch
sys.path.insert(0,'/root/repo')
from oracle import riesz_oracle as O
from paper_1805_06688_b200.configs import make_case
from paper_1805_06688_b200.engine import Engine
case = make_case("cfg3", Nt=8); g = case.grid
eng = Engine.for_problem(g, case.beta, case.gamma, case.kx, case.ky)
ops = O.Operators(O.Grid(g.mx, g.my), case.kx, case.ky, case.beta, case.gamma)
rng=np.random.default_rng(0)
V = rng.standard_normal((3, g.ndof))
for dt in (0.0, 1e-4, 1.0):
    got = eng.apply_probe(torch.from_numpy(V).cuda(), torch.full((3,), dt, dtype=torch.float64).cuda()).cpu().numpy()
    for k in range(1):
        ref = ops.step_apply(dt, +1, V[k]) if dt > 0 else ops.mass(V[k])
        d = (got[k]-ref).reshape(g.ny, g.nx)
        print(dt, 'rel', np.linalg.norm(d)/np.linalg.norm(ref), 'rows with err', np.nonzero(np.abs(d).max(1) > 1e-9*np.abs(ref).max())[0][:20], 'cols', np.nonzero(np.abs(d).max(0) > 1e-9*np.abs(ref).max())[0][:20])
