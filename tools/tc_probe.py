import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_1805_06688_b200.configs import make_case
from paper_1805_06688_b200.engine import Engine
from paper_1805_06688_b200.precond import dst_matrix, tau_diagonals
case = make_case("cfg3", Nt=8)
g = case.grid
eng = Engine.for_problem(g, case.beta, case.gamma, case.kx, case.ky)
dm, dk = tau_diagonals(g, case.beta, case.gamma, case.kx, case.ky)
S = dst_matrix(g.nx)
rng = np.random.default_rng(0)
V = rng.standard_normal((3, g.ndof))
dts = np.array([1/16384, 1/1024, 1/4])
for mode in ("tau64", "tau"):
    got = eng.precond_apply(torch.from_numpy(V).cuda(), torch.from_numpy(dts).cuda(), mode).cpu().numpy()
    for b in range(3):
        d = dm + 0.5 * dts[b] * dk
        R = V[b].reshape(g.ny, g.nx)
        ref = (S @ ((S @ R @ S) / d.reshape(g.ny, g.nx)) @ S).reshape(-1)
        print(mode, b, np.linalg.norm(got[b] - ref) / np.linalg.norm(ref))
