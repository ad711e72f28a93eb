import sys, os, numpy as np, json
sys.path.insert(0, os.environ.get('GRAFT_REPO_ROOT', '/root/repo'))
import paper_2004_05756_b200 as tb
from paper_2004_05756_b200 import configs
from oracle.fem import build_grid
from oracle.hdm import Filter, Hdm, Material
prob = configs.cfg1(seed=7, nx=400, ny=17)
mat = tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP)
grid = build_grid(400, 17, 1.0)
ora = Hdm(grid, prob.k_e, Filter(grid, prob.radius), prob.f, prob.fixed, Material(configs.RHO_L, configs.P_SIMP))
ref = ora.solve(prob.psi); gref = ora.gradient(ref)
out = {}
for pc in ["mg", "jacobi"]:
    for rtol in [None, 1e-10, 1e-8]:
        s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed, mat, rtol=rtol, preconditioner=pc)
        obj = tb.ComplianceObjective(s.f)
        try:
            sol = s.solve(prob.psi, obj); g = s.gradient(prob.psi, sol, obj)
            out[f"{pc} {rtol}"] = dict(J=abs(sol.j-ref['j'])/abs(ref['j']), g=float(np.linalg.norm(g-gref)/np.linalg.norm(gref)), it=sol.iterations, relres=sol.relres)
        except Exception as e:
            out[f"{pc} {rtol}"] = repr(e)[:150]
print(json.dumps(out, indent=1))
