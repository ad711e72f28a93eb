"""One HDM evaluation (solve + gradient) of a BASELINE config, for ncu launch lists / captures.

    python profiles/run_once.py [cfg2|cfg3-small|cfg3] [n_evals]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2004_05756_b200 as tb  # noqa: E402
from paper_2004_05756_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
if name == "cfg2":
    prob = configs.cfg2()
elif name == "cfg3-small":
    prob = configs.cfg3(nx=48, ny=24, nz=24)
else:
    prob = configs.cfg3()
s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed,
                 tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=prob.rtol)
obj = tb.ComplianceObjective(s.f)
psi = torch.as_tensor(prob.psi, device="cuda")
for _ in range(n):
    sol = s.solve(psi, obj)
    g = s.gradient(psi, sol, obj)
torch.cuda.synchronize()
print(f"{name}: J={sol.j:.10f} iters={sol.iterations}")
