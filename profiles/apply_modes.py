"""cfg 3: one Jacobi solve (its true-residual check runs k_hex8_cg<1>, the pitched TMA apply) and
three apply_stiffness calls (k_hex8, user layout); for an ncu capture of the two apply kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2004_05756_b200 as tb  # noqa: E402
from paper_2004_05756_b200 import configs  # noqa: E402

prob = configs.cfg3()
s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed,
                 tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=prob.rtol)
psi = torch.as_tensor(prob.psi, device="cuda")
sol = s.solve(psi, tb.ComplianceObjective(s.f))
print("J", sol.j)
v = torch.randn(prob.mesh.n_dofs, dtype=torch.float64, device="cuda")
for _ in range(3):
    s.apply_device(psi, v)
torch.cuda.synchronize()
