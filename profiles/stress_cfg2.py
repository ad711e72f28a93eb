"""Repeat the cfg2 Jacobi-pCG solve N times (hang / determinism stress for the persistent kernel)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_05756_b200 as tb  # noqa: E402
from paper_2004_05756_b200 import configs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
prob = configs.cfg2()
s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed,
                 tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=prob.rtol)
psi = torch.as_tensor(prob.psi, device="cuda")
rho, _ = s.filtered_density_device(psi)
ref = s.pcg_device(rho, s._f_d).clone()
t0 = time.time()
for k in range(n):
    u = s.pcg_device(rho, s._f_d)
    assert torch.equal(u, ref), f"solve {k} not bit-identical"
torch.cuda.synchronize()
print(f"stress: {n} cfg2 solves bit-identical in {time.time() - t0:.1f} s")
