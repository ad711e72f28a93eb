"""Where the numpy-API (e2e) evaluation spends time beyond the device-resident one (argv[1]:
cfg2 multigrid, default, or cfg3 Jacobi: the headline)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2004_05756_b200 as tb  # noqa: E402
from paper_2004_05756_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
prob = getattr(configs, name)()
s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed,
                 tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=prob.rtol,
                 preconditioner="mg" if name == "cfg2" else "jacobi")
obj = tb.ComplianceObjective(s.f)
psi_h = np.ascontiguousarray(prob.psi)
psi_d = torch.as_tensor(psi_h, device="cuda")


def wall(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3, out


t, sol_d = wall(lambda: s.solve(psi_d, obj))
print(f"solve(device)            {t:8.3f} ms")
t, sol_h = wall(lambda: s.solve(psi_h, obj))
print(f"solve(numpy)             {t:8.3f} ms")
t, _ = wall(lambda: s.gradient(psi_d, sol_d, obj))
print(f"gradient(device)         {t:8.3f} ms")
t, _ = wall(lambda: s.gradient(psi_h, sol_h, obj))
print(f"gradient(numpy)          {t:8.3f} ms")
t, _ = wall(lambda: sol_h.psi_hash)
print(f"psi_hash                 {t:8.3f} ms")
t, _ = wall(lambda: torch.as_tensor(psi_h, device="cuda"))
print(f"H2D psi                  {t:8.3f} ms")
u = sol_d.u
t, _ = wall(lambda: u.cpu().numpy())
print(f"D2H u                    {t:8.3f} ms")
