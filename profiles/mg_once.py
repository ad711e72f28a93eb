"""Time the parts of one multigrid-preconditioned cfg 2 evaluation (filter, MG set-up + pCG,
sensitivity, adjoint) with CUDA events; under ncu, the last evaluation's launches.

    python profiles/mg_once.py [cfg2|cfg3] [n_evals]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2004_05756_b200 as tb  # noqa: E402
from paper_2004_05756_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
prob = getattr(configs, name)()
mat = tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP)
s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed, mat,
                 rtol=prob.rtol, preconditioner="mg")
obj = tb.ComplianceObjective(s.f)
psi = torch.as_tensor(prob.psi, device="cuda")
for it in range(n):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    ev[0].record()
    rho, _ = s.filtered_density_device(psi)
    ev[1].record()
    u = s.pcg_device(rho, s._f_d)
    ev[2].record()
    sens = s.sensitivity_device(rho, u, u)
    ev[3].record()
    g = s.filter.apply_adjoint_device(sens)
    ev[4].record()
    torch.cuda.synchronize()
    parts = [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]
    print(f"eval {it}: filter {parts[0]:.3f} ms, mg+pcg {parts[1]:.3f} ms ({s.last_iterations} its), "
          f"sens {parts[2]:.3f} ms, adjoint {parts[3]:.3f} ms, total {sum(parts):.3f} ms", flush=True)
