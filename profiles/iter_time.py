"""Time one pCG solve of a BASELINE config and report microseconds per iteration."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_05756_b200 as tb  # noqa: E402
from paper_2004_05756_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
kw = {}
if name.startswith("cfg3s"):
    prob = configs.cfg3(nx=96, ny=48, nz=48)
else:
    prob = getattr(configs, name)()
pc = os.environ.get("TB_PRECOND", "jacobi")
s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed,
                 tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=prob.rtol, preconditioner=pc)
psi = torch.as_tensor(prob.psi, device="cuda")
rho, _ = s.filtered_density_device(psi)
if os.environ.get("TB_MAXIT"):  # ablation timing: fixed iteration budget, results not meaningful
    s.maxit = int(os.environ["TB_MAXIT"])
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(2):
        a.record()
        try:
            s.pcg_device(rho, s._f_d)
        except Exception:
            pass
        b.record()
        torch.cuda.synchronize()
    print(f"{name} maxit={s.maxit} dbg={os.environ.get('TB_CGCG_DBG')}: {a.elapsed_time(b) * 1e3 / s.maxit:.3f} us/iteration")
    sys.exit(0)
for _ in range(2):
    s.pcg_device(rho, s._f_d)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
u = s.pcg_device(rho, s._f_d)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b)
print(f"{name} [{pc}]: pCG {ms:.3f} ms, {s.last_iterations} iterations, {ms * 1e3 / s.last_iterations:.3f} us/iteration, "
      f"J={float(s._f_d @ u):.10f}")
