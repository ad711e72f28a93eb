"""Per-phase %globaltimer sums of k_mg_gj_inverse (TB_GJ_PROF build, CTAs 0 and 100): one cfg 2
multigrid evaluation after a warm-up."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2004_05756_b200 as tb
from paper_2004_05756_b200 import _lib, configs
prob = configs.cfg2()
s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed,
                 tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=prob.rtol, preconditioner="mg")
psi = torch.as_tensor(prob.psi, device="cuda")
obj = tb.ComplianceObjective(s.f)
s.solve(psi, obj)
buf = (ctypes.c_ulonglong * 16)()
_lib.lib().tb_gj_prof_read(buf)
s.solve(psi, obj)
torch.cuda.synchronize()
_lib.lib().tb_gj_prof_read(buf)
names = ["issue", "Pinv", "wait", "sync1", "Gm+R", "sync2", "update", "gridbar"]
for c in range(2):
    print("cta", (0, 100)[c], " ".join(f"{names[k]}={buf[c * 8 + k] / 1e3:.1f}us" for k in range(8)))
