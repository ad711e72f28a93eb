"""3D multigrid with the in-house Gauss-Jordan coarsest inverse vs cuSOLVER (TB_MG_CUSOLVER=1):
cfg 3 evaluation time, iterations, J."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2004_05756_b200 as tb
from paper_2004_05756_b200 import configs
dev = torch.device("cuda", 0)
prob = configs.cfg3(prefilter=lambda mesh, p0: tb.HelmholtzFilter(mesh, 2.0).apply(torch.as_tensor(p0, device=dev)).rho.cpu().numpy())
s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed,
                 tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=prob.rtol, preconditioner="mg")
obj = tb.ComplianceObjective(s.f)
psi = torch.as_tensor(prob.psi, device=dev)
for _ in range(2):
    sol = s.solve(psi, obj); s.gradient(psi, sol, obj)
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); sol = s.solve(psi, obj); g = s.gradient(psi, sol, obj); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(json.dumps({"cusolver": bool(os.environ.get("TB_MG_CUSOLVER")), "ms": sorted(ts)[2], "iters": sol.iterations, "J": sol.j}))
