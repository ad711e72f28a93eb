import gc, sys, os, time
sys.path.insert(0, '/root/repo')
import torch
import paper_2004_05756_b200 as tb
from paper_2004_05756_b200 import configs
prob = configs.cfg2()
s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed,
                 tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=prob.rtol)
obj = tb.ComplianceObjective(s.f)
psi = torch.as_tensor(prob.psi, device="cuda")
for mode in ("gc-on", "gc-off", "gc-on"):
    if mode == "gc-off": gc.disable()
    else: gc.enable()
    for _ in range(3):
        sol = s.solve(psi, obj); s.gradient(psi, sol, obj)
    torch.cuda.synchronize()
    ms = []
    for k in range(8):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(); sol = s.solve(psi, obj); g = s.gradient(psi, sol, obj); b.record()
        torch.cuda.synchronize()
        ms.append((round(a.elapsed_time(b), 1), round((time.perf_counter() - t0) * 1e3, 1), sol.iterations))
    print(mode, ms)
