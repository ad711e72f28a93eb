"""Break one trust-region inner step (cfg2, k=32) into its parts."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_05756_b200 as tb  # noqa: E402
from paper_2004_05756_b200 import configs  # noqa: E402

prob = configs.cfg2()
s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed,
                 tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=prob.rtol)
obj = tb.ComplianceObjective(s.f)
psi = (0.9 * torch.as_tensor(prob.psi, device="cuda")).clamp(0, 1)
n_u, k = prob.mesh.n_dofs, 32
phi = torch.linalg.qr(torch.randn(n_u, k, dtype=torch.float64, device="cuda"))[0].contiguous()
basis = tb.ReducedBasis(phi, None, None, phi.T @ s._f_d)
rom = tb.RomModel(s)
w = torch.ones(prob.mesh.n_elems, dtype=torch.float64, device="cuda")
opt = tb.MmaOptimizer(torch.zeros_like(w), torch.ones_like(w), w, float(w @ psi) * 1.05)
sol = s.solve(psi, obj)
g = s.gradient(psi, sol, obj)


def timed(name, fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        out = fn()
    b.record()
    torch.cuda.synchronize()
    print(f"{name:28s} {a.elapsed_time(b) / reps:8.3f} ms")
    return out


x = timed("mma step", lambda: opt.step(psi, 0.0, g))
rho = timed("filtered_density", lambda: s.filtered_density_device(x)[0])
timed("rom.solve(grad)", lambda: rom.solve(basis, rho, obj, compute_gradient=True))
timed("rom.solve", lambda: rom.solve(basis, rho, obj))
timed("reduced_stiffness", lambda: rom.reduced_stiffness_device(basis, rho))
timed("filter adjoint", lambda: s.filter.apply_adjoint_device(rho))
