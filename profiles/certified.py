"""Certified error bound (sigma_min) at cfg2: shift-invert Lanczos vs inverse power iteration."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2004_05756_b200 as tb  # noqa: E402
from paper_2004_05756_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
pc = sys.argv[2] if len(sys.argv) > 2 else "jacobi"
prob = getattr(configs, name)()
s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed,
                 tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=prob.rtol, preconditioner=pc)
obj = tb.ComplianceObjective(s.f)
snaps = [np.where(s.free_mask, s.solve(d, obj).u, 0.0) for d in prob.rom_designs[:4]]
phi = tb.gram_schmidt(snaps)
basis = tb.ReducedBasis(phi, None, None, phi.T @ s.f)
rom = tb.RomModel(s)
rho, _ = s.filtered_density(prob.psi)
rs = rom.solve(basis, rho, obj)
for method in ("lanczos", "power"):
    n0 = s.stats.factorizations
    c0 = [0]
    orig = s.pcg_device

    def counted(*a, **k):
        c0[0] += 1
        return orig(*a, **k)
    s.pcg_device = counted
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = rom.error_bounds(basis, rho, rs, obj, mode="certified", method=method)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    s.pcg_device = orig
    print(f"{name} [{pc}] {method:8s}: sigma_min {rep.sigma_min:.10e} converged {rep.sigma_min_converged} "
          f"solves {c0[0]} time {dt:.3f} s")
