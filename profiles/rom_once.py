"""cfg 5: build the k = 64 basis and run the 16-design ROM step (solve_batch) NREP times --
for ncu launch lists / captures of k_rom_fused."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2004_05756_b200 as tb  # noqa: E402
from paper_2004_05756_b200 import configs  # noqa: E402

dev = torch.device("cuda", 0)
prob = configs.cfg5()
m = prob.mesh
s = tb.HdmSolver(m, prob.k_e, tb.HelmholtzFilter(m, prob.radius), prob.f, prob.fixed,
                 tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP))
cols = configs.phi_columns(m, prob.rom_k, seed=0, xp=torch, device=dev)
cols[:, torch.as_tensor(~s.free_mask, device=dev)] = 0.0
phi = tb.gram_schmidt(list(cols))
del cols
basis = tb.ReducedBasis(phi, None, None, phi.T @ s._f_d)
rom = tb.RomModel(s)
rhos = torch.as_tensor(np.stack(prob.rom_designs), device=dev)
for _ in range(int(os.environ.get("NREP", "2"))):
    khat, uhat, norms = rom.solve_batch(basis, rhos)
torch.cuda.synchronize()
print("norm0", norms[0])
