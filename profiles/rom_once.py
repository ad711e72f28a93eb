"""One cfg-5 reduced-stiffness evaluation (k = 64, one design) for ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2004_05756_b200 as tb  # noqa: E402
from paper_2004_05756_b200 import configs  # noqa: E402

scale = sys.argv[1] if len(sys.argv) > 1 else "full"
prob = configs.cfg5(n_designs=2) if scale == "full" else configs.cfg5(nx=64, ny=32, nz=32, n_designs=2)
m = prob.mesh
s = tb.HdmSolver(m, prob.k_e, tb.HelmholtzFilter(m, prob.radius), prob.f, prob.fixed,
                 tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP))
dev = torch.device("cuda", 0)
phi = torch.linalg.qr(torch.randn(m.n_dofs, 64, dtype=torch.float64, device=dev))[0].contiguous()
basis = tb.ReducedBasis(phi, None, None, phi.T @ s._f_d)
rho = torch.as_tensor(np.stack(prob.rom_designs), device=dev)
rom = tb.RomModel(s)
for _ in range(2):
    kh = rom.reduced_stiffness_device(basis, rho[0])
torch.cuda.synchronize()
print("khat norm", float(torch.linalg.norm(kh)))
