"""Time HdmSolver.apply_device (tb_apply_stiffness) on a BASELINE config; for launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_05756_b200 as tb  # noqa: E402
from paper_2004_05756_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
prob = getattr(configs, name)()
s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed,
                 tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=prob.rtol)
rho = torch.as_tensor(prob.psi, device="cuda")
v = torch.randn(prob.mesh.n_dofs, dtype=torch.float64, device="cuda")
for mask in (True, False):
    for _ in range(3):
        s.apply_device(rho, v, mask_rows=mask)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        s.apply_device(rho, v, mask_rows=mask)
    b.record()
    torch.cuda.synchronize()
    print(f"{name} apply mask={mask}: {a.elapsed_time(b) / 20 * 1e3:.1f} us")
