"""A/B check of the 3D Jacobi-pCG paths (run with and without TB_NO_SWEEP=1): small grids
against the oracle's direct solve, cfg 3 timing / iterations / J, per-iteration kernel time."""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2004_05756_b200 as tb  # noqa: E402
from oracle.fem import build_grid  # noqa: E402
from oracle.hdm import Filter, Hdm, Material  # noqa: E402
from paper_2004_05756_b200 import _lib, configs  # noqa: E402

MAT = tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP)
out = {"sweep": os.environ.get("TB_NO_SWEEP", "0") in ("", "0")}
for dims in [(8, 4, 4), (12, 6, 5), (40, 10, 7), (70, 16, 9)]:
    prob = configs.cfg3(seed=3, nx=dims[0], ny=dims[1], nz=dims[2])
    s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed, MAT, rtol=1e-10)
    obj = tb.ComplianceObjective(s.f)
    sol = s.solve(prob.psi, obj)
    g = build_grid(*dims[:2], 1.0, nz=dims[2])
    ora = Hdm(g, prob.k_e, Filter(g, prob.radius), prob.f, prob.fixed, Material(configs.RHO_L, configs.P_SIMP))
    ref = ora.solve(prob.psi)
    out[str(dims)] = {"path": int(_lib.lib().tb_pcg_path(s._plan)), "iters": sol.iterations,
                      "J_rel": abs(sol.j - ref["j"]) / abs(ref["j"]),
                      "u_rel": float(np.abs(sol.u - ref["u"]).max() / np.abs(ref["u"]).max())}
dev = torch.device("cuda", 0)


def prefilter(mesh, psi0):
    return tb.HelmholtzFilter(mesh, 2.0).apply(torch.as_tensor(psi0, device=dev)).rho.cpu().numpy()


prob = configs.cfg3(prefilter=prefilter)
s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed, MAT,
                 rtol=prob.rtol)
obj = tb.ComplianceObjective(s.f)
psi = torch.as_tensor(prob.psi, device=dev)
rho, _ = s.filtered_density_device(psi)
s.pcg_device(rho, s._f_d)
torch.cuda.synchronize()
t0 = time.perf_counter()
u = s.pcg_device(rho, s._f_d)
torch.cuda.synchronize()
out["cfg3_solve_s"] = time.perf_counter() - t0
out["cfg3_iters"] = s.last_iterations
out["cfg3_relres"] = s.last_relres
out["cfg3_J"] = float(s._f_d @ u)
msf, msu = ctypes.c_double(0), ctypes.c_double(0)
_lib.check(_lib.lib().tb_pcg_profile(s._plan, _lib.ptr(rho), _lib.ptr(s._f_d), 50, ctypes.byref(msf), ctypes.byref(msu),
                                     _lib.stream_ptr(dev)), "profile")
out["us_iter_kernelA"] = msf.value * 1e3
out["us_iter_kernelB"] = msu.value * 1e3
print(json.dumps(out))
