"""cfg 3 (192x96x96 Hex8): a handful of single-sweep Jacobi-pCG iterations via tb_pcg_profile
(the per-iteration kernel alone), for ncu captures of k_hex8_cg."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_05756_b200 as tb  # noqa: E402
from paper_2004_05756_b200 import _lib, configs  # noqa: E402

dev = torch.device("cuda", 0)
prob = configs.cfg3()  # raw U[0.01,1] design (the pre-filter does not change the kernel's work)
s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed,
                 tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=prob.rtol)
rho = torch.as_tensor(prob.psi, device=dev)
msf, msu = ctypes.c_double(0), ctypes.c_double(0)
n = int(os.environ.get("NREP", "6"))
_lib.check(_lib.lib().tb_pcg_profile(s._plan, _lib.ptr(rho), _lib.ptr(s._f_d), n, ctypes.byref(msf), ctypes.byref(msu),
                                     _lib.stream_ptr(dev)), "profile")
print(f"path={_lib.lib().tb_pcg_path(s._plan)} us/iter={msf.value * 1e3:.1f} update={msu.value * 1e3:.1f}")
