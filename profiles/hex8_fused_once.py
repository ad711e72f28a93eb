"""Launch the fused Hex8 pCG kernel (k_hex8<FUSED>) and the update kernel outside the
conditional graph via tb_pcg_profile, so ncu can capture them (graph kernel nodes with
conditional nodes are not profiled)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_05756_b200 as tb  # noqa: E402
from paper_2004_05756_b200 import _lib, configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
prob = getattr(configs, name)()
s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed,
                 tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=prob.rtol)
rho = torch.as_tensor(prob.psi, device="cuda")
msf, msu = ctypes.c_double(0.0), ctypes.c_double(0.0)
nrep = int(os.environ.get("TB_NREP", "3"))
_lib.check(_lib.lib().tb_pcg_profile(s._plan, _lib.ptr(rho), _lib.ptr(s._f_d), nrep, ctypes.byref(msf),
                                     ctypes.byref(msu), _lib.stream_ptr(rho.device)), "profile")
torch.cuda.synchronize()
print(f"{name}: fused operator {msf.value * 1e3:.1f} us, update {msu.value * 1e3:.1f} us")
