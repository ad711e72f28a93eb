"""Per-phase time of the persistent 2D multigrid pCG (needs tools/libtopo_mgprof.so from
tools/build_prof.sh; run with TB_LIB_PATH=tools/libtopo_mgprof.so).

    TB_LIB_PATH=tools/libtopo_mgprof.so python profiles/mg_prof.py [cfg1|cfg2]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_05756_b200 as tb  # noqa: E402
from paper_2004_05756_b200 import _lib, configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
prob = getattr(configs, name)()
s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed,
                 tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=prob.rtol, preconditioner="mg")
psi = torch.as_tensor(prob.psi, device="cuda")
rho, _ = s.filtered_density_device(psi)
buf = (ctypes.c_ulonglong * 32)()
for rep in range(3):
    _lib.lib().tb_mgp_prof_read(buf)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    s.pcg_device(rho, s._f_d)
    b.record()
    torch.cuda.synchronize()
    _lib.lib().tb_mgp_prof_read(buf)
    its = s.last_iterations
    names = {0: "A (p, Kp, p.q)", 1: "B (x, r, r.r, sweep 1)", 3: "coarsest (restriction, dense solve)",
             16: "level 0 up (prolong, 2 sweeps, r.z)"}
    names.update({8 + l: f"level {l} down" for l in range(8)})
    names.update({16 + l: f"level {l} up" for l in range(1, 8)})
    tot = sum(buf[k] for k in range(31))
    print(f"rep {rep}: solve {a.elapsed_time(b):.3f} ms, {its} iterations, {buf[31]} launches, "
          f"kernel-timed {tot / 1e6:.3f} ms")
    for k in range(31):
        if buf[k]:
            print(f"   {names.get(k, k):40s} {buf[k] / 1e3 / max(its, 1):8.2f} us/iteration")
