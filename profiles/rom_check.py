"""Reduced stiffness on 3D Hex8 plans: the element-form DMMA kernel (k_rom_fused) against the
oracle's element form (reference rom.py:254-262) on small grids, and the cfg 5 timing (run with
and without TB_NO_ROM_FUSED=1)."""
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
from oracle.rom import Rom  # noqa: E402
from paper_2004_05756_b200 import configs  # noqa: E402

MAT = tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP)
dev = torch.device("cuda", 0)
out = {"fused": os.environ.get("TB_NO_ROM_FUSED", "0") in ("", "0")}
for dims, k in [((8, 4, 4), 10), ((9, 5, 3), 16), ((13, 6, 5), 64), ((12, 6, 5), 9)]:
    prob = configs.cfg3(seed=2, nx=dims[0], ny=dims[1], nz=dims[2])
    s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed, MAT)
    g = build_grid(*dims[:2], 1.0, nz=dims[2])
    ora = Rom(Hdm(g, prob.k_e, Filter(g, prob.radius), prob.f, prob.fixed, Material(configs.RHO_L, configs.P_SIMP)))
    rng = np.random.default_rng(k)
    phi = np.linalg.qr(rng.standard_normal((prob.mesh.n_dofs, k)))[0]
    phi[~s.free_mask] = 0.0
    rhos = [np.clip(prob.psi * (1 + rng.uniform(-0.05, 0.05, prob.psi.size)), 0.01, 1.0) for _ in range(3)]
    basis = tb.ReducedBasis(phi, None, None, phi.T @ s.f)
    kh = tb.RomModel(s).reduced_stiffness_device(basis, torch.as_tensor(np.stack(rhos), device=dev)).cpu().numpy()
    errs = []
    for d in range(3):
        ref = ora.reduced_stiffness_elemform(phi, rhos[d])
        errs.append(float(np.linalg.norm(kh[d] - ref) / np.linalg.norm(ref)))
    out[f"{dims} k={k}"] = max(errs)

prob = configs.cfg5()
m = prob.mesh
s = tb.HdmSolver(m, prob.k_e, tb.HelmholtzFilter(m, prob.radius), prob.f, prob.fixed, MAT)
cols = configs.phi_columns(m, prob.rom_k, seed=0, xp=torch, device=dev)
cols[:, torch.as_tensor(~s.free_mask, device=dev)] = 0.0
phi = tb.gram_schmidt(list(cols))
del cols
basis = tb.ReducedBasis(phi, None, None, phi.T @ s._f_d)
rom = tb.RomModel(s)
rhos = torch.as_tensor(np.stack(prob.rom_designs), device=dev)
for _ in range(2):
    kh = rom.reduced_stiffness_device(basis, rhos)
torch.cuda.synchronize()
ts = []
for _ in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    kh = rom.reduced_stiffness_device(basis, rhos)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
out["cfg5_khat16_ms"] = min(ts)
for _ in range(2):
    rom.solve_batch(basis, rhos)
torch.cuda.synchronize()
t0 = time.perf_counter()
khat, uhat, norms = rom.solve_batch(basis, rhos)
torch.cuda.synchronize()
out["cfg5_step_ms"] = (time.perf_counter() - t0) * 1e3
out["cfg5_khat0_trace"] = float(torch.trace(kh[0]))
out["cfg5_norm0"] = norms[0]
np.save("gpurun_out/khat_cfg5_%s.npy" % ("fused" if out["fused"] else "old"), kh.cpu().numpy())
print(json.dumps(out))
