"""GPU parity at BASELINE cfg 2 full size (600x200, 241,602 DOF) against the reference's own
run (golden_cfg2.npz: scalars + strided samples), plus size-independent identities."""

import numpy as np
import pytest

import paper_2004_05756_b200 as tb
from conftest import golden
from paper_2004_05756_b200 import configs

pytestmark = pytest.mark.gpu


def test_cfg2_hdm_and_rom_vs_reference(cuda):
    G = golden("golden_cfg2.npz")
    prob = configs.cfg2()
    s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed,
                     tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=prob.rtol)
    obj = tb.ComplianceObjective(s.f)
    sol = s.solve(prob.psi, obj)
    g = s.gradient(prob.psi, sol, obj)
    sens = s.element_sensitivity(sol.rho, sol.u, sol.lam, obj)
    se, su = int(G["stride_e"]), int(G["stride_u"])
    assert abs(sol.j - float(G["j"])) <= 1e-8 * abs(float(G["j"]))
    assert np.max(np.abs(sol.rho[::se] - G["rho_s"]) / G["rho_s"]) <= 1e-6
    assert abs(sol.rho.sum() - float(G["rho_sum"])) <= 1e-10 * float(G["rho_sum"])
    assert np.abs(sol.u[::su] - G["u_s"]).max() <= 1e-6 * np.abs(G["u_s"]).max()
    assert np.abs(sens[::se] - G["s_s"]).max() <= 1e-6 * float(G["s_inf"])
    assert np.abs(g[::se] - G["g_s"]).max() <= 1e-6 * float(G["g_inf"])
    # identities: compliance = u^T K u ; sum(-s rho)/p ~ J (alpha ~ rho^p with rho_l = 1e-9)
    ku = s.apply_stiffness(sol.rho, sol.u)
    assert abs(sol.u @ ku - sol.j) <= 1e-9 * sol.j
    assert abs(np.sum(-sens * sol.rho) / 3.0 - sol.j) <= 1e-6 * sol.j
    # ROM k = 32 chain (same snapshot recipe)
    snaps = [np.where(s.free_mask, s.solve(d, obj).u, 0.0) for d in prob.rom_designs]
    phi = tb.gram_schmidt(snaps)
    assert phi.shape[1] == int(G["rom_kept"])
    basis = tb.ReducedBasis(phi, None, None, phi.T @ s.f)
    rom = tb.RomModel(s)
    kh = rom.reduced_stiffness(basis, sol.rho)
    ref = G["rom_k_hat"]
    assert np.linalg.norm(kh - ref) <= 1e-6 * np.linalg.norm(ref)
    rs = rom.solve(basis, sol.rho, obj)
    assert abs(rs.j - float(G["rom_j"])) <= 1e-8 * abs(float(G["rom_j"]))
    assert abs(rs.residual_norm - float(G["rom_residual"])) <= 1e-6 * float(G["rom_residual"])


def test_cfg2_full_fields_vs_oracle(cuda):
    """Every entry of rho, u, s and g at full cfg 2 size against the CPU oracle (oracle/hdm.py,
    SuperLU; pinned to the reference by golden_cfg1.npz in full and golden_cfg2.npz's samples),
    not only the strided samples of the reference run."""
    from oracle.fem import build_grid
    from oracle.hdm import Filter, Hdm, Material

    prob = configs.cfg2()
    s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed,
                     tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=prob.rtol)
    obj = tb.ComplianceObjective(s.f)
    sol = s.solve(prob.psi, obj)
    g = s.gradient(prob.psi, sol, obj)
    sens = s.element_sensitivity(sol.rho, sol.u, sol.lam, obj)
    grid = build_grid(600, 200, 1.0)
    ora = Hdm(grid, prob.k_e, Filter(grid, prob.radius), prob.f, prob.fixed, Material(configs.RHO_L, configs.P_SIMP))
    ref = ora.solve(prob.psi)
    g_ref = ora.gradient(ref)
    s_ref = ora.element_sensitivity(ref["rho"], ref["u"], ref["lam"])
    assert abs(sol.j - ref["j"]) <= 1e-8 * abs(ref["j"])
    assert np.max(np.abs(sol.rho - ref["rho"]) / ref["rho"]) <= 1e-6          # element-wise
    assert np.linalg.norm(sol.u - ref["u"]) <= 1e-6 * np.linalg.norm(ref["u"])
    assert np.linalg.norm(sens - s_ref) <= 1e-6 * np.linalg.norm(s_ref)
    assert np.linalg.norm(g - g_ref) <= 1e-6 * np.linalg.norm(g_ref)
    assert np.abs(g - g_ref).max() <= 1e-6 * np.abs(g_ref).max()
