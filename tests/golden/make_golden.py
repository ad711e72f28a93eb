"""Generate golden fixtures by running the REFERENCE package itself (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--with-cfg2]

Inputs come from paper_2004_05756_b200.configs (seeded, host numpy); outputs come from the
reference's public API (romtopt.fem / filtering / hdm / rom).  The resulting .npz files are
committed; nothing at test or bench time reads /root/reference.

Files:
  golden_cfg1.npz   BASELINE cfg 1 (120x40): rho, phi, u, J, s, g, K(rho)v, ROM k=10 chain
  golden_small.npz  reference test-fixture problems (cantilever 6x2 / 12x4 / 4x2, filters)
  golden_cfg2.npz   BASELINE cfg 2 (600x200): scalars + strided samples (needs --with-cfg2)
  ref3d_small.npz   reference HdmSolver / RomModel run on a duck-typed Hex8 mesh (6x3x3)
  ref3d_medium.npz  the same at 20x10x10 (7,623 dofs)
  golden_mma.npz    reference MmaOptimizer trajectories (box + volume bound, move caps)
  golden_subproblem.npz  reference TrustRegionDriver.solve_subproblem on a 48x16 half-MBB
"""

from __future__ import annotations

import os
import sys
import time
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from romtopt.fem import build_mesh, elasticity_element_matrix  # noqa: E402
from romtopt.filtering import HelmholtzFilter  # noqa: E402
from romtopt.hdm import ComplianceObjective, HdmSolver, MaterialModel  # noqa: E402
from romtopt.rom import ReducedBasis, RomModel, gram_schmidt, pod  # noqa: E402

from paper_2004_05756_b200 import configs  # noqa: E402

MAT = MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP)


def ref_problem(prob):
    mesh = build_mesh(prob.mesh.nx, prob.mesh.ny, prob.mesh.h)
    filt = HelmholtzFilter(mesh, prob.radius)
    solver = HdmSolver(mesh, elasticity_element_matrix(configs.E0, configs.NU), filt, prob.f, prob.fixed, MAT)
    return mesh, filt, solver


def rom_chain(mesh, solver, prob, psi_eval):
    """Snapshot solves at the ROM designs -> masked -> gram_schmidt -> basis -> solve at psi_eval."""
    obj = ComplianceObjective(solver.f)
    snaps = []
    for d in prob.rom_designs:
        u = solver.solve(d, obj).u
        snaps.append(np.where(solver.free_mask, u, 0.0))
    phi = gram_schmidt(snaps)
    basis = ReducedBasis(phi=phi, elem_phi=phi[mesh.elem_dofs], elem_k_phi=np.matmul(solver.k_e, phi[mesh.elem_dofs]),
                         f_hat=phi.T @ solver.f)
    rom = RomModel(solver)
    rho, _ = solver.filtered_density(psi_eval)
    k_hat = rom.reduced_stiffness(basis, rho)
    rs = rom.solve(basis, rho, obj)
    return dict(rom_k_hat=k_hat, rom_f_hat=basis.f_hat, rom_uhat=rs.uhat, rom_j=rs.j,
                rom_residual=rs.residual_norm, rom_kept=phi.shape[1], rom_phi=phi)


def make_cfg1():
    prob = configs.cfg1()
    mesh, filt, solver = ref_problem(prob)
    obj = ComplianceObjective(solver.f)
    fr = filt.apply(prob.psi)
    sol = solver.solve(prob.psi, obj)
    g = solver.gradient(prob.psi, sol, obj)
    s = solver.element_sensitivity(sol.rho, sol.u, sol.lam, obj)
    rng = np.random.default_rng(123)
    v = rng.standard_normal(mesh.n_dofs)
    kv = solver.apply_stiffness(sol.rho, v)
    adj_v = rng.standard_normal(mesh.n_elems)
    adj = filt.apply_adjoint(adj_v)
    out = dict(psi=prob.psi, phi=fr.phi, rho_raw=fr.rho, rho=sol.rho, u=sol.u, j=sol.j, clamp_width=sol.clamp_width,
               s=s, g=g, v=v, kv=kv, adj_v=adj_v, adj=adj, load=filt.load_vector(prob.psi),
               elem_dofs_head=mesh.elem_dofs[:64], fixed=prob.fixed)
    out.update({k: v for k, v in rom_chain(mesh, solver, prob, prob.psi).items() if k != "rom_phi"})
    np.savez_compressed(os.path.join(HERE, "golden_cfg1.npz"), **out)
    print("cfg1: J=%.10f  J_rom=%.10f  ||r||=%.4e kept=%d" % (sol.j, out["rom_j"], out["rom_residual"],
                                                              out["rom_kept"]))


def make_cfg2():
    prob = configs.cfg2()
    mesh, filt, solver = ref_problem(prob)
    obj = ComplianceObjective(solver.f)
    t0 = time.perf_counter()
    sol = solver.solve(prob.psi, obj)
    g = solver.gradient(prob.psi, sol, obj)
    s = solver.element_sensitivity(sol.rho, sol.u, sol.lam, obj)
    print("cfg2 HDM eval %.2f s" % (time.perf_counter() - t0))
    st_e, st_u = 16, 16
    out = dict(j=sol.j, clamp_width=sol.clamp_width, rho_s=sol.rho[::st_e], u_s=sol.u[::st_u], s_s=s[::st_e],
               g_s=g[::st_e], s_inf=np.abs(s).max(), g_inf=np.abs(g).max(), u_norm=np.linalg.norm(sol.u),
               rho_sum=sol.rho.sum(), stride_e=st_e, stride_u=st_u)
    out.update({k: v for k, v in rom_chain(mesh, solver, prob, prob.psi).items() if k != "rom_phi"})
    np.savez_compressed(os.path.join(HERE, "golden_cfg2.npz"), **out)
    print("cfg2: J=%.10f  J_rom=%.10f  ||r||=%.4e kept=%d" % (sol.j, out["rom_j"], out["rom_residual"],
                                                              out["rom_kept"]))


def make_cantilever(nx, ny, h=1.0, radius=None):
    """Reference tests/conftest.py:15-33 fixture (default MaterialModel rho_l = 1e-3)."""
    mesh = build_mesh(nx, ny, h)
    radius = 1.5 * h if radius is None else radius
    filt = HelmholtzFilter(mesh, radius)
    f = np.zeros(mesh.n_dofs)
    f[2 * mesh.node_id(nx, ny // 2) + 1] = -1.0
    left = mesh.boundary_nodes("left")
    fixed = np.concatenate([2 * left, 2 * left + 1])
    return mesh, filt, HdmSolver(mesh, elasticity_element_matrix(1.0, 0.3, h), filt, f, fixed, MaterialModel()), f, fixed


def make_small():
    out = {}
    for nx, ny in ((6, 2), (12, 4), (4, 2)):
        mesh, filt, solver, f, fixed = make_cantilever(nx, ny)
        obj = ComplianceObjective(solver.f)
        rng = np.random.default_rng(nx * 100 + ny)
        psi = 0.2 + 0.6 * rng.random(mesh.n_elems)
        sol = solver.solve(psi, obj)
        key = f"cant{nx}x{ny}"
        out[f"{key}_psi"] = psi
        out[f"{key}_f"] = f
        out[f"{key}_fixed"] = fixed
        out[f"{key}_u"] = sol.u
        out[f"{key}_rho"] = sol.rho
        out[f"{key}_j"] = sol.j
        out[f"{key}_g"] = solver.gradient(psi, sol, obj)
        # ROM: window of 3 perturbed snapshots + center, n_k = 2
        from romtopt.rom import SnapshotWindow

        win = SnapshotWindow(5)
        for _ in range(3):
            p2 = np.clip(psi + 0.1 * rng.standard_normal(mesh.n_elems), 0, 1)
            s2 = solver.solve(p2, obj)
            win.append(s2.u, s2.lam, key=s2.psi_hash)
        rom = RomModel(solver)
        basis = rom.build_basis(win, sol.u, sol.lam, True, 2, center_rho=sol.rho)
        rho_t = np.clip(0.3 + 0.5 * rng.random(mesh.n_elems), 1e-3, 1.0)
        rs = rom.solve(basis, rho_t, obj)
        out[f"{key}_win"] = win.primal_matrix()
        out[f"{key}_pod2"] = pod(win.primal_matrix(), 2)
        out[f"{key}_rom_phi"] = basis.phi
        out[f"{key}_rom_fhat"] = basis.f_hat
        out[f"{key}_rom_rho"] = rho_t
        out[f"{key}_rom_khat"] = rom.reduced_stiffness(basis, rho_t)
        out[f"{key}_rom_uhat"] = rs.uhat
        out[f"{key}_rom_j"] = rs.j
        out[f"{key}_rom_res"] = rs.residual_norm
        eb = rom.error_bounds(basis, rho_t, rs, obj, mode="certified")
        out[f"{key}_rom_sigma"] = eb.sigma_min
    # filter fixtures (reference tests/test_filtering.py cases)
    for nx, ny, h, radius in ((4, 3, 0.25, 0.3), (12, 12, 0.25, 0.25), (6, 9, 0.25, 0.0), (8, 5, 0.25, 0.6),
                              (9, 5, 0.2, 2.0)):
        mesh = build_mesh(nx, ny, h)
        filt = HelmholtzFilter(mesh, radius)
        rng = np.random.default_rng(nx + ny)
        psi = rng.random(mesh.n_elems)
        v = rng.standard_normal(mesh.n_elems)
        key = f"filt{nx}x{ny}_{h}_{radius}"
        out[f"{key}_psi"] = psi
        res = filt.apply(psi)
        out[f"{key}_phi"] = res.phi
        out[f"{key}_rho"] = res.rho
        out[f"{key}_v"] = v
        out[f"{key}_adj"] = filt.apply_adjoint(v)
    np.savez_compressed(os.path.join(HERE, "golden_small.npz"), **out)
    print("small fixtures:", len(out), "arrays")


def make_ref3d():
    """Reference solver code run unchanged on a duck-typed Hex8 mesh."""
    from oracle.fem import build_grid, elasticity_element_matrix as ke_any

    for (nx, ny, nz), name in (((6, 3, 3), "ref3d_small.npz"), ((20, 10, 10), "ref3d_medium.npz")):
        g = build_grid(nx, ny, 1.0, nz=nz)
        mesh = SimpleNamespace(elem_dofs=g.elem_dofs, elem_nodes=g.elem_nodes, n_elems=g.n_elems, n_nodes=g.n_nodes,
                               n_dofs=g.n_dofs, elem_volume=1.0, h=1.0, nx=nx, ny=ny)
        k_e = ke_any(1.0, 0.3, 1.0, dim=3)
        prob = configs.cfg3(seed=1, nx=nx, ny=ny, nz=nz)
        assert np.array_equal(prob.k_e, k_e) or np.abs(prob.k_e - k_e).max() < 1e-15

        class IdentityFilter:
            def apply(self, psi):
                return SimpleNamespace(rho=np.asarray(psi, float).copy(), phi=None)

            def apply_adjoint(self, v):
                return np.asarray(v, float).copy()

        solver = HdmSolver(mesh, prob.k_e, IdentityFilter(), prob.f, prob.fixed, MAT)
        obj = ComplianceObjective(solver.f)
        sol = solver.solve(prob.psi, obj)
        s = solver.element_sensitivity(sol.rho, sol.u, sol.lam, obj)
        rng = np.random.default_rng(5)
        v = rng.standard_normal(g.n_dofs)
        kv = solver.apply_stiffness(sol.rho, v)
        # ROM on a seeded sine basis
        raw = configs.phi_columns(prob.mesh, 6, seed=3)
        raw[:, ~solver.free_mask] = 0.0
        phi = gram_schmidt(list(raw))
        basis = ReducedBasis(phi=phi, elem_phi=phi[g.elem_dofs], elem_k_phi=np.matmul(prob.k_e, phi[g.elem_dofs]),
                             f_hat=phi.T @ solver.f)
        rom = RomModel(solver)
        k_hat = rom.reduced_stiffness(basis, sol.rho)
        rs = rom.solve(basis, sol.rho, obj)
        np.savez_compressed(os.path.join(HERE, name), psi=prob.psi, u=sol.u, j=sol.j, s=s, v=v, kv=kv,
                            phi=phi, k_hat=k_hat, f_hat=basis.f_hat, uhat=rs.uhat, rom_j=rs.j,
                            rom_res=rs.residual_norm, dims=np.array([nx, ny, nz]))
        print("ref3d: J=%.10f  J_rom=%.10f" % (sol.j, rs.j))


def make_mma():
    from romtopt.mma import MmaOptimizer

    sys.path.insert(0, os.path.dirname(HERE))
    from mma_cases import mma_cases

    out = {}
    for name, lower, upper, w, cap, x0, grads, caps in mma_cases():
        opt = MmaOptimizer(lower, upper, w, cap)
        x, xs = x0.copy(), []
        for g, mc in zip(grads, caps):
            x = opt.step(x, 0.0, g, move_cap=mc)
            xs.append(x.copy())
        out[f"{name}_xs"] = np.stack(xs)
        out[f"{name}_low"], out[f"{name}_upp"] = opt.low, opt.upp
        print(f"mma {name}: n={len(x0)} final volume {w @ x:.12g} cap {cap:.12g}")
    np.savez_compressed(os.path.join(HERE, "golden_mma.npz"), **out)


def subproblem_setup():
    """Shared recipe (also restated in tests/test_gpu_subproblem.py): 48x16 cfg-1 geometry,
    centre psi_k = 0.9 psi (feasible for V = 0.5 |domain|), basis = GS of the centre solution
    and the seeded ROM-design snapshots."""
    prob = configs.cfg1(seed=4, nx=48, ny=16)
    psi_k = np.clip(0.9 * prob.psi, 0.0, 1.0)
    return prob, psi_k


def make_subproblem():
    from romtopt.trustregion import TrConfig, TrustRegionDriver

    prob, psi_k = subproblem_setup()
    mesh, filt, solver = ref_problem(prob)
    obj = ComplianceObjective(solver.f)
    sol = solver.solve(psi_k, obj)
    g = solver.gradient(psi_k, sol, obj)
    snaps = [np.where(solver.free_mask, sol.u, 0.0)]
    snaps += [np.where(solver.free_mask, solver.solve(d, obj).u, 0.0) for d in prob.rom_designs[:5]]
    phi = gram_schmidt(snaps)
    basis = ReducedBasis(phi=phi, elem_phi=phi[mesh.elem_dofs], elem_k_phi=np.matmul(solver.k_e, phi[mesh.elem_dofs]),
                         f_hat=phi.T @ solver.f)
    rom = RomModel(solver)
    w = np.full(mesh.n_elems, mesh.elem_volume)
    cap = 0.5 * mesh.n_elems * mesh.elem_volume
    out = dict(psi_k=psi_k, phi=phi, j_center=sol.j, grad_center=g, cap=cap)
    for kind, delta, inner in (("res", 4.7, 12), ("dist", 5.2, 12)):
        drv = TrustRegionDriver(solver, rom, obj, w, cap, TrConfig(constraint=kind, max_inner=inner))
        r = drv.solve_subproblem(basis, psi_k, delta, sol.j, g)
        out.update({f"{kind}_delta": delta, f"{kind}_inner": inner, f"{kind}_candidate": r.candidate,
                    f"{kind}_model_value": r.model_value, f"{kind}_theta": r.theta, f"{kind}_steps": r.steps,
                    f"{kind}_rom_solves": r.rom_solves, f"{kind}_curvature": r.curvature,
                    f"{kind}_first": r.first_iterate})
        print(f"subproblem {kind}: steps={r.steps} rom_solves={r.rom_solves} J_m={r.model_value:.10f} "
              f"theta={r.theta:.4e} curvature={r.curvature:.4e}")
    np.savez_compressed(os.path.join(HERE, "golden_subproblem.npz"), **out)


if __name__ == "__main__":
    if "--subproblem-only" in sys.argv:
        make_subproblem()
        sys.exit(0)
    if "--mma-only" in sys.argv:
        make_mma()
        sys.exit(0)
    make_mma()
    make_subproblem()
    make_cfg1()
    make_small()
    make_ref3d()
    if "--with-cfg2" in sys.argv:
        make_cfg2()
