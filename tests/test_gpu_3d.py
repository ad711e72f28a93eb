"""GPU parity of the Hex8 (3D) path against the reference run on a duck-typed 3D mesh
(golden ref3d_small.npz) and against the 3D oracle restatement."""

import numpy as np
import pytest

import paper_2004_05756_b200 as tb
from conftest import golden
from oracle.fem import build_grid
from oracle.hdm import Filter, Hdm, Material
from oracle.rom import Rom
from paper_2004_05756_b200 import configs

pytestmark = pytest.mark.gpu

MAT = tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP)


def nrel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300)


def build(prob, rtol=1e-12):
    return tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed, MAT,
                        rtol=rtol)


@pytest.mark.parametrize("fixture", ["ref3d_small.npz", "ref3d_medium.npz"])
def test_kernels_vs_reference_duck_typed_3d(cuda, fixture):
    """The reference's own HdmSolver / RomModel run unchanged on a duck-typed Hex8 mesh
    (tests/golden/make_golden.py), 6x3x3 and 20x10x10 elements."""
    G = golden(fixture)
    nx, ny, nz = (int(v) for v in G["dims"])
    prob = configs.cfg3(seed=1, nx=nx, ny=ny, nz=nz)
    s = build(prob)
    rho = G["psi"]  # the reference run used the identity filter: rho = psi
    assert nrel(s.apply_stiffness(rho, G["v"]), G["kv"]) <= 1e-13
    obj = tb.ComplianceObjective(s.f)
    assert nrel(s.element_sensitivity(rho, G["u"], G["u"], obj), G["s"]) <= 1e-12
    # pCG solve at rho vs the reference direct solve
    u = s.pcg_device(tb._lib.to_dev(rho, s.device), s._f_d).cpu().numpy()
    assert nrel(u, G["u"]) <= 1e-8
    assert abs(float(s.f @ u) - float(G["j"])) <= 1e-10 * abs(float(G["j"]))
    rom = tb.RomModel(s)
    basis = tb.ReducedBasis(G["phi"], None, None, G["f_hat"])
    kh = rom.reduced_stiffness(basis, rho)
    assert np.linalg.norm(kh - G["k_hat"]) <= 1e-12 * np.linalg.norm(G["k_hat"])
    rs = rom.solve(basis, rho, obj)
    assert abs(rs.j - float(G["rom_j"])) <= 1e-10 * abs(float(G["rom_j"]))
    assert abs(rs.residual_norm - float(G["rom_res"])) <= 1e-9 * float(G["rom_res"])


@pytest.mark.parametrize("dims", [(8, 4, 4), (12, 6, 5)])
def test_3d_full_evaluation_vs_oracle(cuda, dims):
    nx, ny, nz = dims
    prob = configs.cfg3(seed=3, nx=nx, ny=ny, nz=nz)
    s = build(prob, rtol=1e-10)
    g = build_grid(nx, ny, 1.0, nz=nz)
    ora = Hdm(g, prob.k_e, Filter(g, prob.radius), prob.f, prob.fixed, Material(configs.RHO_L, configs.P_SIMP))
    obj = tb.ComplianceObjective(s.f)
    sol = s.solve(prob.psi, obj)
    ref = ora.solve(prob.psi)
    assert abs(sol.j - ref["j"]) <= 1e-8 * abs(ref["j"])
    assert np.max(np.abs(sol.rho - ref["rho"]) / ref["rho"]) <= 1e-6
    assert nrel(s.gradient(prob.psi, sol, obj), ora.gradient(ref)) <= 1e-6


def test_3d_filter_identities_and_parity(cuda):
    mesh = tb.build_mesh_3d(6, 4, 3, 0.5)
    f = tb.HelmholtzFilter(mesh, 0.8)
    g = build_grid(6, 4, 0.5, nz=3)
    fo = Filter(g, 0.8)
    rng = np.random.default_rng(0)
    psi = rng.random(mesh.n_elems)
    res = f.apply(psi)
    phi_o, rho_o = fo.apply(psi)
    assert nrel(res.rho, rho_o) <= 1e-12 and nrel(res.phi, phi_o) <= 1e-12
    assert abs(res.rho.sum() - psi.sum()) <= 1e-10 * psi.sum()
    assert np.abs(f.apply(np.full(mesh.n_elems, 0.3)).rho - 0.3).max() < 1e-12
    assert np.abs(f.apply_adjoint(np.ones(mesh.n_elems)) - 1.0).max() < 1e-10
    v = rng.standard_normal(mesh.n_elems)
    assert nrel(f.apply_adjoint(v), fo.apply_adjoint(v)) <= 1e-12
    assert np.abs(f.load_vector(psi) - fo.load_vector(psi)).max() <= 1e-15


def test_3d_rom_batch_vs_oracle(cuda):
    import torch

    prob = configs.cfg5(nx=10, ny=5, nz=5, n_designs=4, k=16)
    s = build(prob)
    g = build_grid(10, 5, 1.0, nz=5)
    ora = Hdm(g, prob.k_e, Filter(g, prob.radius), prob.f, prob.fixed, Material(configs.RHO_L, configs.P_SIMP))
    raw = configs.phi_columns(prob.mesh, 16, seed=0)
    raw[:, ~s.free_mask] = 0.0
    phi = tb.gram_schmidt(list(raw))
    assert phi.shape[1] == 16
    basis = tb.ReducedBasis(phi, None, None, phi.T @ s.f)
    rom = tb.RomModel(s)
    rhos = np.stack(prob.rom_designs)
    khat, uhat, norms = rom.solve_batch(basis, torch.as_tensor(rhos, device=cuda))
    for d in range(4):
        rr = Rom(ora).solve(phi, phi.T @ ora.f, rhos[d])
        kr = Rom(ora).reduced_stiffness_elemform(phi, rhos[d])
        assert np.linalg.norm(khat[d].cpu().numpy() - kr) <= 1e-12 * np.linalg.norm(kr)
        assert np.abs(uhat[d].cpu().numpy() - rr["uhat"]).max() <= 1e-9 * np.abs(rr["uhat"]).max()
        assert abs(norms[d] - rr["residual_norm"]) <= 1e-9 * rr["residual_norm"]


def test_3d_non_isotropic_element_matrix_falls_back_to_node_owner(cuda):
    """A Hex8 element matrix without the isotropic WHT-block pattern (here D K D with a
    per-component scaling D) runs on the generic node-owner kernels; parity vs the oracle and a
    ROM chain on the same path."""
    prob = configs.cfg3(seed=8, nx=8, ny=4, nz=4)
    d = np.tile([1.0, 1.3, 0.8], 8)
    k_e = d[:, None] * prob.k_e * d[None, :]
    s = tb.HdmSolver(prob.mesh, k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed, MAT,
                     rtol=1e-11)
    g = build_grid(8, 4, 1.0, nz=4)
    ora = Hdm(g, k_e, Filter(g, prob.radius), prob.f, prob.fixed, Material(configs.RHO_L, configs.P_SIMP))
    obj = tb.ComplianceObjective(s.f)
    sol = s.solve(prob.psi, obj)
    ref = ora.solve(prob.psi)
    assert abs(sol.j - ref["j"]) <= 1e-8 * abs(ref["j"])
    assert nrel(s.gradient(prob.psi, sol, obj), ora.gradient(ref)) <= 1e-6
    rng = np.random.default_rng(2)
    v = rng.standard_normal(prob.mesh.n_dofs)
    kv = s.apply_stiffness(sol.rho, v)
    k = s.assemble_stiffness(sol.rho)
    ref_kv = k @ v
    ref_kv[~s.free_mask] = 0.0
    assert nrel(kv, ref_kv) <= 1e-12
    phi = tb.gram_schmidt([np.where(s.free_mask, rng.standard_normal(prob.mesh.n_dofs), 0.0) for _ in range(4)])
    kh = tb.RomModel(s).reduced_stiffness(tb.ReducedBasis(phi, None, None, phi.T @ s.f), sol.rho)
    assert np.linalg.norm(kh - phi.T @ (k @ phi)) <= 1e-12 * np.linalg.norm(kh)


@pytest.mark.parametrize("dims", [(12, 6, 5), (7, 9, 4)])
def test_3d_filter_direct_solve_matches_pcg(cuda, monkeypatch, dims):
    """The direct (tensor-product cosine basis, spectral.cu) whole-grid filter solve against the
    pCG solve of the same system (TB_FILTER_PCG=1) and against the oracle's assembled operator
    (filtering.py:59-76): filter and adjoint."""
    nx, ny, nz = dims
    prob = configs.cfg3(seed=5, nx=nx, ny=ny, nz=nz)
    rng = np.random.default_rng(11)
    psi = rng.uniform(0.01, 1.0, prob.mesh.n_elems)
    v = rng.standard_normal(prob.mesh.n_elems)
    direct = tb.HelmholtzFilter(prob.mesh, prob.radius)
    monkeypatch.setenv("TB_FILTER_PCG", "1")
    pcg = tb.HelmholtzFilter(prob.mesh, prob.radius)
    monkeypatch.delenv("TB_FILTER_PCG")
    a, b = direct.apply(psi), pcg.apply(psi)
    assert nrel(a.rho, b.rho) <= 1e-10
    assert nrel(direct.apply_adjoint(v), pcg.apply_adjoint(v)) <= 1e-10
    g = build_grid(nx, ny, 1.0, nz=nz)
    ora = Filter(g, prob.radius)
    assert nrel(a.rho, ora.apply(psi)[1]) <= 1e-12
    assert nrel(direct.apply_adjoint(v), ora.apply_adjoint(v)) <= 1e-12
