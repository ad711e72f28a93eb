"""CPU: pin the oracle to golden vectors produced by the reference itself, and check the
3D restatement against the reference-style invariants (tests/oracles.py patterns)."""

import numpy as np
import pytest

from conftest import golden
from oracle.fem import DirectSolver, assemble, build_grid, elasticity_element_matrix, quad_elasticity
from oracle.hdm import Filter, Hdm, Material
from oracle.rom import Rom, gram_schmidt, pod
from paper_2004_05756_b200 import configs

MAT = Material(configs.RHO_L, configs.P_SIMP)


def oracle_for(prob, mat=MAT):
    g = build_grid(prob.mesh.nx, prob.mesh.ny, prob.mesh.h, nz=(prob.mesh.nz or None))
    return g, Hdm(g, prob.k_e, Filter(g, prob.radius), prob.f, prob.fixed, mat)


def test_cfg1_hdm_matches_reference_golden():
    G = golden("golden_cfg1.npz")
    prob = configs.cfg1()
    assert np.array_equal(prob.psi, G["psi"])  # inputs reproduced byte-for-byte
    assert np.array_equal(prob.fixed, G["fixed"])
    g, hdm = oracle_for(prob)
    assert np.array_equal(g.elem_dofs[:64], G["elem_dofs_head"])
    phi, rho_raw = hdm.filter.apply(prob.psi)
    assert np.abs(phi - G["phi"]).max() <= 1e-13
    assert np.abs(rho_raw - G["rho_raw"]).max() <= 1e-13
    assert np.abs(hdm.filter.load_vector(prob.psi) - G["load"]).max() == 0.0
    sol = hdm.solve(prob.psi)
    assert abs(sol["j"] - G["j"]) <= 1e-10 * abs(G["j"])  # direct solves differ in assembly order
    assert np.abs(sol["u"] - G["u"]).max() <= 1e-9 * np.abs(G["u"]).max()
    g_ = hdm.gradient(sol)
    assert np.abs(g_ - G["g"]).max() <= 1e-9 * np.abs(G["g"]).max()
    s = hdm.element_sensitivity(sol["rho"], sol["u"], sol["lam"])
    assert np.abs(s - G["s"]).max() <= 1e-9 * np.abs(G["s"]).max()
    assert np.abs(hdm.apply_stiffness(sol["rho"], G["v"]) - G["kv"]).max() <= 1e-13 * np.abs(G["kv"]).max()
    assert np.abs(hdm.filter.apply_adjoint(G["adj_v"]) - G["adj"]).max() <= 1e-13


def test_cfg1_rom_chain_matches_reference_golden():
    G = golden("golden_cfg1.npz")
    prob = configs.cfg1()
    g, hdm = oracle_for(prob)
    snaps = [np.where(hdm.free_mask, hdm.solve(d)["u"], 0.0) for d in prob.rom_designs]
    phi = gram_schmidt(snaps)
    assert phi.shape[1] == int(G["rom_kept"])
    rom = Rom(hdm)
    rho, _ = hdm.filtered_density(prob.psi)
    kh_e = rom.reduced_stiffness_elemform(phi, rho)
    kh_n = rom.reduced_stiffness_nodeform(phi, rho)
    ref = G["rom_k_hat"]
    assert np.linalg.norm(kh_e - ref) <= 1e-10 * np.linalg.norm(ref)
    assert np.linalg.norm(kh_n - ref) <= 1e-10 * np.linalg.norm(ref)
    rs = rom.solve(phi, phi.T @ hdm.f, rho)
    assert abs(rs["j"] - G["rom_j"]) <= 1e-10 * abs(G["rom_j"])
    assert abs(rs["residual_norm"] - G["rom_residual"]) <= 1e-8 * G["rom_residual"]


@pytest.mark.parametrize("nx,ny", [(6, 2), (12, 4), (4, 2)])
def test_small_cantilevers_match_reference(nx, ny):
    G = golden("golden_small.npz")
    key = f"cant{nx}x{ny}"
    g = build_grid(nx, ny, 1.0)
    hdm = Hdm(g, elasticity_element_matrix(1.0, 0.3), Filter(g, 1.5), G[f"{key}_f"], G[f"{key}_fixed"], Material())
    sol = hdm.solve(G[f"{key}_psi"])
    assert abs(sol["j"] - G[f"{key}_j"]) <= 1e-12 * abs(G[f"{key}_j"])
    assert np.abs(hdm.gradient(sol) - G[f"{key}_g"]).max() <= 1e-10 * np.abs(G[f"{key}_g"]).max()
    # POD sign rule and span
    p2 = pod(G[f"{key}_win"], 2)
    assert np.abs(p2 - G[f"{key}_pod2"]).max() <= 1e-8
    rom = Rom(hdm)
    phi, fhat = rom.build_basis(G[f"{key}_win"], sol["u"], sol["lam"], True, 2, center_rho=sol["rho"])
    assert np.abs(np.abs(phi) - np.abs(G[f"{key}_rom_phi"])).max() <= 1e-8
    kh = rom.reduced_stiffness_nodeform(phi, G[f"{key}_rom_rho"])
    assert np.linalg.norm(kh - G[f"{key}_rom_khat"]) <= 1e-9 * np.linalg.norm(G[f"{key}_rom_khat"])
    sig, ok = rom.smallest_eigenvalue(G[f"{key}_rom_rho"])
    assert ok and abs(sig - G[f"{key}_rom_sigma"]) <= 1e-8 * G[f"{key}_rom_sigma"]


def test_filter_fixtures_match_reference():
    G = golden("golden_small.npz")
    for nx, ny, h, radius in ((4, 3, 0.25, 0.3), (12, 12, 0.25, 0.25), (6, 9, 0.25, 0.0), (8, 5, 0.25, 0.6),
                              (9, 5, 0.2, 2.0)):
        key = f"filt{nx}x{ny}_{h}_{radius}"
        f = Filter(build_grid(nx, ny, h), radius)
        phi, rho = f.apply(G[f"{key}_psi"])
        assert np.abs(rho - G[f"{key}_rho"]).max() <= 1e-13
        assert np.abs(f.apply_adjoint(G[f"{key}_v"]) - G[f"{key}_adj"]).max() <= 1e-12


@pytest.mark.parametrize("fixture", ["ref3d_small.npz", "ref3d_medium.npz"])
def test_3d_oracle_matches_reference_on_duck_typed_mesh(fixture):
    G = golden(fixture)
    nx, ny, nz = (int(v) for v in G["dims"])
    prob = configs.cfg3(seed=1, nx=nx, ny=ny, nz=nz)
    g = build_grid(nx, ny, 1.0, nz=nz)

    class Ident:
        def apply(self, psi):
            return None, np.asarray(psi, float).copy()

        def apply_adjoint(self, v):
            return np.asarray(v, float).copy()

    hdm = Hdm(g, prob.k_e, Ident(), prob.f, prob.fixed, MAT)
    sol = hdm.solve(G["psi"])
    assert abs(sol["j"] - G["j"]) <= 1e-10 * abs(G["j"])  # direct solves differ in assembly order
    s = hdm.element_sensitivity(sol["rho"], sol["u"], sol["lam"])
    assert np.abs(s - G["s"]).max() <= 1e-9 * np.abs(G["s"]).max()
    assert np.abs(hdm.apply_stiffness(sol["rho"], G["v"]) - G["kv"]).max() <= 1e-13 * np.abs(G["kv"]).max()
    kh = Rom(hdm).reduced_stiffness_nodeform(G["phi"], sol["rho"])
    assert np.linalg.norm(kh - G["k_hat"]) <= 1e-10 * np.linalg.norm(G["k_hat"])


def test_hex8_element_matrix_invariants():
    k = quad_elasticity(3, 1.0, 0.3, 1.0)
    assert np.abs(k - k.T).max() == 0.0
    ev = np.linalg.eigvalsh(k)
    assert np.sum(np.abs(ev) < 1e-12) == 6 and ev.min() > -1e-14
    g = build_grid(1, 1, 1.0, nz=1)
    xyz = np.array([[i % 2, (i // 2) % 2, i // 4] for i in range(8)], float)[[0, 1, 3, 2, 4, 5, 7, 6]]
    assert np.array_equal(g.elem_nodes[0], [0, 1, 3, 2, 4, 5, 7, 6])
    for rot in ((0, 1), (1, 2), (0, 2)):
        m = np.zeros((8, 3))
        a, b = rot
        m[:, a], m[:, b] = -xyz[:, b], xyz[:, a]
        assert np.abs(k @ m.ravel()).max() < 1e-13
    # h scaling: K_e(h) = h K_e(1) in 3D
    assert np.abs(quad_elasticity(3, 1.0, 0.3, 0.5) - 0.5 * k).max() < 1e-15


@pytest.mark.parametrize("dims", [(3, 2, 2), (4, 3, 2)])
def test_3d_filter_identities(dims):
    nx, ny, nz = dims
    g = build_grid(nx, ny, 0.5, nz=nz)
    f = Filter(g, 0.8)
    rng = np.random.default_rng(0)
    psi = rng.random(g.n_elems)
    _, rho = f.apply(psi)
    assert abs(rho.sum() - psi.sum()) <= 1e-12 * psi.sum()  # volume preservation
    _, rc = f.apply(np.full(g.n_elems, 0.4))
    assert np.abs(rc - 0.4).max() < 1e-13  # constants preserved
    assert np.abs(f.apply_adjoint(np.ones(g.n_elems)) - 1.0).max() < 1e-12
    # exact transpose against the dense psi->rho map
    dense = np.column_stack([f.apply(e)[1] for e in np.eye(g.n_elems)])
    v = rng.standard_normal(g.n_elems)
    assert np.abs(f.apply_adjoint(v) - dense.T @ v).max() < 1e-12


def test_3d_solve_dense_consistency():
    prob = configs.cfg3(seed=2, nx=4, ny=2, nz=2)
    g, hdm = oracle_for(prob)
    sol = hdm.solve(prob.psi)
    k = hdm.stiffness(sol["rho"]).toarray()
    free = hdm.free_mask
    r = (k @ sol["u"] - hdm.f)[free]
    assert np.linalg.norm(r) <= 1e-10 * np.linalg.norm(hdm.f)
    assert abs(sol["j"] - sol["u"] @ k @ sol["u"]) <= 1e-10 * sol["j"]
    s = hdm.element_sensitivity(sol["rho"], sol["u"], sol["u"])
    # compliance identity sum(-s * rho / p) = J for alpha ~ rho^p (rho_l tiny)
    assert abs(np.sum(-s * sol["rho"] / 3.0) - sol["j"]) <= 1e-7 * sol["j"]


def test_direct_solver_rejects_singular():
    from oracle.fem import OracleIndefinite

    g = build_grid(2, 2, 1.0)
    with pytest.raises(OracleIndefinite):
        DirectSolver(assemble(g, elasticity_element_matrix(1.0, 0.3)))


def test_mma_oracle_replays_reference_trajectories():
    """oracle/mma.py against the reference MmaOptimizer's own trajectories (golden_mma.npz)."""
    from mma_cases import mma_cases

    from oracle.mma import MmaOracle

    G = golden("golden_mma.npz")
    for name, lower, upper, w, cap, x0, grads, caps in mma_cases():
        opt = MmaOracle(lower, upper, w, cap)
        x = x0
        for k, (g, mc) in enumerate(zip(grads, caps)):
            x = opt.step(x, g, move_cap=mc)
            ref = G[f"{name}_xs"][k]
            assert np.abs(x - ref).max() <= 1e-13, (name, k, np.abs(x - ref).max())
        assert np.abs(opt.asy[0] - G[f"{name}_low"]).max() <= 1e-13
        assert np.abs(opt.asy[1] - G[f"{name}_upp"]).max() <= 1e-13


def test_cone_oracle_is_normalised_and_symmetric_in_weights():
    """Rows of the cone filter sum to 1 and W_e A[e, j] = w(e, j) is symmetric (A = D^-1 W)."""
    from oracle.filters import cone_matrix

    radius = 2.2
    a = cone_matrix(7, 5, 0, 1.0, radius).toarray()
    assert np.abs(a.sum(axis=1) - 1.0).max() <= 1e-15
    w_e = radius / np.diag(a)  # A[e, e] = w(e, e) / W_e = R / W_e
    raw = a * w_e[:, None]
    assert np.allclose(raw, raw.T, rtol=0, atol=1e-13)
    assert np.all(raw[raw > 0] <= radius + 1e-15)
