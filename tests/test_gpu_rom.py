"""GPU parity of the ROM path (Gram-Schmidt, POD, Phi^T f, Phi^T K Phi, reduced solve,
residual / error estimates) against reference golden vectors and the CPU oracle.
Tolerances: reduced operators and error estimates 1e-6 relative (BASELINE north_star)."""

import numpy as np
import pytest

import paper_2004_05756_b200 as tb
from conftest import golden
from oracle.fem import build_grid
from oracle.hdm import Filter, Hdm, Material
from oracle.rom import Rom, gram_schmidt as gs_ref, pod as pod_ref
from paper_2004_05756_b200 import configs

pytestmark = pytest.mark.gpu

MAT = tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP)


def frel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


def build(prob, rtol=1e-12):
    return tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed, MAT,
                        rtol=rtol)


def test_gram_schmidt_matches_oracle(cuda):
    rng = np.random.default_rng(3)
    vecs = [rng.standard_normal(1000) for _ in range(6)]
    vecs.insert(2, 2.0 * vecs[0])  # dependent -> dropped
    vecs.insert(4, np.zeros(1000))  # zero -> skipped
    q = tb.gram_schmidt(vecs)
    q_ref = gs_ref(vecs)
    assert q.shape == q_ref.shape == (1000, 6)
    assert np.abs(q - q_ref).max() < 1e-12
    assert np.abs(q.T @ q - np.eye(6)).max() < 1e-12
    with pytest.raises(ValueError):
        tb.gram_schmidt([np.zeros(5)])
    assert tb.gram_schmidt([np.ones(5), -np.ones(5)]).shape[1] == 1


def test_block_gram_schmidt_panels_vs_oracle(cuda):
    """Several panels of 8 (tb_gram_schmidt's block CGS2): drops inside a panel, across panels,
    zero and near-dependent vectors; the kept set and the basis equal rom.py:76-97's MGS x2."""
    rng = np.random.default_rng(11)
    n = 20_000
    base = [rng.standard_normal(n) for _ in range(15)]
    vecs = list(base[:9])
    vecs.append(3.0 * base[2] - base[7])                       # depends on the previous panel -> dropped
    vecs.append(base[9])
    vecs.append(np.zeros(n))                                    # zero -> skipped
    vecs.append(base[9] - 2.0 * base[8] + 1e-14 * base[10])     # residual ~1e-15 of its norm -> dropped
    vecs.append(base[0] + 1e-6 * base[14])                      # residual ~1e-6 of its norm -> kept
    vecs += base[10:14]
    vecs.append(base[13] + base[12])                            # same panel -> dropped
    vecs += [rng.standard_normal(n) for _ in range(6)]
    q = tb.gram_schmidt(vecs)
    q_ref = gs_ref(vecs)
    assert q.shape == q_ref.shape == (n, 21)
    assert np.abs(q.T @ q - np.eye(21)).max() < 1e-12
    # column 10 is determined by a 1e-6 residual: its round-off is amplified ~1e6 on both sides
    err = np.abs(q - q_ref).max(axis=0)
    assert err[np.arange(21) != 10].max() < 1e-12 and err[10] < 1e-8, err
    for m in (1, 8, 9, 17):  # panel boundaries
        vs = [rng.standard_normal(300) for _ in range(m)]
        assert np.abs(tb.gram_schmidt(vs) - gs_ref(vs)).max() < 1e-12


def test_pod_matches_oracle(cuda):
    rng = np.random.default_rng(1)
    snaps = rng.standard_normal((50, 6))
    u = tb.pod(snaps, 3)
    u_ref = pod_ref(snaps, 3)
    assert np.abs(u - u_ref).max() < 1e-10  # same sign convention, same vectors
    assert tb.pod(snaps, 0).shape == (50, 0)
    with pytest.raises(ValueError):
        tb.pod(np.ones((5, 2)), 3)
    G = golden("golden_small.npz")
    assert np.abs(tb.pod(G["cant6x2_win"], 2) - G["cant6x2_pod2"]).max() < 1e-8


def test_cfg1_rom_chain_vs_reference_golden(cuda):
    G = golden("golden_cfg1.npz")
    prob = configs.cfg1()
    s = build(prob, rtol=1e-10)
    obj = tb.ComplianceObjective(s.f)
    snaps = [np.where(s.free_mask, s.solve(d, obj).u, 0.0) for d in prob.rom_designs]
    phi = tb.gram_schmidt(snaps)
    assert phi.shape[1] == int(G["rom_kept"])
    basis = tb.ReducedBasis(phi, None, None, phi.T @ s.f)
    rom = tb.RomModel(s)
    rho, _ = s.filtered_density(prob.psi)
    assert frel(rom.reduced_stiffness(basis, rho), G["rom_k_hat"]) <= 1e-6
    rs = rom.solve(basis, rho, obj)
    assert abs(rs.j - G["rom_j"]) <= 1e-8 * abs(G["rom_j"])
    assert abs(rs.residual_norm - G["rom_residual"]) <= 1e-6 * G["rom_residual"]
    assert rom.residual_norm(basis, rho, rs) == rs.residual_norm
    assert s.stats.rom_solves == 1


def test_reduced_operators_vs_oracle_exact_basis(cuda):
    """Same Phi on both sides: k_hat, f_hat, uhat, residual to round-off."""
    for k in (3, 10, 33, 64):
        prob = configs.cfg1(seed=k, nx=40, ny=20)
        s = build(prob)
        g = build_grid(40, 20, 1.0)
        ora = Hdm(g, prob.k_e, Filter(g, prob.radius), prob.f, prob.fixed, Material(configs.RHO_L, configs.P_SIMP))
        rng = np.random.default_rng(k)
        raw = rng.standard_normal((k, g.n_dofs))
        raw[:, ~ora.free_mask] = 0.0
        phi = gs_ref(list(raw))
        rho = np.clip(rng.random(g.n_elems), 1e-3, 1.0)
        rom = tb.RomModel(s)
        basis = tb.ReducedBasis(phi, None, None, phi.T @ s.f)
        kh = rom.reduced_stiffness(basis, rho)
        kr = Rom(ora).reduced_stiffness_elemform(phi, rho)
        assert frel(kh, kr) <= 1e-12
        rs = rom.solve(basis, rho, tb.ComplianceObjective(s.f))
        rr = Rom(ora).solve(phi, phi.T @ ora.f, rho)
        assert frel(rs.uhat, rr["uhat"]) <= 1e-9
        assert abs(rs.residual_norm - rr["residual_norm"]) <= 1e-9 * rr["residual_norm"]


def test_batched_reduced_stiffness(cuda):
    import torch

    prob = configs.cfg1(seed=5, nx=32, ny=16)
    s = build(prob)
    g = build_grid(32, 16, 1.0)
    ora = Hdm(g, prob.k_e, Filter(g, prob.radius), prob.f, prob.fixed, Material(configs.RHO_L, configs.P_SIMP))
    rng = np.random.default_rng(0)
    raw = rng.standard_normal((12, g.n_dofs))
    raw[:, ~ora.free_mask] = 0.0
    phi = gs_ref(list(raw))
    rhos = np.clip(rng.random((5, g.n_elems)), 1e-3, 1.0)
    rom = tb.RomModel(s)
    basis = tb.ReducedBasis(phi, None, None, phi.T @ s.f)
    khat, uhat, norms = rom.solve_batch(basis, torch.as_tensor(rhos, device=cuda))
    for d in range(5):
        rr = Rom(ora).solve(phi, phi.T @ ora.f, rhos[d])
        assert frel(khat[d].cpu().numpy(), rr["k_hat"]) <= 1e-12
        assert frel(uhat[d].cpu().numpy(), rr["uhat"]) <= 1e-9
        assert abs(norms[d] - rr["residual_norm"]) <= 1e-9 * rr["residual_norm"]


def test_small_fixture_build_basis_and_bounds(cuda):
    G = golden("golden_small.npz")
    key = "cant6x2"
    mesh = tb.build_mesh(6, 2, 1.0)
    s = tb.HdmSolver(mesh, tb.elasticity_element_matrix(1.0, 0.3), tb.HelmholtzFilter(mesh, 1.5), G[f"{key}_f"],
                     G[f"{key}_fixed"], tb.MaterialModel(), rtol=1e-13)
    obj = tb.ComplianceObjective(s.f)
    sol = s.solve(G[f"{key}_psi"], obj)
    win = tb.SnapshotWindow(5)
    for c in range(G[f"{key}_win"].shape[1]):
        win.append(G[f"{key}_win"][:, c], G[f"{key}_win"][:, c])
    rom = tb.RomModel(s)
    basis = rom.build_basis(win, sol.u, sol.lam, True, 2, center_rho=sol.rho)
    assert basis.size == G[f"{key}_rom_phi"].shape[1]
    # span/orientation: compare projectors
    P = basis.phi @ basis.phi.T
    Pr = G[f"{key}_rom_phi"] @ G[f"{key}_rom_phi"].T
    assert np.abs(P - Pr).max() < 1e-8
    rho_t = G[f"{key}_rom_rho"]
    assert frel(rom.reduced_stiffness(basis, rho_t), G[f"{key}_rom_khat"]) <= 1e-6
    rs = rom.solve(basis, rho_t, obj)
    assert abs(rs.j - G[f"{key}_rom_j"]) <= 1e-8 * abs(G[f"{key}_rom_j"])
    assert abs(rs.residual_norm - G[f"{key}_rom_res"]) <= 1e-6 * G[f"{key}_rom_res"]
    rep = rom.error_bounds(basis, rho_t, rs, obj, mode="cheap")
    assert rep.primal_residual == pytest.approx(rs.residual_norm, rel=1e-12)
    assert rep.adjoint_residual == pytest.approx(rep.primal_residual, rel=1e-10)
    rep = rom.error_bounds(basis, rho_t, rs, obj, mode="certified")
    assert rep.sigma_min == pytest.approx(float(G[f"{key}_rom_sigma"]), rel=1e-6)
    with pytest.raises(ValueError):
        rom.error_bounds(basis, rho_t, rs, obj, mode="tight")


def test_exact_span_and_errors(cuda):
    mesh = tb.build_mesh(6, 2, 1.0)
    f = np.zeros(mesh.n_dofs)
    f[2 * mesh.node_id(6, 1) + 1] = -1.0
    left = mesh.boundary_nodes("left")
    s = tb.HdmSolver(mesh, tb.elasticity_element_matrix(1.0, 0.3), tb.HelmholtzFilter(mesh, 1.5), f,
                     np.concatenate([2 * left, 2 * left + 1]), tb.MaterialModel(), rtol=1e-13)
    obj = tb.ComplianceObjective(s.f)
    psi = np.full(mesh.n_elems, 0.55)
    sol = s.solve(psi, obj)
    rom = tb.RomModel(s)
    basis = rom.build_basis(tb.SnapshotWindow(20), sol.u, sol.lam, True, 0, center_rho=sol.rho)
    assert basis.size == 1
    rs = rom.solve(basis, sol.rho, obj)
    assert np.linalg.norm(rs.u - sol.u) <= 1e-9 * np.linalg.norm(sol.u)
    assert abs(rs.j - sol.j) <= 1e-9 * abs(sol.j)
    assert rs.residual_norm <= 1e-9 * np.linalg.norm(s.f)
    r0 = rom.residual_vector(basis, sol.rho, np.zeros(basis.size))
    assert abs(np.linalg.norm(r0) - np.linalg.norm(s.f)) <= 1e-12
    # rank-deficient basis -> DegenerateBasisError (reference tests/test_rom.py:293-307)
    v = sol.u / np.linalg.norm(sol.u)
    phi = np.column_stack([v, v])
    with pytest.raises(tb.DegenerateBasisError):
        rom.solve(tb.ReducedBasis(phi, None, None, phi.T @ s.f), sol.rho, obj)
    # generation mismatch
    basis2 = rom.build_basis(tb.SnapshotWindow(20), sol.u, sol.lam, True, 0, center_rho=sol.rho)
    with pytest.raises(tb.BasisMismatchError):
        rom.residual_norm(basis2, sol.rho, rs)
    with pytest.raises(ValueError):
        rom.build_basis(tb.SnapshotWindow(5), np.zeros(mesh.n_dofs), None, True, 0)


def test_certified_lanczos_matches_power_iteration(cuda):
    """Certified sigma_min: shift-invert Lanczos (default) and the reference's inverse power
    iteration agree, Lanczos in far fewer solves."""
    prob = configs.cfg1(seed=2, nx=48, ny=16)
    s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed,
                     tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=1e-11)
    obj = tb.ComplianceObjective(s.f)
    snaps = [np.where(s.free_mask, s.solve(d, obj).u, 0.0) for d in prob.rom_designs[:3]]
    phi = tb.gram_schmidt(snaps)
    basis = tb.ReducedBasis(phi, None, None, phi.T @ s.f)
    rom = tb.RomModel(s)
    rho, _ = s.filtered_density(prob.psi)
    rs = rom.solve(basis, rho, obj)
    n0 = s.stats.factorizations
    lz = rom.error_bounds(basis, rho, rs, obj, mode="certified")
    pw = rom.error_bounds(basis, rho, rs, obj, mode="certified", method="power")
    assert lz.sigma_min_converged and pw.sigma_min_converged
    assert lz.sigma_min == pytest.approx(pw.sigma_min, rel=1e-6)
    with pytest.raises(ValueError):
        rom.error_bounds(basis, rho, rs, obj, mode="certified", method="qr")
    del n0


@pytest.mark.parametrize("k,nvec", [(1, 1), (2, 3), (3, 16), (10, 5), (33, 2), (64, 16), (64, 20), (100, 4)])
def test_project_and_reconstruct_kernels_vs_numpy(cuda, k, nvec):
    """tb_rom_project (Phi^T V: single-vector, shared-memory tiled and tiny-k kernels) and
    tb_rom_reconstruct (Phi Uhat: DMMA kernel for k <= 64) against numpy on a ragged size."""
    import ctypes

    import torch

    from paper_2004_05756_b200 import _lib

    dev = torch.device("cuda", 0)
    n = 40037
    rng = np.random.default_rng(k * 100 + nvec)
    phi = rng.standard_normal((n, k))
    vec = rng.standard_normal((nvec, n))
    phi_d, vec_d = torch.as_tensor(phi, device=dev), torch.as_tensor(vec, device=dev)
    out = torch.empty(nvec, k, dtype=torch.float64, device=dev)
    lib = _lib.lib()
    _lib.check(lib.tb_rom_project(ctypes.c_int64(n), _lib.ptr(phi_d), k, _lib.ptr(vec_d), nvec, _lib.ptr(out),
                                  _lib.stream_ptr(dev)), "project")
    ref = vec @ phi
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-12 * np.abs(ref).max()
    nd = min(nvec, 16)
    uhat = rng.standard_normal((nd, k))
    u = torch.empty(nd, n, dtype=torch.float64, device=dev)
    _lib.check(lib.tb_rom_reconstruct(ctypes.c_int64(n), _lib.ptr(phi_d), k, _lib.ptr(torch.as_tensor(uhat, device=dev)),
                                      nd, _lib.ptr(u), _lib.stream_ptr(dev)), "reconstruct")
    ref_u = uhat @ phi.T
    assert np.abs(u.cpu().numpy() - ref_u).max() <= 1e-12 * np.abs(ref_u).max()
