"""Mirrors of reference unit tests (pkg/tests/test_hdm.py, test_rom.py) not covered elsewhere,
restated on the drop-in: symmetry, counters, gradient sign, Galerkin optimality, enrichment,
reduced-gradient finite differences, certified bounds against a dense eigen-solve, and the
sigma_min failure flag."""

import numpy as np
import pytest

import paper_2004_05756_b200 as tb

pytestmark = pytest.mark.gpu

MAT = tb.MaterialModel(rho_l=1e-9, p=3.0)


def cantilever(nx, ny, radius=1.5, rtol=1e-12):
    """Reference conftest cantilever: left edge clamped, unit downward load mid-right."""
    mesh = tb.build_mesh(nx, ny, 1.0)
    f = np.zeros(mesh.n_dofs)
    f[2 * mesh.node_id(nx, ny // 2) + 1] = -1.0
    left = mesh.boundary_nodes("left")
    fixed = np.concatenate([2 * left, 2 * left + 1])
    return tb.HdmSolver(mesh, tb.elasticity_element_matrix(1.0, 0.3), tb.HelmholtzFilter(mesh, radius), f, fixed,
                        MAT, rtol=rtol)


def dense_kff(s, rho):
    k = s.assemble_stiffness(rho).toarray()
    free = np.where(s.free_mask)[0]
    return k, free, k[np.ix_(free, free)]


def test_mirror_symmetry():
    """test_hdm.py:200-219: symmetric supports and load -> the gradient mirrors in x."""
    nx, ny = 12, 6
    mesh = tb.build_mesh(nx, ny, 1.0)
    f = np.zeros(mesh.n_dofs)
    for i, w in ((nx // 2 - 1, 0.5), (nx // 2, 1.0), (nx // 2 + 1, 0.5)):
        f[2 * mesh.node_id(i, ny) + 1] = -w
    fixed = np.array([0, 1, 2 * mesh.node_id(nx, 0), 2 * mesh.node_id(nx, 0) + 1])
    s = tb.HdmSolver(mesh, tb.elasticity_element_matrix(1.0, 0.3), tb.HelmholtzFilter(mesh, 1.2), f, fixed, MAT,
                     rtol=1e-12)
    obj = tb.ComplianceObjective(s.f)
    psi = np.full(mesh.n_elems, 1.0)
    sol = s.solve(psi, obj)
    g = s.gradient(psi, sol, obj).reshape(ny, nx)
    assert np.abs(g - g[:, ::-1]).max() <= 1e-8 * np.abs(g).max()


def test_solve_counters_audit():
    """test_hdm.py:120-149: the statistics sink counts every solve / factorisation / filter."""
    s = cantilever(6, 3)
    obj = tb.ComplianceObjective(s.f)
    rng = np.random.default_rng(1)
    n = 5
    for _ in range(n):
        psi = rng.uniform(0.1, 1.0, s.mesh.n_elems)
        sol = s.solve(psi, obj)
        s.gradient(psi, sol, obj)
    assert s.stats.hdm_solves == s.stats.factorizations == n
    assert s.stats.filter_solves == n
    assert s.stats.hdm_adjoint_solves == 0  # compliance is self-adjoint


def test_compliance_gradient_nonpositive_uniform():
    """test_hdm.py: stiffening any element cannot increase compliance."""
    s = cantilever(12, 4)
    obj = tb.ComplianceObjective(s.f)
    psi = np.full(s.mesh.n_elems, 0.5)
    sol = s.solve(psi, obj)
    assert np.all(s.gradient(psi, sol, obj) <= 1e-14)
    assert sol.lam is sol.u  # adjoint is the displacement for compliance (hdm.py:183-184)


def rom_setup(s, n_snap=3, seed=7):
    obj = tb.ComplianceObjective(s.f)
    rng = np.random.default_rng(seed)
    window = tb.SnapshotWindow(20)
    for _ in range(n_snap):
        psi = np.clip(0.5 + 0.2 * rng.standard_normal(s.mesh.n_elems), 0, 1)
        snap = s.solve(psi, obj)
        window.append(snap.u, snap.lam, key=snap.psi_hash)
    psi_c = np.full(s.mesh.n_elems, 0.5)
    sol = s.solve(psi_c, obj)
    rom = tb.RomModel(s)
    basis = rom.build_basis(window, sol.u, sol.lam, True, n_snap)
    rho = np.clip(0.5 + 0.2 * rng.standard_normal(s.mesh.n_elems), 1e-3, 1.0)
    return obj, rom, basis, rho, rng


def test_galerkin_energy_norm_optimality():
    """test_rom.py:201-225: the reduced solution minimises the energy error over span(Phi)."""
    s = cantilever(6, 2)
    obj, rom, basis, rho, rng = rom_setup(s)
    rsol = rom.solve(basis, rho, obj)
    k, free, kff = dense_kff(s, rho)
    u_star = np.zeros(s.mesh.n_dofs)
    u_star[free] = np.linalg.solve(kff, s.f[free])

    def energy(v):
        return np.sqrt(v @ (k @ v))

    e_rom = energy(u_star - rsol.u)
    for _ in range(20):
        other = basis.phi @ (rsol.uhat + 0.05 * rng.standard_normal(basis.size))
        assert e_rom <= energy(u_star - other) * (1 + 1e-10)


def test_enrichment_monotonicity():
    """test_rom.py:227-256: adding basis vectors never increases the energy error."""
    s = cantilever(6, 2)
    obj, rom, basis, rho, rng = rom_setup(s, seed=8)
    k, free, kff = dense_kff(s, rho)
    u_star = np.zeros(s.mesh.n_dofs)
    u_star[free] = np.linalg.solve(kff, s.f[free])

    def energy(v):
        return np.sqrt(v @ (k @ v))

    prev = energy(u_star - rom.solve(basis, rho, obj).u)
    cols = list(basis.phi.T)
    for _ in range(8):
        v = rng.standard_normal(s.mesh.n_dofs)
        v[~s.free_mask] = 0.0
        phi = tb.gram_schmidt(cols + [v])
        cols = list(phi.T)
        b = tb.ReducedBasis(phi, None, None, phi.T @ s.f)
        err = energy(u_star - rom.solve(b, rho, obj).u)
        assert err <= prev * (1 + 1e-9)
        prev = err


def test_reduced_gradient_finite_differences():
    """test_rom.py:258-309: the reduced model's gradient matches finite differences of J_rom."""
    s = cantilever(6, 2)
    obj, rom, basis, rho, rng = rom_setup(s, n_snap=2, seed=9)

    def model(p):
        r, _ = s.filtered_density(p)
        return rom.solve(basis, r, obj).j

    psi_t = np.clip(0.4 + 0.2 * rng.random(s.mesh.n_elems), 0, 1)
    rho_t, _ = s.filtered_density(psi_t)
    g = rom.solve(basis, rho_t, obj, compute_gradient=True).grad
    d = 1e-6
    for e in rng.choice(s.mesh.n_elems, 5, replace=False):
        up, dn = psi_t.copy(), psi_t.copy()
        up[e] += d
        dn[e] -= d
        fd = (model(up) - model(dn)) / (2 * d)
        assert abs(fd - g[e]) <= 1e-5 * max(1.0, abs(g[e]))


@pytest.mark.parametrize("method", ["lanczos", "power"])
def test_certified_bounds_hold_with_dense_reference(method):
    """test_rom.py:367-381: sigma_min equals the dense smallest eigenvalue and both certified
    bounds hold."""
    s = cantilever(8, 4)
    obj, rom, basis, rho, _ = rom_setup(s, n_snap=2, seed=3)
    rsol = rom.solve(basis, rho, obj)
    rep = rom.error_bounds(basis, rho, rsol, obj, mode="certified", method=method)
    k, free, kff = dense_kff(s, rho)
    assert rep.sigma_min_converged
    assert rep.sigma_min == pytest.approx(np.linalg.eigvalsh(kff)[0], rel=1e-6)
    u_star = np.zeros(s.mesh.n_dofs)
    u_star[free] = np.linalg.solve(kff, s.f[free])
    err_energy = np.sqrt((u_star - rsol.u) @ k @ (u_star - rsol.u))
    assert err_energy <= rep.energy_error_bound * (1 + 1e-6)
    assert abs(s.f @ u_star - rsol.j) <= rep.objective_error_bound * (1 + 1e-6)


@pytest.mark.parametrize("method", ["lanczos", "power"])
def test_sigma_min_failure_flag(method):
    """test_rom.py:396-402: one iteration cannot certify; the bounds stay None."""
    s = cantilever(8, 4)
    obj, rom, basis, rho, _ = rom_setup(s, n_snap=2, seed=3)
    rsol = rom.solve(basis, rho, obj)
    rep = rom.error_bounds(basis, rho, rsol, obj, mode="certified", power_max_iter=1, method=method)
    assert not rep.sigma_min_converged
    assert rep.energy_error_bound is None and rep.objective_error_bound is None


def test_filter_indicator_spreads_with_monotone_decay():
    """test_filtering.py:97-113: a single-element indicator spreads with monotone decay."""
    mesh = tb.build_mesh(8, 8, 1.0)
    psi = np.zeros(mesh.n_elems)
    psi[4 * 8 + 4] = 1.0
    rho = tb.HelmholtzFilter(mesh, 2.0).apply(psi).rho
    grid = rho.reshape(8, 8)
    assert np.all(np.diff(grid[4, 4:]) < 0) and np.all(np.diff(grid[4:, 4]) < 0)
    assert grid[4, 4] == rho.max()


def test_filter_adjoint_consistent_with_finite_differences():
    """test_filtering.py: d/dpsi of <c, rho(psi)> equals apply_adjoint(c) (the map is linear)."""
    mesh = tb.build_mesh(10, 6, 1.0)
    f = tb.HelmholtzFilter(mesh, 1.5)
    rng = np.random.default_rng(4)
    c = rng.standard_normal(mesh.n_elems)
    psi = rng.random(mesh.n_elems)
    g = f.apply_adjoint(c)
    for e in rng.choice(mesh.n_elems, 5, replace=False):
        up, dn = psi.copy(), psi.copy()
        up[e] += 1e-4
        dn[e] -= 1e-4
        fd = (c @ f.apply(up).rho - c @ f.apply(dn).rho) / 2e-4
        assert abs(fd - g[e]) <= 1e-8 * max(1.0, abs(g[e]))


def test_filter_load_vector_sums_to_domain_volume():
    """test_filtering.py: b(1) sums to the domain volume (the load is a partition of unity)."""
    mesh = tb.build_mesh(7, 3, 0.5)
    b = tb.HelmholtzFilter(mesh, 1.0).load_vector(np.ones(mesh.n_elems))
    assert abs(b.sum() - mesh.n_elems * mesh.elem_volume) <= 1e-12
