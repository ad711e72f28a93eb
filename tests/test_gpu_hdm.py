"""GPU parity of the HDM path (filter, pCG solve, compliance, sensitivity, adjoint, K(rho)v)
against golden vectors from the reference and against the CPU oracle.

Tolerances (BASELINE.json north_star): compliance 1e-8 relative;
sensitivities / gradients / filtered densities 1e-6 norm-wise relative; pure arithmetic
kernels (K(rho)v, filter transfers) 1e-12.
"""

import numpy as np
import torch
import pytest

import paper_2004_05756_b200 as tb
from conftest import golden
from oracle.fem import build_grid
from oracle.hdm import Filter, Hdm, Material
from paper_2004_05756_b200 import configs

pytestmark = pytest.mark.gpu

MAT = tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP)


def nrel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300)


def build(prob, rtol=None, mat=MAT):
    filt = tb.HelmholtzFilter(prob.mesh, prob.radius)
    return tb.HdmSolver(prob.mesh, prob.k_e, filt, prob.f, prob.fixed, mat, rtol=rtol or prob.rtol)


def make_cantilever(nx, ny, h=1.0, radius=None):
    """Reference tests/conftest.py:15-33 on the drop-in."""
    mesh = tb.build_mesh(nx, ny, h)
    filt = tb.HelmholtzFilter(mesh, 1.5 * h if radius is None else radius)
    f = np.zeros(mesh.n_dofs)
    f[2 * mesh.node_id(nx, ny // 2) + 1] = -1.0
    left = mesh.boundary_nodes("left")
    fixed = np.concatenate([2 * left, 2 * left + 1])
    return tb.HdmSolver(mesh, tb.elasticity_element_matrix(1.0, 0.3, h), filt, f, fixed, tb.MaterialModel(),
                        rtol=1e-12)


def test_cfg1_full_evaluation_vs_reference_golden(cuda):
    G = golden("golden_cfg1.npz")
    prob = configs.cfg1()
    s = build(prob)
    obj = tb.ComplianceObjective(s.f)
    res = s.filter.apply(prob.psi)
    assert nrel(res.rho, G["rho_raw"]) <= 1e-12
    assert nrel(res.phi, G["phi"]) <= 1e-12
    assert np.abs(s.filter.load_vector(prob.psi) - G["load"]).max() == 0.0  # same summation order
    sol = s.solve(prob.psi, obj)
    assert sol.lam is sol.u
    assert abs(sol.j - G["j"]) <= 1e-8 * abs(G["j"])
    assert np.max(np.abs(sol.rho - G["rho"]) / G["rho"]) <= 1e-6
    assert nrel(sol.u, G["u"]) <= 1e-6
    g = s.gradient(prob.psi, sol, obj)
    assert nrel(g, G["g"]) <= 1e-6
    sens = s.element_sensitivity(sol.rho, sol.u, sol.lam, obj)
    assert nrel(sens, G["s"]) <= 1e-6
    assert abs(sol.clamp_width - float(G["clamp_width"])) <= 1e-12
    assert s.stats.hdm_solves == 1 and s.stats.filter_solves == 1 and s.stats.factorizations == 1


def test_cfg1_kernels_exact_vs_reference(cuda):
    G = golden("golden_cfg1.npz")
    s = build(configs.cfg1())
    assert nrel(s.apply_stiffness(G["rho"], G["v"]), G["kv"]) <= 1e-13
    # sensitivity kernel on the reference's own state
    obj = tb.ComplianceObjective(s.f)
    assert nrel(s.element_sensitivity(G["rho"], G["u"], G["u"], obj), G["s"]) <= 1e-12
    assert nrel(s.filter.apply_adjoint(G["adj_v"]), G["adj"]) <= 1e-12


@pytest.mark.parametrize("nx,ny", [(6, 2), (12, 4), (4, 2)])
def test_reference_fixture_cantilevers(cuda, nx, ny):
    G = golden("golden_small.npz")
    key = f"cant{nx}x{ny}"
    s = make_cantilever(nx, ny)
    obj = tb.ComplianceObjective(s.f)
    sol = s.solve(G[f"{key}_psi"], obj)
    assert abs(sol.j - G[f"{key}_j"]) <= 1e-10 * abs(G[f"{key}_j"])
    assert nrel(sol.u, G[f"{key}_u"]) <= 1e-9
    assert nrel(s.gradient(G[f"{key}_psi"], sol, obj), G[f"{key}_g"]) <= 1e-8


def test_filter_reference_fixtures(cuda):
    G = golden("golden_small.npz")
    for nx, ny, h, radius in ((4, 3, 0.25, 0.3), (12, 12, 0.25, 0.25), (6, 9, 0.25, 0.0), (8, 5, 0.25, 0.6),
                              (9, 5, 0.2, 2.0)):
        key = f"filt{nx}x{ny}_{h}_{radius}"
        f = tb.HelmholtzFilter(tb.build_mesh(nx, ny, h), radius)
        assert np.abs(f.apply(G[f"{key}_psi"]).rho - G[f"{key}_rho"]).max() < 1e-11  # reference tolerance
        assert np.abs(f.apply_adjoint(G[f"{key}_v"]) - G[f"{key}_adj"]).max() < 1e-11


def test_filter_identities(cuda):
    # reference tests/test_filtering.py:12-94
    mesh = tb.build_mesh(8, 5, 0.25)
    f = tb.HelmholtzFilter(mesh, 0.6)
    res = f.apply(np.full(mesh.n_elems, 0.5))
    assert np.abs(res.rho - 0.5).max() < 1e-12 and np.abs(res.phi - 0.5).max() < 1e-12
    mesh = tb.build_mesh(10, 6, 0.2)
    f = tb.HelmholtzFilter(mesh, 0.5)
    rng = np.random.default_rng(0)
    for _ in range(5):
        psi = rng.random(mesh.n_elems)
        assert abs(f.apply(psi).rho.sum() - psi.sum()) <= 1e-10 * psi.sum()
    p1, p2 = rng.random(mesh.n_elems), rng.random(mesh.n_elems)
    lhs = f.apply(0.7 * p1 - 1.3 * p2).rho
    assert np.abs(lhs - (0.7 * f.apply(p1).rho - 1.3 * f.apply(p2).rho)).max() < 1e-12
    for radius in (0.0, 0.3, 2.0):
        m = tb.build_mesh(9, 5, 0.2)
        assert np.abs(tb.HelmholtzFilter(m, radius).apply_adjoint(np.ones(m.n_elems)) - 1.0).max() < 1e-10
    with pytest.raises(ValueError):
        f.apply(np.ones(5))
    with pytest.raises(ValueError):
        tb.HelmholtzFilter(mesh, -0.1)


def test_oracle_parity_random_sizes(cuda):
    for nx, ny, seed in ((30, 10, 1), (64, 32, 2)):
        prob = configs.cfg1(seed=seed, nx=nx, ny=ny)
        s = build(prob, rtol=1e-12)
        g = build_grid(nx, ny, 1.0)
        ora = Hdm(g, prob.k_e, Filter(g, prob.radius), prob.f, prob.fixed, Material(configs.RHO_L, configs.P_SIMP))
        obj = tb.ComplianceObjective(s.f)
        sol = s.solve(prob.psi, obj)
        ref = ora.solve(prob.psi)
        assert abs(sol.j - ref["j"]) <= 1e-8 * abs(ref["j"])
        assert nrel(s.gradient(prob.psi, sol, obj), ora.gradient(ref)) <= 1e-6
        # true residual of the returned state
        k = ora.stiffness(sol.rho)
        r = (k @ sol.u - ora.f)[ora.free_mask]
        assert np.linalg.norm(r) <= 1e-11 * np.linalg.norm(ora.f)


class SyntheticObjective(tb.Objective):
    """Reference tests/oracles.py:161-181: j = f^T u + |u|^2/2 + |rho|^2."""

    def __init__(self, f):
        self.f = np.asarray(f, float)

    def value(self, u, rho):
        return float(self.f @ u + 0.5 * u @ u + rho @ rho)

    def du(self, u, rho):
        return self.f + u

    def drho(self, u, rho):
        return 2.0 * rho


def test_general_objective_adjoint_path(cuda):
    prob = configs.cfg1(seed=4, nx=24, ny=8)
    s = build(prob, rtol=1e-10)
    obj = SyntheticObjective(s.f)
    sol = s.solve(prob.psi, obj)
    assert s.stats.hdm_adjoint_solves == 1
    g = build_grid(24, 8, 1.0)
    ora = Hdm(g, prob.k_e, Filter(g, prob.radius), prob.f, prob.fixed, Material(configs.RHO_L, configs.P_SIMP))
    ref = ora.solve(prob.psi, du=lambda u, rho: ora.f + u)
    assert nrel(sol.lam, ref["lam"]) <= 1e-6
    grad = s.gradient(prob.psi, sol, obj)
    assert nrel(grad, ora.gradient(ref, drho=2.0 * ref["rho"])) <= 1e-6


def test_error_behaviour(cuda):
    s = make_cantilever(6, 2)
    obj = tb.ComplianceObjective(s.f)
    psi = np.full(s.mesh.n_elems, 0.5)
    sol = s.solve(psi, obj)
    other = psi.copy()
    other[0] += 0.01
    with pytest.raises(tb.StaleSolutionError):
        s.gradient(other, sol, obj)
    with pytest.raises(ValueError):
        s.solve(np.ones(3), obj)
    # no Dirichlet conditions: rigid modes make K singular -> IndefiniteMatrixError or no convergence
    mesh = tb.build_mesh(4, 2, 1.0)
    f = np.zeros(mesh.n_dofs)
    f[1] = 1.0
    free = tb.HdmSolver(mesh, tb.elasticity_element_matrix(1.0, 0.3), tb.HelmholtzFilter(mesh, 1.0), f,
                        np.array([], dtype=np.int64), tb.MaterialModel(), maxit=500)
    with pytest.raises((tb.IndefiniteMatrixError, tb.NotConvergedError)):
        free.solve(np.full(mesh.n_elems, 0.5), tb.ComplianceObjective(free.f))


def test_deterministic_and_native_mode(cuda):
    import torch

    prob = configs.cfg1(seed=9, nx=48, ny=16)
    s = build(prob)
    obj = tb.ComplianceObjective(s.f)
    a = s.solve(prob.psi, obj)
    b = s.solve(prob.psi, obj)
    assert a.j == b.j and np.array_equal(a.u, b.u)
    ga, gb = s.gradient(prob.psi, a, obj), s.gradient(prob.psi, b, obj)
    assert np.array_equal(ga, gb)
    psi_t = torch.as_tensor(prob.psi, device=cuda)
    c = s.solve(psi_t, obj)
    assert isinstance(c.u, torch.Tensor) and c.u.is_cuda
    assert c.j == a.j and np.array_equal(c.u.cpu().numpy(), a.u)
    gc = s.gradient(psi_t, c, obj)
    assert np.array_equal(gc.cpu().numpy(), ga)
    assert c.psi_hash == a.psi_hash
    with pytest.raises(tb.StaleSolutionError):
        s.gradient(psi_t + 1e-3, c, obj)


def test_compliance_identity(cuda):
    # reference tests/test_hdm.py:99-106
    s = make_cantilever(12, 4)
    obj = tb.ComplianceObjective(s.f)
    sol = s.solve(np.full(s.mesh.n_elems, 0.4), obj)
    k = s.assemble_stiffness(sol.rho)
    assert abs(sol.j - s.f @ sol.u) <= 1e-12 * abs(sol.j)
    assert abs(sol.j - sol.u @ (k @ sol.u)) <= 1e-9 * abs(sol.j)


def test_gradient_finite_differences(cuda):
    # reference tests/test_hdm.py:175-188
    s = make_cantilever(12, 4)
    obj = tb.ComplianceObjective(s.f)
    rng = np.random.default_rng(12)
    psi = 0.25 + 0.5 * rng.random(s.mesh.n_elems)
    sol = s.solve(psi, obj)
    g = s.gradient(psi, sol, obj)
    # the reference uses d = 1e-6 with a direct solver; with pCG at rtol 1e-12, J carries
    # ~1e-12 relative solve noise, which a 2e-6 difference quotient amplifies to ~1e-4.
    # d = 1e-5 keeps that noise 10x smaller; the O(d^2) truncation error stays ~1e-10.
    d = 1e-5
    for e in rng.choice(s.mesh.n_elems, 6, replace=False):
        up, dn = psi.copy(), psi.copy()
        up[e] += d
        dn[e] -= d
        fd = (s.solve(up, obj).j - s.solve(dn, obj).j) / (2 * d)
        assert abs(fd - g[e]) <= 1e-5 * max(1.0, abs(g[e]))


def test_persistent_pcg_repeats_bit_identical(cuda):
    """The persistent 2D kernel decides convergence redundantly in every CTA from parity-buffered
    partial sums; 200 back-to-back solves must all finish and agree bit for bit (a shared
    partial buffer once let a CTA race ahead, desynchronise the branch and deadlock)."""
    prob = configs.cfg1(seed=3)
    s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed,
                     tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=1e-10)
    rho, _ = s.filtered_density_device(torch.as_tensor(prob.psi, device=cuda))
    ref = s.pcg_device(rho, s._f_d).clone()
    for _ in range(200):
        assert torch.equal(s.pcg_device(rho, s._f_d), ref)


def test_graph_path_matches_persistent_kernel(cuda, monkeypatch):
    """2D grids too large for the persistent kernel's shared memory run the graph-captured
    pCG (k_pcg_fused + k_pcg_update under a conditional node); forced here on cfg 1."""
    G = golden("golden_cfg1.npz")
    prob = configs.cfg1()
    obj_sol = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("TB_NO_PERSIST", env)
        s = build(prob, rtol=1e-10)
        obj = tb.ComplianceObjective(s.f)
        sol = s.solve(prob.psi, obj)
        obj_sol.append((sol.j, s.gradient(prob.psi, sol, obj)))
    monkeypatch.delenv("TB_NO_PERSIST")
    for j, g in obj_sol:
        assert abs(j - float(G["j"])) <= 1e-8 * abs(float(G["j"]))
        assert np.abs(g - G["g"]).max() <= 1e-6 * np.abs(G["g"]).max()


def test_integration_md_ctypes_stub(cuda):
    """The raw-ctypes binding shown in INTEGRATION.md §2 (what a romtopt maintainer would add)
    runs as written and reproduces HdmSolver's solve."""
    import ctypes

    import torch

    from paper_2004_05756_b200 import _lib

    prob = configs.cfg1(seed=6, nx=24, ny=8)
    mesh = prob.mesh
    lib = ctypes.CDLL(_lib.LIB_PATH)
    P, I, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
    lib.tb_plan_create.argtypes = [I, I, I, I, D, P, D, D, P, I, ctypes.POINTER(P)]
    lib.tb_pcg_solve.argtypes = [P, P, P, P, D, I, ctypes.POINTER(I), ctypes.POINTER(D), P]
    lib.tb_plan_destroy.argtypes = [P]
    lib.tb_last_error.restype = ctypes.c_char_p
    k_e = np.ascontiguousarray(tb.elasticity_element_matrix(1.0, 0.3))
    fixed = np.zeros(mesh.n_dofs, np.uint8)
    fixed[prob.fixed] = 1
    plan = P()
    assert lib.tb_plan_create(2, mesh.nx, mesh.ny, 0, mesh.h, k_e.ctypes.data, 1e-9, 3.0, fixed.ctypes.data,
                              cuda.index or 0, ctypes.byref(plan)) == 0, lib.tb_last_error()
    s = build(prob, rtol=1e-10)
    rho, _ = s.filtered_density(prob.psi)
    rho_d = torch.as_tensor(rho, device=cuda)
    f_d = torch.as_tensor(np.where(fixed == 0, prob.f, 0.0), device=cuda)
    u_d = torch.empty_like(f_d)
    it, rr = I(), D()
    rc = lib.tb_pcg_solve(plan, rho_d.data_ptr(), f_d.data_ptr(), u_d.data_ptr(), 1e-10, 200000, ctypes.byref(it),
                          ctypes.byref(rr), torch.cuda.current_stream().cuda_stream)
    assert rc == 0, lib.tb_last_error()
    lib.tb_plan_destroy(plan)
    u_ref = s.pcg_device(torch.as_tensor(rho, device=cuda), s._f_d)
    assert torch.equal(u_d, u_ref)
