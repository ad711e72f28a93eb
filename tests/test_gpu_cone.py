"""Cone ("linear hat") density filter against oracle/filters.py, plus the
identities of a normalised averaging filter and its exact transpose; drop-in for HdmSolver."""

import numpy as np
import pytest

import paper_2004_05756_b200 as tb
from oracle.filters import cone_matrix
from paper_2004_05756_b200 import configs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims,h,radius", [((24, 8, None), 1.0, 1.5), ((60, 20, None), 0.5, 1.6),
                                           ((12, 6, 5), 1.0, 2.5), ((9, 7, 4), 2.0, 3.0),
                                           ((10, 5, None), 1.0, 0.0)])
def test_cone_filter_vs_oracle(cuda, dims, h, radius):
    nx, ny, nz = dims
    mesh = tb.build_mesh(nx, ny, h) if nz is None else tb.build_mesh_3d(nx, ny, nz, h)
    f = tb.ConeFilter(mesh, radius)
    a = cone_matrix(nx, ny, nz or 0, h, radius)
    rng = np.random.default_rng(7)
    psi = rng.uniform(0.01, 1.0, mesh.n_elems)
    v = rng.standard_normal(mesh.n_elems)
    rho = f.apply(psi).rho
    assert np.abs(rho - a @ psi).max() <= 1e-13
    w = f.apply_adjoint(v)
    assert np.abs(w - a.T @ v).max() <= 1e-12 * max(1.0, np.abs(w).max())
    assert np.abs(f.apply(np.ones(mesh.n_elems)).rho - 1.0).max() <= 1e-14  # partition of unity
    assert abs(rho @ v - psi @ w) <= 1e-12 * abs(psi @ w)                   # exact transpose
    assert rho.min() >= psi.min() - 1e-15 and rho.max() <= psi.max() + 1e-15  # convex averages


def test_cone_filter_in_hdm_solver(cuda):
    """HdmSolver with the cone filter: gradient matches finite differences of J."""
    prob = configs.cfg1(seed=5, nx=16, ny=6)
    s = tb.HdmSolver(prob.mesh, prob.k_e, tb.ConeFilter(prob.mesh, 1.5), prob.f, prob.fixed,
                     tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=1e-12)
    obj = tb.ComplianceObjective(s.f)
    psi = prob.psi
    sol = s.solve(psi, obj)
    g = s.gradient(psi, sol, obj)
    rng = np.random.default_rng(3)
    for e in rng.choice(prob.mesh.n_elems, 4, replace=False):
        d = 1e-5
        up, dn = psi.copy(), psi.copy()
        up[e] += d
        dn[e] -= d
        fd = (s.solve(up, obj).j - s.solve(dn, obj).j) / (2 * d)
        assert abs(fd - g[e]) <= 1e-5 * max(1.0, abs(g[e]))


def test_cone_filter_rejects_bad_input(cuda):
    mesh = tb.build_mesh(4, 2, 1.0)
    with pytest.raises(ValueError):
        tb.ConeFilter(mesh, -1.0)
    f = tb.ConeFilter(mesh, 1.2)
    with pytest.raises(ValueError):
        f.apply(np.ones(3))
