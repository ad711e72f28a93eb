"""Device trust-region subproblem against the reference
TrustRegionDriver.solve_subproblem run on the same centre and basis (golden_subproblem.npz)."""

import numpy as np
import pytest
import torch

import paper_2004_05756_b200 as tb
from conftest import golden
from paper_2004_05756_b200 import configs

pytestmark = pytest.mark.gpu


def setup():
    G = golden("golden_subproblem.npz")
    prob = configs.cfg1(seed=4, nx=48, ny=16)  # recipe of make_golden.subproblem_setup
    psi_k = np.clip(0.9 * prob.psi, 0.0, 1.0)
    assert np.array_equal(psi_k, G["psi_k"])
    solver = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed,
                          tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=1e-12)
    obj = tb.ComplianceObjective(solver.f)
    phi = G["phi"]
    basis = tb.ReducedBasis(phi, None, None, phi.T @ solver.f)
    w = np.ones(prob.mesh.n_elems)
    return G, prob, psi_k, solver, obj, basis, w


@pytest.mark.parametrize("kind", ["res", "dist"])
def test_subproblem_matches_reference(cuda, kind):
    G, prob, psi_k, solver, obj, basis, w = setup()
    sol = solver.solve(psi_k, obj)
    g = solver.gradient(psi_k, sol, obj)
    assert abs(sol.j - float(G["j_center"])) <= 1e-8 * abs(float(G["j_center"]))
    sp = tb.TrustRegionSubproblem(solver, tb.RomModel(solver), obj, w, float(G["cap"]), constraint=kind,
                                  max_inner=int(G[f"{kind}_inner"]))
    before = solver.stats.rom_solves
    r = sp.solve_subproblem(basis, psi_k, float(G[f"{kind}_delta"]), sol.j, g)
    assert r.steps == int(G[f"{kind}_steps"])
    assert r.rom_solves == int(G[f"{kind}_rom_solves"])
    assert solver.stats.rom_solves - before == r.rom_solves
    assert isinstance(r.candidate, np.ndarray)
    assert np.abs(r.candidate - G[f"{kind}_candidate"]).max() <= 1e-6
    assert np.abs(r.first_iterate - G[f"{kind}_first"]).max() <= 1e-6
    assert r.model_value == pytest.approx(float(G[f"{kind}_model_value"]), rel=1e-8)
    assert r.theta == pytest.approx(float(G[f"{kind}_theta"]), rel=1e-6, abs=1e-12)
    assert r.curvature == pytest.approx(float(G[f"{kind}_curvature"]), rel=1e-6)


def test_subproblem_device_tensors(cuda):
    """Native mode: the whole sweep runs on device tensors and returns them."""
    G, prob, psi_k, solver, obj, basis, w = setup()
    psi_d = torch.as_tensor(psi_k, device=cuda)
    sol = solver.solve(psi_d, obj)
    g = solver.gradient(psi_d, sol, obj)
    sp = tb.TrustRegionSubproblem(solver, tb.RomModel(solver), obj, torch.as_tensor(w, device=cuda),
                                  float(G["cap"]), constraint="res", max_inner=int(G["res_inner"]))
    r = sp.solve_subproblem(basis, psi_d, float(G["res_delta"]), sol.j, g)
    assert r.candidate.is_cuda and r.first_iterate.is_cuda
    assert r.steps == int(G["res_steps"])
    assert np.abs(r.candidate.cpu().numpy() - G["res_candidate"]).max() <= 1e-6


def test_constraint_kinds():
    with pytest.raises(ValueError):
        tb.TrustRegionSubproblem.__init__(object.__new__(tb.TrustRegionSubproblem), None, None, None, None, 1.0,
                                          constraint="box")
