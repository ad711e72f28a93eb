"""Geometric multigrid preconditioner: same answers as the Jacobi path and
the reference, far fewer iterations."""

import numpy as np
import pytest

import paper_2004_05756_b200 as tb
from conftest import golden
from paper_2004_05756_b200 import configs

pytestmark = pytest.mark.gpu

MAT = tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP)


def nrel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / np.abs(np.asarray(b)).max()


def build(prob, pc, rtol=None):
    return tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed, MAT,
                        rtol=rtol or prob.rtol, preconditioner=pc)


def test_mg_cfg1_vs_reference_golden(cuda):
    G = golden("golden_cfg1.npz")
    prob = configs.cfg1()
    s = build(prob, "mg")
    obj = tb.ComplianceObjective(s.f)
    sol = s.solve(prob.psi, obj)
    assert abs(sol.j - G["j"]) <= 1e-8 * abs(G["j"])
    assert nrel(s.gradient(prob.psi, sol, obj), G["g"]) <= 1e-6
    jac = build(prob, "jacobi").solve(prob.psi, obj)
    assert sol.iterations < jac.iterations / 5


def test_mg_cfg2_vs_reference_golden(cuda):
    G = golden("golden_cfg2.npz")
    prob = configs.cfg2()
    s = build(prob, "mg")
    obj = tb.ComplianceObjective(s.f)
    sol = s.solve(prob.psi, obj)
    assert abs(sol.j - float(G["j"])) <= 1e-8 * abs(float(G["j"]))
    se = int(G["stride_e"])
    g = s.gradient(prob.psi, sol, obj)
    assert np.abs(g[::se] - G["g_s"]).max() <= 1e-6 * float(G["g_inf"])
    assert sol.iterations < 200


@pytest.mark.parametrize("dims", [(16, 8, 8), (24, 12, 12)])
def test_mg_3d_matches_jacobi(cuda, dims):
    prob = configs.cfg3(seed=4, nx=dims[0], ny=dims[1], nz=dims[2])
    obj = None
    out = {}
    for pc in ("jacobi", "mg"):
        s = build(prob, pc, rtol=1e-10)
        obj = tb.ComplianceObjective(s.f)
        sol = s.solve(prob.psi, obj)
        out[pc] = (sol.j, sol.u, s.gradient(prob.psi, sol, obj), sol.iterations)
    assert abs(out["mg"][0] - out["jacobi"][0]) <= 1e-8 * abs(out["jacobi"][0])
    assert nrel(out["mg"][2], out["jacobi"][2]) <= 1e-6
    assert out["mg"][3] < out["jacobi"][3] / 4


@pytest.mark.parametrize("dims", [(61, 23, None), (15, 9, 7), (25, 7, 11), (237, 61, None)])
def test_mg_odd_grids_match_jacobi(cuda, dims):
    """Odd element counts coarsen with a short last coarse element; the preconditioned answer
    is the Jacobi answer."""
    nx, ny, nz = dims
    prob = configs.cfg1(seed=2, nx=nx, ny=ny) if nz is None else configs.cfg3(seed=2, nx=nx, ny=ny, nz=nz)
    out = {}
    for pc in ("jacobi", "mg"):
        s = build(prob, pc, rtol=1e-10)
        obj = tb.ComplianceObjective(s.f)
        sol = s.solve(prob.psi, obj)
        out[pc] = (sol.j, s.gradient(prob.psi, sol, obj), sol.iterations)
    assert abs(out["mg"][0] - out["jacobi"][0]) <= 1e-8 * abs(out["jacobi"][0])
    assert nrel(out["mg"][1], out["jacobi"][1]) <= 1e-6
    assert out["mg"][2] < out["jacobi"][2] / 3


def test_mg_rejects_grids_without_a_coarse_level(cuda):
    mesh = tb.build_mesh(4, 2, 1.0)  # 30 dofs: already below the coarsest-level size
    f = np.zeros(mesh.n_dofs)
    f[-1] = -1.0
    left = mesh.boundary_nodes("left")
    with pytest.raises(ValueError):
        tb.HdmSolver(mesh, tb.elasticity_element_matrix(1.0, 0.3), tb.HelmholtzFilter(mesh, 1.5), f,
                     np.concatenate([2 * left, 2 * left + 1]), MAT, preconditioner="mg")


def test_mg_certified_error_bound_matches_jacobi(cuda):
    """Certified mode's inverse power iteration (rom.py:393-407) runs one pCG solve per step;
    with the multigrid preconditioner it converges to the same sigma_min."""
    prob = configs.cfg1(seed=1)
    out = {}
    for pc in ("jacobi", "mg"):
        s = build(prob, pc, rtol=1e-11)
        obj = tb.ComplianceObjective(s.f)
        snaps = [np.where(s.free_mask, s.solve(d, obj).u, 0.0) for d in prob.rom_designs[:3]]
        phi = tb.gram_schmidt(snaps)
        basis = tb.ReducedBasis(phi, None, None, phi.T @ s.f)
        rom = tb.RomModel(s)
        rho, _ = s.filtered_density(prob.psi)
        rs = rom.solve(basis, rho, obj)
        out[pc] = rom.error_bounds(basis, rho, rs, obj, mode="certified")
    assert out["mg"].sigma_min_converged and out["jacobi"].sigma_min_converged
    assert out["mg"].sigma_min == pytest.approx(out["jacobi"].sigma_min, rel=1e-6)
    assert out["mg"].energy_error_bound == pytest.approx(out["jacobi"].energy_error_bound, rel=1e-6)


@pytest.mark.parametrize("case", ["cfg1", "cfg2", "odd"])
def test_mg_2d_persistent_kernel_matches_graph_vcycle(cuda, monkeypatch, case):
    """2D MG-pCG runs as one persistent cooperative kernel (mgpcg2d.cu); with TB_NO_PERSIST the
    same V(2,2) cycle runs as the captured graph of mg.cu.  Same iterates up to the order of
    the dot-product sums: same iteration count (+-1), same answer to the solve tolerance."""
    prob = {"cfg1": configs.cfg1, "cfg2": configs.cfg2}.get(case, lambda: configs.cfg1(seed=3, nx=61, ny=23))()
    out = {}
    for mode in ("persistent", "graph"):
        if mode == "graph":
            monkeypatch.setenv("TB_NO_PERSIST", "1")
        s = build(prob, "mg", rtol=1e-10)
        obj = tb.ComplianceObjective(s.f)
        sol = s.solve(prob.psi, obj)
        out[mode] = (sol.j, sol.u, s.gradient(prob.psi, sol, obj), sol.iterations)
        monkeypatch.delenv("TB_NO_PERSIST", raising=False)
    (jp, up, gp, ip), (jg, ug, gg, ig) = out["persistent"], out["graph"]
    assert abs(ip - ig) <= 1
    assert abs(jp - jg) <= 1e-9 * abs(jg)
    assert nrel(up, ug) <= 1e-8
    assert nrel(gp, gg) <= 1e-7


def test_mg_2d_persistent_repeatable(cuda):
    """Deterministic reductions: back-to-back persistent solves are bit-identical."""
    prob = configs.cfg2()
    s = build(prob, "mg")
    obj = tb.ComplianceObjective(s.f)
    a = s.solve(prob.psi, obj)
    for _ in range(5):
        b = s.solve(prob.psi, obj)
        assert b.iterations == a.iterations
        assert np.array_equal(np.asarray(a.u), np.asarray(b.u))


def test_mg_2d_kernel_time_reported(cuda):
    """tb_pcg_kernel_time: the persistent launch of a 2D MG solve is timed on the solve's stream
    (the bench roofline reads it); the 3D graph path reports no persistent launch."""
    prob = configs.cfg1(seed=2)
    s = build(prob, "mg")
    s.solve(prob.psi, tb.ComplianceObjective(s.f))
    ms, launches = s.last_kernel_time()
    assert launches >= 1 and ms > 0.0
    p3 = configs.cfg3(seed=4, nx=16, ny=8, nz=8)
    s3 = build(p3, "mg", rtol=1e-10)
    s3.solve(p3.psi, tb.ComplianceObjective(s3.f))
    assert s3.last_kernel_time() == (0.0, 0)


@pytest.mark.parametrize("n", [192, 682, 1092])
def test_mg_gauss_jordan_coarsest_inverse(cuda, n):
    """The 2D coarsest inverse (k_mg_gj_inverse, blocked Gauss-Jordan) equals cuSOLVER's to
    round-off: same iterates of the preconditioned solve with either (TB_MG_CUSOLVER)."""
    import os

    dims = {192: (120, 40), 682: (120, 40), 1092: (600, 200)}[n]
    prob = configs.cfg1(seed=5, nx=dims[0], ny=dims[1])
    env = {192: "600", 682: "1200", 1092: "1200"}[n]
    out = {}
    for mode in ("gj", "cusolver"):
        os.environ["TB_MG_MIN_DOFS"] = env
        if mode == "cusolver":
            os.environ["TB_MG_CUSOLVER"] = "1"
        try:
            s = build(prob, "mg", rtol=1e-10)
            obj = tb.ComplianceObjective(s.f)
            sol = s.solve(prob.psi, obj)
            out[mode] = (sol.j, np.asarray(sol.u), sol.iterations)
        finally:
            os.environ.pop("TB_MG_MIN_DOFS", None)
            os.environ.pop("TB_MG_CUSOLVER", None)
    assert abs(out["gj"][2] - out["cusolver"][2]) <= 1
    assert abs(out["gj"][0] - out["cusolver"][0]) <= 1e-9 * abs(out["cusolver"][0])
    assert nrel(out["gj"][1], out["cusolver"][1]) <= 1e-8


def test_mg_elongated_grid_vs_oracle(cuda):
    """A slender 400 x 17 cantilever (not a BASELINE config): in fp64 the attainable true
    residual stagnates near 1e-9 here for multigrid (Jacobi-pCG near 1.5e-8).  A solve asked for
    less than that REPORTS it (NotConvergedError) instead of returning silently; a solve to 1e-8
    meets the north_star tolerances against the oracle's direct solve (J 1e-8, g 1e-6), and so
    does the drop-in's round-off mode (rtol=None)."""
    from oracle.fem import build_grid
    from oracle.hdm import Filter, Hdm, Material

    prob = configs.cfg1(seed=7, nx=400, ny=17)
    grid = build_grid(400, 17, 1.0)
    ora = Hdm(grid, prob.k_e, Filter(grid, prob.radius), prob.f, prob.fixed, Material(configs.RHO_L, configs.P_SIMP))
    ref = ora.solve(prob.psi)
    g_ref = ora.gradient(ref)
    for rtol in (1e-8, None):
        s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed, MAT,
                         rtol=rtol, preconditioner="mg")  # None: round-off mode
        obj = tb.ComplianceObjective(s.f)
        sol = s.solve(prob.psi, obj)
        g = s.gradient(prob.psi, sol, obj)
        assert abs(sol.j - ref["j"]) <= 1e-8 * abs(ref["j"])
        assert nrel(g, g_ref) <= 1e-6
    s = build(prob, "mg", rtol=1e-10)
    with pytest.raises(tb.NotConvergedError):
        s.solve(prob.psi, tb.ComplianceObjective(s.f))


_NOFUSE_SCRIPT = """
import sys, json
import numpy as np
import paper_2004_05756_b200 as tb
from paper_2004_05756_b200 import configs
prob = configs.cfg3(seed=4, nx=24, ny=12, nz=12)
s = tb.HdmSolver(prob.mesh, prob.k_e, tb.HelmholtzFilter(prob.mesh, prob.radius), prob.f, prob.fixed,
                 tb.MaterialModel(rho_l=configs.RHO_L, p=configs.P_SIMP), rtol=1e-10, preconditioner="mg")
sol = s.solve(prob.psi, tb.ComplianceObjective(s.f))
np.save(sys.argv[1], sol.u)
print(json.dumps({"j": sol.j, "iterations": sol.iterations}))
"""


def test_mg_3d_fused_epilogues_match_separate_kernels(cuda, tmp_path):
    """The V-cycle with the smoothing sweeps and residuals as operator-kernel epilogues (k_hex8
    EPI, k_mg_sapply EPI) against the separate update kernels (TB_MG_NOFUSE=1, read once per
    process: run in a child process): the same preconditioner up to rounding, so the same
    iteration count and solution."""
    import json
    import os
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for label, env in (("fused", {}), ("separate", {"TB_MG_NOFUSE": "1"})):
        path = str(tmp_path / f"u_{label}.npy")
        r = subprocess.run([sys.executable, "-c", _NOFUSE_SCRIPT, path], cwd=repo, capture_output=True, text=True,
                           env={**os.environ, **env, "PYTHONPATH": repo}, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        out[label] = (json.loads(r.stdout.strip().splitlines()[-1]), np.load(path))
    a, b = out["fused"], out["separate"]
    assert abs(a[0]["iterations"] - b[0]["iterations"]) <= 1
    assert abs(a[0]["j"] - b[0]["j"]) <= 1e-9 * abs(b[0]["j"])
    assert nrel(a[1], b[1]) <= 1e-7
