"""Seeded synthetic inputs for the five BASELINE.json configurations.

Every builder is a pure function of (seed, grid size) and returns host numpy data shared
byte-for-byte by the GPU path and the CPU oracle.  Default sizes are BASELINE's; smaller
sizes give the parity variants of the same recipe.  Decisions the BASELINE text leaves
open are fixed here and recorded in DESIGN.md:

* material E0 = 1, nu = 0.3, MaterialModel(rho_l = 1e-9, p = 3) (G4); h = 1, so filter
  radii are in element units and are the reference's R (G3);
* cfg 3/5 load: f_z totalling -1 along the edge (x = Lx, z = 0), trapezoid weights;
* cfg 4 (G6): u_x = 0 on x = 0, u_z = 0 on the line (x = Lx, z = 0), plus u_y = 0 on
  y = 0 (quarter-symmetry plane) and an f_z line load totalling -1 along (x = 0, z = Lz);
  filter R = 2.5 as cfg 3;
* seeds default to 0 (G9).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .fem import StructuredMesh, build_mesh, build_mesh_3d, elasticity_element_matrix, hex8_element_matrix

E0, NU, RHO_L, P_SIMP = 1.0, 0.3, 1e-9, 3.0


@dataclass
class Problem:
    name: str
    mesh: StructuredMesh
    k_e: np.ndarray
    f: np.ndarray
    fixed: np.ndarray
    radius: float
    rtol: float
    psi: np.ndarray
    rom_k: int = 0
    rom_designs: list = field(default_factory=list)
    notes: str = ""

    @property
    def n_free(self) -> int:
        return self.mesh.n_dofs - self.fixed.size


def _node_ids_3d(mesh, i, j, k):
    return (np.asarray(k) * (mesh.ny + 1) + np.asarray(j)) * (mesh.nx + 1) + np.asarray(i)


def _trapezoid(n_edges):
    w = np.full(n_edges + 1, 1.0 / n_edges)
    w[0] = w[-1] = 0.5 / n_edges
    return w


def _perturbed(rng, base, count, lo, hi):
    return [np.clip(base * (1.0 + rng.uniform(-0.05, 0.05, base.size)), lo, hi) for _ in range(count)]


def cfg1(seed: int = 0, nx: int = 120, ny: int = 40) -> Problem:
    """2D half-MBB: u_x = 0 on the left edge, u_y = 0 at node (nx, 0), f_y = -1 at (0, ny);
    psi ~ U[0.01, 1] i.i.d.; R = 1.5; ROM k = 10 from ±5% perturbations."""
    mesh = build_mesh(nx, ny, 1.0)
    f = np.zeros(mesh.n_dofs)
    f[2 * mesh.node_id(0, ny) + 1] = -1.0
    fixed = np.unique(np.concatenate([2 * mesh.boundary_nodes("left"), [2 * mesh.node_id(nx, 0) + 1]]))
    rng = np.random.default_rng(seed)
    psi = rng.uniform(0.01, 1.0, mesh.n_elems)
    designs = _perturbed(rng, psi, 10, 0.0, 1.0)
    return Problem("cfg1-halfmbb-2d", mesh, elasticity_element_matrix(E0, NU), f, fixed.astype(np.int64), 1.5,
                   1e-10, psi, 10, designs)


def cfg2(seed: int = 0, nx: int = 600, ny: int = 200) -> Problem:
    """2D cantilever: left edge clamped, f_y = -1 at (nx, ny//2); smooth seeded field; R = 3;
    pCG to 1e-10; ROM k = 32."""
    mesh = build_mesh(nx, ny, 1.0)
    f = np.zeros(mesh.n_dofs)
    f[2 * mesh.node_id(nx, ny // 2) + 1] = -1.0
    left = mesh.boundary_nodes("left")
    fixed = np.unique(np.concatenate([2 * left, 2 * left + 1]))
    rng = np.random.default_rng(seed)
    a, b = rng.integers(1, 5, 2)
    e = np.arange(mesh.n_elems)
    x = (e % nx + 0.5) / nx
    y = (e // nx + 0.5) / ny
    psi = np.clip(0.5 + 0.4 * np.sin(2 * np.pi * a * x) * np.cos(2 * np.pi * b * y), 0.01, 1.0)
    designs = _perturbed(rng, psi, 32, 0.0, 1.0)
    return Problem("cfg2-cantilever-2d", mesh, elasticity_element_matrix(E0, NU), f, fixed.astype(np.int64), 3.0,
                   1e-10, psi, 32, designs, notes=f"a={a}, b={b}")


def _cantilever3d(mesh):
    """Face x = 0 clamped; f_z totalling -1 along the edge (x = Lx, z = 0)."""
    f = np.zeros(mesh.n_dofs)
    j = np.arange(mesh.ny + 1)
    f[3 * _node_ids_3d(mesh, mesh.nx, j, 0) + 2] = -_trapezoid(mesh.ny)
    left = mesh.boundary_nodes("left")
    fixed = np.unique(np.concatenate([3 * left, 3 * left + 1, 3 * left + 2]))
    return f, fixed.astype(np.int64)


def cfg3(seed: int = 0, nx: int = 192, ny: int = 96, nz: int = 96, prefilter=None) -> Problem:
    """3D cantilever; psi0 ~ U[0.01, 1] pre-filtered with R = 2 by ``prefilter(psi0)``
    (a HelmholtzFilter(mesh, 2.0).apply(.).rho, device or oracle), clipped to [0.01, 1];
    filter R = 2.5; pCG to 1e-8."""
    mesh = build_mesh_3d(nx, ny, nz, 1.0)
    f, fixed = _cantilever3d(mesh)
    rng = np.random.default_rng(seed)
    psi0 = rng.uniform(0.01, 1.0, mesh.n_elems)
    psi = psi0 if prefilter is None else np.clip(np.asarray(prefilter(mesh, psi0)), 0.01, 1.0)
    return Problem("cfg3-cantilever-3d", mesh, hex8_element_matrix(E0, NU), f, fixed, 2.5, 1e-8, psi,
                   notes="prefiltered R=2" if prefilter is not None else "NOT prefiltered")


def cfg4(seed: int = 0, nx: int = 384, ny: int = 192, nz: int = 192) -> Problem:
    """3D MBB/bridge box (quarter model, see module docstring); 50/50 blend of U[0.01, 1] and a
    Gaussian(sigma = 4)-smoothed noise field thresholded at volume fraction 0.3."""
    from scipy.ndimage import gaussian_filter

    mesh = build_mesh_3d(nx, ny, nz, 1.0)
    f = np.zeros(mesh.n_dofs)
    j = np.arange(ny + 1)
    f[3 * _node_ids_3d(mesh, 0, j, nz) + 2] = -_trapezoid(ny)
    left = mesh.boundary_nodes("left")
    bottom_y = mesh.boundary_nodes("bottom")
    support = _node_ids_3d(mesh, nx, j, 0)
    fixed = np.unique(np.concatenate([3 * left, 3 * bottom_y + 1, 3 * support + 2])).astype(np.int64)
    rng = np.random.default_rng(seed)
    uni = rng.uniform(0.01, 1.0, mesh.n_elems)
    noise = rng.standard_normal((nz, ny, nx))
    smooth = gaussian_filter(noise, sigma=4.0, mode="reflect").ravel()
    thr = np.quantile(smooth, 0.7)
    blob = np.where(smooth >= thr, 1.0, 0.01)
    psi = 0.5 * uni + 0.5 * blob
    return Problem("cfg4-mbb-3d", mesh, hex8_element_matrix(E0, NU), f, fixed, 2.5, 1e-8, psi)


def cfg5(seed: int = 0, nx: int = 256, ny: int = 128, nz: int = 128, n_designs: int = 16, k: int = 64) -> Problem:
    """Batched ROM build on the cfg-3 geometry: base U[0.01, 1], n_designs ±5% perturbations
    (clipped to [0.01, 1]); basis: ``phi_columns`` (k sums of 8 seeded sine modes) then MGS."""
    mesh = build_mesh_3d(nx, ny, nz, 1.0)
    f, fixed = _cantilever3d(mesh)
    rng = np.random.default_rng(seed)
    base = rng.uniform(0.01, 1.0, mesh.n_elems)
    designs = _perturbed(rng, base, n_designs, 0.01, 1.0)
    return Problem("cfg5-rom-3d", mesh, hex8_element_matrix(E0, NU), f, fixed, 2.5, 1e-8, base, k, designs)


def phi_mode_params(seed: int, k: int):
    """Per column c and displacement component d: 8 (amplitude, p, q, r) sine modes."""
    rng = np.random.default_rng(seed + 7919)
    amp = rng.standard_normal((k, 3, 8))
    pqr = rng.integers(1, 5, (k, 3, 8, 3))
    return amp, pqr


def phi_columns(mesh: StructuredMesh, k: int, seed: int = 0, xp=np, device=None):
    """(k, n_dofs) raw basis columns: column c, component d =
    sum_m a_m sin(pi (p_m - 1/2) x/Lx) cos(pi (q_m - 1) y/Ly) cos(pi (r_m - 1) z/Lz) at the
    nodes, p, q, r in [1, 4]; fixed dofs are zeroed by the caller.  ``xp`` may be numpy or torch (device generation for cfg 5)."""
    amp, pqr = phi_mode_params(seed, k)
    nnx, nny, nnz = mesh.nx + 1, mesh.ny + 1, mesh.nz + 1
    kw = {} if xp is np else {"device": device, "dtype": xp.float64}
    ar = (lambda n: xp.arange(n, **kw)) if xp is not np else (lambda n: np.arange(n, dtype=float))
    x, y, z = ar(nnx) / mesh.nx, ar(nny) / mesh.ny, ar(nnz) / mesh.nz
    out = xp.zeros((k, mesh.n_nodes, 3), **kw)
    pi = np.pi
    for c in range(k):
        for d in range(3):
            acc = xp.zeros((nnz, nny, nnx), **kw)
            for m in range(8):
                p, q, r = (int(v) for v in pqr[c, d, m])
                # quarter-wave in x (vanishes on the clamped face x = 0, not on the loaded
                # edge x = Lx), cosines in y and z
                sx, sy, sz = xp.sin(pi * (p - 0.5) * x), xp.cos(pi * (q - 1) * y), xp.cos(pi * (r - 1) * z)
                acc = acc + float(amp[c, d, m]) * (sz[:, None, None] * sy[None, :, None] * sx[None, None, :])
            out[c, :, d] = acc.reshape(-1)
    return out.reshape(k, -1)


ALL = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5}
