"""Oracle HDM evaluation: Helmholtz filter, SIMP material, solve, sensitivity, K(rho)v.

Restates reference filtering.py:47-114 and hdm.py:40-233 (numpy/scipy).
Dimension generic: 2D Q4 follows the reference exactly; 3D Hex8 uses the
same formulas with 2^3 nodes per element and h^3 element volume.
"""

from __future__ import annotations

import hashlib

import numpy as np
import scipy.sparse as sp

from .fem import DirectSolver, Grid, assemble, helmholtz_element_matrices

LENGTH_SCALE_FACTOR = 1.0 / (2.0 * np.sqrt(3.0))  # reference filtering.py:29-32


class Material:
    """alpha(rho) = rho_l + (1-rho_l) rho^p (reference hdm.py:40-55)."""

    def __init__(self, rho_l=1e-3, p=3.0):
        self.rho_l, self.p = rho_l, p

    def alpha(self, rho):
        return self.rho_l + (1.0 - self.rho_l) * rho**self.p

    def dalpha(self, rho):
        return (1.0 - self.rho_l) * self.p * rho ** (self.p - 1.0)


class Filter:
    """PDE filter with radius R (reference filtering.py:47-114)."""

    def __init__(self, grid: Grid, radius: float):
        if radius < 0:
            raise ValueError("radius")
        self.grid = grid
        self.radius = float(radius)
        self.r = LENGTH_SCALE_FACTOR * self.radius
        self.npe = 2**grid.dim
        h_e, self.b_e = helmholtz_element_matrices(self.r, grid.h, grid.dim)
        rows = grid.elem_nodes.ravel()
        cols = np.repeat(np.arange(grid.n_elems), self.npe)
        self.inc = sp.csr_matrix((np.ones(rows.size), (rows, cols)), shape=(grid.n_nodes, grid.n_elems))
        self.H = assemble(grid, h_e, None, scalar=True)
        self.fact = DirectSolver(self.H)

    def load_vector(self, psi):  # filtering.py:73-76
        return self.inc @ (psi * (self.grid.elem_volume / self.npe))

    def apply(self, psi):  # filtering.py:78-97 -> (phi, rho)
        psi = np.asarray(psi, float)
        phi = self.fact.solve(self.load_vector(psi))
        return phi, (self.inc.T @ phi) / self.npe

    def apply_adjoint(self, v):  # filtering.py:99-114
        q = self.inc @ (np.asarray(v, float) / self.npe)
        mu = self.fact.solve(q)
        return (self.inc.T @ mu) * (self.grid.elem_volume / self.npe)


def digest(psi):  # hdm.py:36-37
    return hashlib.sha256(np.ascontiguousarray(psi, dtype=float).tobytes()).hexdigest()


class Hdm:
    """Full-order evaluation (reference hdm.py:112-233) for compliance j = f^T u."""

    def __init__(self, grid: Grid, k_e, filt: Filter, f, fixed, material: Material):
        self.grid, self.k_e, self.filter, self.material = grid, np.asarray(k_e, float), filt, material
        self.fixed = np.asarray(fixed, np.int64)
        f = np.asarray(f, float).copy()
        f[self.fixed] = 0.0  # hdm.py:136-137
        self.f = f
        self.free_mask = np.ones(grid.n_dofs, bool)
        self.free_mask[self.fixed] = False

    def filtered_density(self, psi):  # hdm.py:144-154
        _, rho_raw = self.filter.apply(psi)
        rho = np.clip(rho_raw, self.material.rho_l, 1.0)
        return rho, float(np.max(np.abs(rho - rho_raw), initial=0.0))

    def stiffness(self, rho):
        return assemble(self.grid, self.k_e, self.material.alpha(rho))

    def solve(self, psi, du=None):
        """hdm.py:170-197.  ``du`` = callable(u, rho) for a non-compliance objective."""
        rho, cw = self.filtered_density(psi)
        lo = self.material.rho_l
        if rho.min() < lo - 1e-12 or rho.max() > 1 + 1e-12:  # hdm.py:156-162
            raise ValueError("density out of range")
        fact = DirectSolver(self.stiffness(rho), self.fixed)
        u = fact.solve(self.f)
        lam = u if du is None else fact.solve(du(u, rho))
        return dict(rho=rho, u=u, lam=lam, j=float(self.f @ u), clamp_width=cw,
                    psi_hash=digest(psi), fact=fact)

    def element_sensitivity(self, rho, u, lam, drho=None):  # hdm.py:211-222
        ul = u[self.grid.elem_dofs]
        ll = lam[self.grid.elem_dofs]
        c = ((ul @ self.k_e) * ll).sum(axis=1)
        base = np.zeros(rho.shape[0]) if drho is None else drho
        return base - self.material.dalpha(rho) * c

    def gradient(self, sol, drho=None):  # hdm.py:199-209
        s = self.element_sensitivity(sol["rho"], sol["u"], sol["lam"], drho)
        return self.filter.apply_adjoint(s)

    def apply_stiffness(self, rho, v):  # hdm.py:224-233
        contrib = (v[self.grid.elem_dofs] @ self.k_e.T) * self.material.alpha(rho)[:, None]
        out = np.bincount(self.grid.elem_dofs.ravel(), weights=contrib.ravel(), minlength=self.grid.n_dofs)
        out[~self.free_mask] = 0.0
        return out
