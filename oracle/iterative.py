"""Matrix-free CPU restatement for the large 3D configs -- TEST INFRASTRUCTURE ONLY.

At cfg 3-5 sizes (5.4M-43M dofs) the reference's direct route (PatternAssembler +
SuperLU, fem.py:270-409) is infeasible in 3D.  This module keeps
the reference's element-by-element arithmetic and replaces only the factorisation:

* ``apply_stiffness`` -- reference hdm.py:224-233 verbatim in numpy (gather, one GEMM
  against K_e^T, alpha scaling, bincount scatter, fixed rows zeroed);
* ``helmholtz_apply`` -- the scalar Q1 operator H = sum_e (r^2 S_e + M_e) of
  filtering.py:54-71, applied the same way (no assembly);
* ``pcg`` -- textbook Jacobi-preconditioned CG on those operators (the BASELINE cfg 3-5
  solver), stopping on the recursive residual, with a separate
  true-residual helper;
* ``filter_apply`` / ``filter_adjoint`` -- filtering.py:73-114 with the Helmholtz solve done
  by ``pcg`` instead of SuperLU.

Used by the full-size parity tests (as the checker) and by bench.py's CPU legs (as the
timed CPU path).  Never imported by the product package.
"""

from __future__ import annotations

import numpy as np

from .fem import Grid, helmholtz_element_matrices
from .hdm import LENGTH_SCALE_FACTOR


def alpha(rho, rho_l, p):  # hdm.py:40-55
    return rho_l + (1.0 - rho_l) * rho**p


def apply_stiffness(grid: Grid, k_e, alpha_e, v, free_mask=None):
    """Z K(rho) v by element scatter (reference hdm.py:224-233)."""
    contrib = (v[grid.elem_dofs] @ k_e.T) * alpha_e[:, None]
    out = np.bincount(grid.elem_dofs.ravel(), weights=contrib.ravel(), minlength=grid.n_dofs)
    if free_mask is not None:
        out[~free_mask] = 0.0
    return out


def stiffness_diagonal(grid: Grid, k_e, alpha_e, free_mask):
    """diag K(rho) on the free dofs, 0 on fixed ones (Jacobi preconditioner)."""
    d = np.bincount(grid.elem_dofs.ravel(), weights=(alpha_e[:, None] * np.diag(k_e)[None, :]).ravel(),
                    minlength=grid.n_dofs)
    return np.where(free_mask, d, 0.0)


def element_sensitivity(grid: Grid, k_e, rho, u, lam, rho_l, p):
    """-alpha'(rho_e) u_e^T K_e lam_e (reference hdm.py:211-222, compliance drho = 0)."""
    c = ((u[grid.elem_dofs] @ k_e) * lam[grid.elem_dofs]).sum(axis=1)
    return -(1.0 - rho_l) * p * rho ** (p - 1.0) * c


class Helmholtz:
    """Scalar Helmholtz filter operator of radius R (filtering.py:47-114), matrix-free."""

    def __init__(self, grid: Grid, radius: float):
        self.grid = grid
        self.radius = float(radius)
        self.r = LENGTH_SCALE_FACTOR * self.radius
        self.npe = 2**grid.dim
        self.h_e, self.b_e = helmholtz_element_matrices(self.r, grid.h, grid.dim)
        self.diag = np.bincount(grid.elem_nodes.ravel(),
                                weights=np.tile(np.diag(self.h_e), grid.n_elems), minlength=grid.n_nodes)

    def apply(self, phi):
        c = phi[self.grid.elem_nodes] @ self.h_e.T
        return np.bincount(self.grid.elem_nodes.ravel(), weights=c.ravel(), minlength=self.grid.n_nodes)

    def load_vector(self, psi):  # filtering.py:73-76
        w = np.repeat(np.asarray(psi, float) * (self.grid.elem_volume / self.npe), self.npe)
        return np.bincount(self.grid.elem_nodes.ravel(), weights=w, minlength=self.grid.n_nodes)

    def average(self, phi):  # filtering.py:96
        return phi[self.grid.elem_nodes].sum(axis=1) / self.npe

    def filter_apply(self, psi, rtol=1e-12, maxit=2000):
        """(phi, rho) of filtering.py:78-97, Helmholtz solve by Jacobi-PCG."""
        phi, _ = pcg(self.apply, 1.0 / self.diag, self.load_vector(psi), rtol, maxit)
        return phi, self.average(phi)

    def filter_adjoint(self, v, rtol=1e-12, maxit=2000):  # filtering.py:99-114
        q = np.bincount(self.grid.elem_nodes.ravel(), weights=np.repeat(np.asarray(v, float) / self.npe, self.npe),
                        minlength=self.grid.n_nodes)
        mu, _ = pcg(self.apply, 1.0 / self.diag, q, rtol, maxit)
        return mu[self.grid.elem_nodes].sum(axis=1) * (self.grid.elem_volume / self.npe)


def pcg(apply, dinv, b, rtol, maxit, x0=None, iters_only=None):
    """Jacobi-PCG on an SPD operator (fixed dofs carry dinv = 0 and stay 0).  Stops when the
    recursive residual satisfies ||r|| <= rtol ||b_free||, after ``maxit`` iterations, or --
    ``iters_only`` -- after exactly that many iterations (timing samples).  Returns (x, its)."""
    free = dinv != 0.0
    b = np.where(free, b, 0.0)
    x = np.zeros_like(b) if x0 is None else x0.copy()
    r = b - np.where(free, apply(x), 0.0) if x0 is not None else b.copy()
    z = dinv * r
    p = z.copy()
    rz = r @ z
    tol2 = (rtol**2) * (b @ b)
    n_its = maxit if iters_only is None else iters_only
    for it in range(1, n_its + 1):
        q = np.where(free, apply(p), 0.0)
        a = rz / (p @ q)
        x += a * p
        r -= a * q
        rr = r @ r
        if iters_only is None and rr <= tol2:
            return x, it
        z = dinv * r
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, n_its


def true_relres(apply, free_mask, b, x):
    """||Z(b - A x)|| / ||Z b|| (PCG termination checked on the true residual)."""
    bz = np.where(free_mask, b, 0.0)
    r = np.where(free_mask, b - apply(x), 0.0)
    return float(np.linalg.norm(r) / np.linalg.norm(bz))
