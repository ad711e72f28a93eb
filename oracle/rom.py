"""Oracle ROM: POD, Gram-Schmidt, basis build, reduced operators, residuals, error bounds.

Restates reference rom.py:53-407 (numpy/scipy).  Element caches
(``elem_phi``/``elem_k_phi``, rom.py:242-243) are built only for the
element-form reduced stiffness on small meshes; ``reduced_stiffness_nodeform``
evaluates the same quantity as Phi^T (K(rho) Phi) through the sparse operator
for larger meshes (mathematically identical, reference PAPER.md:444).
"""

from __future__ import annotations

import numpy as np
import scipy.linalg

from .hdm import Hdm

GS_DROP_TOL = 1e-10  # rom.py:42


def pod(snapshots, n):  # rom.py:53-73
    s = np.atleast_2d(np.asarray(snapshots, float))
    if n > s.shape[1]:
        raise ValueError("too many modes")
    if n == 0:
        return np.zeros((s.shape[0], 0))
    u = np.linalg.svd(s, full_matrices=False)[0][:, :n].copy()
    for c in range(n):
        if u[np.argmax(np.abs(u[:, c])), c] < 0.0:
            u[:, c] = -u[:, c]
    return u


def gram_schmidt(vectors, drop_tol=GS_DROP_TOL):  # rom.py:76-97
    out = []
    for v in vectors:
        v = np.asarray(v, float).copy()
        n0 = np.linalg.norm(v)
        if n0 == 0.0:
            continue
        for _ in range(2):
            for b in out:
                v -= (b @ v) * b
        n1 = np.linalg.norm(v)
        if n1 >= drop_tol * n0:
            out.append(v / n1)
    if not out:
        raise ValueError("no independent vectors")
    return np.column_stack(out)


class Rom:
    """RomModel restated (rom.py:182-390)."""

    def __init__(self, hdm: Hdm):
        self.hdm = hdm

    def build_basis(self, primal_window, center_u, center_lambda, is_compliance, n_k, center_rho=None,
                    adjoint_window=None):  # rom.py:199-252
        if center_u is None or np.linalg.norm(center_u) == 0.0:
            raise ValueError("zero center")
        n_win = 0 if primal_window is None else primal_window.shape[1]
        n_k = min(n_k, n_win)
        blocks = [center_u]
        if not is_compliance:
            blocks.append(center_lambda)
        if n_k > 0:
            blocks.extend(pod(primal_window, n_k).T)
            if not is_compliance:
                blocks.extend(pod(adjoint_window, n_k).T)
        blocks = [np.where(self.hdm.free_mask, v, 0.0) for v in blocks]
        phi = gram_schmidt(blocks)
        f_eff = self.hdm.f if center_rho is None else self.hdm.apply_stiffness(center_rho, center_u)
        return phi, phi.T @ f_eff

    def reduced_stiffness_elemform(self, phi, rho):  # rom.py:254-262
        ed = self.hdm.grid.elem_dofs
        ep = phi[ed]
        ekp = np.matmul(self.hdm.k_e, ep)
        a = self.hdm.material.alpha(rho)
        j = phi.shape[1]
        return (ep * a[:, None, None]).reshape(-1, j).T @ ekp.reshape(-1, j)

    def reduced_stiffness_nodeform(self, phi, rho):
        k = self.hdm.stiffness(rho)
        return phi.T @ (k @ phi)

    def solve(self, phi, f_hat, rho, du=None):  # rom.py:264-307 (without gradient)
        k_hat = self.reduced_stiffness_nodeform(phi, rho)
        cho = scipy.linalg.cho_factor(k_hat)
        uhat = scipy.linalg.cho_solve(cho, f_hat)
        u = phi @ uhat
        if du is None:
            lamhat, lam = uhat, u
        else:
            lamhat = scipy.linalg.cho_solve(cho, phi.T @ du(u, rho))
            lam = phi @ lamhat
        res = self.residual_vector(phi, rho, uhat)
        return dict(k_hat=k_hat, uhat=uhat, u=u, lamhat=lamhat, lam=lam, j=float(self.hdm.f @ u),
                    residual_norm=float(np.linalg.norm(res)))

    def residual_vector(self, phi, rho, uhat):  # rom.py:309-325
        k = self.hdm.stiffness(rho)
        r = k @ (phi @ uhat) - self.hdm.f
        r[~self.hdm.free_mask] = 0.0
        return r

    def smallest_eigenvalue(self, rho, max_iter=200, rtol=1e-10):  # rom.py:393-407
        from .fem import DirectSolver
        fact = DirectSolver(self.hdm.stiffness(rho), self.hdm.fixed)
        n = fact.a.shape[0]
        x = np.ones(n) + 1e-3 * np.sin(np.arange(n))
        x /= np.linalg.norm(x)
        prev = np.inf
        for _ in range(max_iter):
            y = fact.lu.solve(x)
            x = y / np.linalg.norm(y)
            ev = float(x @ (fact.a @ x))
            if abs(ev - prev) <= rtol * abs(ev):
                return ev, True
            prev = ev
        return prev, False
