"""Oracle FE core: structured grids, element matrices, sparse assembly, direct solve.

Restates /root/reference/pkg/src/romtopt/fem.py for 2D and extends the same
conventions to 3D (Hex8) where the reference has no code.

Conventions (reference fem.py:1-9, 154-229):
* node id ``j*(nx+1) + i`` (x fastest); 3D: ``(k*(ny+1) + j)*(nx+1) + i``;
* element id ``j*nx + i``; 3D: ``(k*ny + j)*nx + i``;
* element nodes counter-clockwise from the bottom-left corner
  (fem.py:225); 3D: bottom face (z=k) CCW then top face (z=k+1) CCW;
* dofs interleaved per node: ``d*n + c`` (fem.py:226-228).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


class OracleIndefinite(RuntimeError):
    """Non-positive pivot (reference fem.py:33-38, 305-311)."""


# ----------------------------------------------------------------------------------------
# Gauss quadrature element matrices (pattern: reference tests/oracles.py:44-89)
# ----------------------------------------------------------------------------------------
_GP = np.array([-1.0, 1.0]) / np.sqrt(3.0)


def _corner_signs(dim: int) -> np.ndarray:
    """(2^dim, dim) reference-cube corner signs in the element node order."""
    if dim == 2:
        return np.array([[-1, -1], [1, -1], [1, 1], [-1, 1]], dtype=float)
    sq = np.array([[-1, -1], [1, -1], [1, 1], [-1, 1]], dtype=float)
    bot = np.column_stack([sq, -np.ones(4)])
    top = np.column_stack([sq, np.ones(4)])
    return np.vstack([bot, top])


def _shape(dim, xi):
    s = _corner_signs(dim)
    n = np.prod(1.0 + s * xi[None, :], axis=1) / 2**dim
    dn = np.zeros((2**dim, dim))
    for a in range(dim):
        other = np.prod(np.delete(1.0 + s * xi[None, :], a, axis=1), axis=1)
        dn[:, a] = s[:, a] * other / 2**dim
    return n, dn


def _gauss_points(dim):
    if dim == 2:
        return [np.array([x, y]) for x in _GP for y in _GP]
    return [np.array([x, y, z]) for x in _GP for y in _GP for z in _GP]


def quad_elasticity(dim: int, e0: float, nu: float, h: float) -> np.ndarray:
    """Unit-density element stiffness by 2^dim-point Gauss quadrature.

    2D: plane stress (reference oracles.py:44-67).  3D: isotropic linear
    elasticity, Voigt order (xx, yy, zz, yz, xz, xy).
    """
    nn = 2**dim
    if dim == 2:
        d = e0 / (1.0 - nu**2) * np.array([[1.0, nu, 0.0], [nu, 1.0, 0.0], [0.0, 0.0, (1.0 - nu) / 2.0]])
    else:
        lam = e0 * nu / ((1 + nu) * (1 - 2 * nu))
        mu = e0 / (2 * (1 + nu))
        d = np.zeros((6, 6))
        d[:3, :3] = lam
        d[np.arange(3), np.arange(3)] += 2 * mu
        d[3:, 3:] = mu * np.eye(3)
    k = np.zeros((dim * nn, dim * nn))
    jac = (h / 2.0) ** dim
    for xi in _gauss_points(dim):
        _, dn = _shape(dim, xi)
        g = dn * 2.0 / h  # physical gradients (nn, dim)
        if dim == 2:
            b = np.zeros((3, 8))
            b[0, 0::2] = g[:, 0]
            b[1, 1::2] = g[:, 1]
            b[2, 0::2] = g[:, 1]
            b[2, 1::2] = g[:, 0]
        else:
            b = np.zeros((6, 24))
            b[0, 0::3] = g[:, 0]
            b[1, 1::3] = g[:, 1]
            b[2, 2::3] = g[:, 2]
            b[3, 1::3] = g[:, 2]
            b[3, 2::3] = g[:, 1]
            b[4, 0::3] = g[:, 2]
            b[4, 2::3] = g[:, 0]
            b[5, 0::3] = g[:, 1]
            b[5, 1::3] = g[:, 0]
        k += b.T @ d @ b * jac
    return 0.5 * (k + k.T)  # exactly symmetric


def quad_scalar(dim: int, h: float):
    """(Laplacian S_e, consistent mass M_e) for the scalar Q1 element."""
    nn = 2**dim
    s = np.zeros((nn, nn))
    m = np.zeros((nn, nn))
    jac = (h / 2.0) ** dim
    for xi in _gauss_points(dim):
        n, dn = _shape(dim, xi)
        g = dn * 2.0 / h
        s += g @ g.T * jac
        m += np.outer(n, n) * jac
    return s, m


# 2D closed-form integer tables, recovered exactly from quadrature
# (reference fem.py:41-92 states them as literals): K_e = E0/(1-nu^2)(A + nu B)/24,
# S_e = S6/6, M_e = h^2 M36/36.
_A2 = np.rint(24.0 * quad_elasticity(2, 1.0, 0.0, 1.0))
_B2 = np.rint((24.0 * (1.0 - 0.25**2) * quad_elasticity(2, 1.0, 0.25, 1.0) - _A2) / 0.25)
_S6 = np.rint(6.0 * quad_scalar(2, 1.0)[0])
_M36 = np.rint(36.0 * quad_scalar(2, 1.0)[1])


def elasticity_element_matrix(e0: float, nu: float, h: float = 1.0, dim: int = 2) -> np.ndarray:
    """Reference fem.py:95-116 (2D closed form, same operation order); 3D by quadrature."""
    if not 0.0 <= nu < 0.5:
        raise ValueError("nu")
    if e0 <= 0.0 or h <= 0.0:
        raise ValueError("e0/h")
    if dim == 2:
        return e0 / (1.0 - nu**2) * (_A2 + nu * _B2) / 24.0
    return quad_elasticity(3, e0, nu, h)


def helmholtz_element_matrices(r: float, h: float, dim: int = 2):
    """Reference fem.py:119-137: H_e = r^2 S_e + M_e, b_e = M_e @ 1."""
    if r < 0.0 or h <= 0.0:
        raise ValueError("r/h")
    if dim == 2:
        m_e = h**2 / 36.0 * _M36
        h_e = r**2 * _S6 / 6.0 + m_e
        return h_e, m_e @ np.ones(4)
    s_e, m_e = quad_scalar(3, h)
    return r**2 * s_e + m_e, m_e @ np.ones(8)


# ----------------------------------------------------------------------------------------
# Structured grid (reference fem.py:154-229)
# ----------------------------------------------------------------------------------------
@dataclass(frozen=True)
class Grid:
    dim: int
    nx: int
    ny: int
    nz: int
    h: float
    elem_nodes: np.ndarray = field(repr=False)
    elem_dofs: np.ndarray = field(repr=False)

    @property
    def n_elems(self):
        return self.nx * self.ny * (self.nz if self.dim == 3 else 1)

    @property
    def n_nodes(self):
        return (self.nx + 1) * (self.ny + 1) * ((self.nz + 1) if self.dim == 3 else 1)

    @property
    def n_dofs(self):
        return self.dim * self.n_nodes

    @property
    def elem_volume(self):
        return self.h**self.dim

    def node_id(self, i, j, k=0):
        return (k * (self.ny + 1) + j) * (self.nx + 1) + i

    def boundary_nodes(self, side):
        """Reference fem.py:201-212 (2D); 3D adds 'front'/'back' (z=0 / z=nz)."""
        nnx, nny = self.nx + 1, self.ny + 1
        nnz = self.nz + 1 if self.dim == 3 else 1
        k, j, i = np.meshgrid(np.arange(nnz), np.arange(nny), np.arange(nnx), indexing="ij")
        ids = (k * nny + j) * nnx + i
        sel = {
            "left": i == 0, "right": i == self.nx, "bottom": j == 0, "top": j == self.ny,
            "front": k == 0, "back": k == (self.nz if self.dim == 3 else 0),
        }[side]
        return np.sort(ids[sel].ravel())


def build_grid(nx, ny, h, nz=None) -> Grid:
    """Reference fem.py:215-229 for 2D; the same numbering extended to Hex8."""
    if nz is None:
        e = np.arange(nx * ny)
        i, j = e % nx, e // nx
        n0 = j * (nx + 1) + i
        en = np.column_stack([n0, n0 + 1, n0 + nx + 2, n0 + nx + 1]).astype(np.int64)
        dim = 2
    else:
        e = np.arange(nx * ny * nz)
        i = e % nx
        j = (e // nx) % ny
        k = e // (nx * ny)
        nnx, nnxy = nx + 1, (nx + 1) * (ny + 1)
        n0 = k * nnxy + j * nnx + i
        face = np.column_stack([n0, n0 + 1, n0 + nnx + 1, n0 + nnx])
        en = np.column_stack([face, face + nnxy]).astype(np.int64)
        dim = 3
    dofs = (dim * en[:, :, None] + np.arange(dim)[None, None, :]).reshape(en.shape[0], -1)
    return Grid(dim=dim, nx=nx, ny=ny, nz=(nz or 0), h=float(h), elem_nodes=en, elem_dofs=dofs)


# ----------------------------------------------------------------------------------------
# Assembly / direct solve (reference fem.py:232-349)
# ----------------------------------------------------------------------------------------
def assemble(grid: Grid, elem_matrix, scales=None, scalar=False) -> sp.csc_matrix:
    """sum_e scales[e] P_e K_e P_e^T as CSC (reference fem.py:232-267)."""
    idx = grid.elem_nodes if scalar else grid.elem_dofs
    n = grid.n_nodes if scalar else grid.n_dofs
    k = idx.shape[1]
    if scales is None:
        scales = np.ones(grid.n_elems)
    rows = np.repeat(idx, k, axis=1).ravel()
    cols = np.tile(idx, (1, k)).ravel()
    vals = (np.asarray(scales, float)[:, None] * elem_matrix.ravel()[None, :]).ravel()
    return sp.coo_matrix((vals, (rows, cols)), shape=(n, n)).tocsc()


class DirectSolver:
    """SuperLU symmetric-mode factorization with pivot check (reference fem.py:270-333)."""

    def __init__(self, a, fixed=None):
        a = a.tocsc()
        self.n_full = a.shape[0]
        if fixed is not None and len(fixed):
            self.free = np.setdiff1d(np.arange(self.n_full), fixed)
            a = a[self.free][:, self.free].tocsc()
        else:
            self.free = None
        self.a = a
        try:
            self.lu = spla.splu(a, permc_spec="MMD_AT_PLUS_A", diag_pivot_thresh=0.0,
                                options=dict(SymmetricMode=True))
        except RuntimeError as err:
            raise OracleIndefinite(str(err)) from err
        d = self.lu.U.diagonal()
        if not np.all(np.isfinite(d)) or np.any(d <= 0.0):
            raise OracleIndefinite("non-positive pivot")

    def solve(self, rhs):
        rhs = np.asarray(rhs, float)
        if self.free is None:
            return self.lu.solve(rhs)
        x = np.zeros(self.n_full)
        x[self.free] = self.lu.solve(rhs[self.free])
        return x
