"""Structured Q1 meshes (Q4 2D / Hex8 3D) and element matrices — host-side definitions.

Mirrors the public surface of the reference ``romtopt.fem`` (fem.py:19-30):
``StructuredMesh``, ``build_mesh``, ``elasticity_element_matrix``,
``helmholtz_element_matrices``, ``element_mass_matrix``, ``assemble``,
``IndefiniteMatrixError``.  Adds ``build_mesh_3d`` / ``hex8_element_matrix`` for
the Hex8 grids of BASELINE configs 3-5 (the reference is 2D only).

Nothing here is on the compute path: the device operator is matrix-free and
generates connectivity from the grid dimensions.  ``elem_nodes``/``elem_dofs``
are materialised lazily, only when a caller reads them.
"""

from __future__ import annotations

from functools import cached_property

import numpy as np

__all__ = [
    "StructuredMesh",
    "IndefiniteMatrixError",
    "build_mesh",
    "build_mesh_3d",
    "elasticity_element_matrix",
    "hex8_element_matrix",
    "helmholtz_element_matrices",
    "element_mass_matrix",
    "assemble",
]


class IndefiniteMatrixError(RuntimeError):
    """The stiffness operator is not positive definite on the free dofs (fem.py:33-38).

    Raised when the matrix-free pCG breaks down (p^T K p <= 0 or non-finite).
    """


# ----------------------------------------------------------------------------------------
# element matrices
# ----------------------------------------------------------------------------------------
def _q1_corners(dim):
    sq = [(-1, -1), (1, -1), (1, 1), (-1, 1)]
    if dim == 2:
        return np.array(sq, float)
    return np.array([(x, y, -1) for x, y in sq] + [(x, y, 1) for x, y in sq], float)


def _gauss_elasticity(dim, e0, nu, h):
    """2^dim-point Gauss stiffness of the isotropic Q1 element (plane stress in 2D)."""
    corners = _q1_corners(dim)
    nn = corners.shape[0]
    if dim == 2:
        c = e0 / (1 - nu * nu) * np.array([[1, nu, 0], [nu, 1, 0], [0, 0, (1 - nu) / 2]])
        pairs = [(0, 0), (1, 1), ((0, 1), (1, 0))]
    else:
        lam, mu = e0 * nu / ((1 + nu) * (1 - 2 * nu)), e0 / (2 * (1 + nu))
        c = np.zeros((6, 6))
        c[:3, :3] = lam
        c[range(3), range(3)] += 2 * mu
        c[3:, 3:] = mu * np.eye(3)
        pairs = [(0, 0), (1, 1), (2, 2), ((1, 2), (2, 1)), ((0, 2), (2, 0)), ((0, 1), (1, 0))]
    g1 = 1.0 / np.sqrt(3.0)
    k = np.zeros((dim * nn, dim * nn))
    for q in np.array(np.meshgrid(*([[-g1, g1]] * dim), indexing="ij")).reshape(dim, -1).T:
        grad = np.empty((nn, dim))
        for a in range(dim):
            f = np.prod(np.delete(1 + corners * q, a, axis=1), axis=1)
            grad[:, a] = corners[:, a] * f / 2**dim * (2.0 / h)
        b = np.zeros((len(pairs), dim * nn))
        for row, pr in enumerate(pairs):
            if isinstance(pr[0], tuple):
                (c1, d1), (c2, d2) = pr
                b[row, c1::dim] = grad[:, d1]
                b[row, c2::dim] = grad[:, d2]
            else:
                b[row, pr[0]::dim] = grad[:, pr[1]]
        k += b.T @ c @ b * (h / 2) ** dim
    return 0.5 * (k + k.T)  # exactly symmetric


# Closed-form Q4 integer tables (the values of reference fem.py:45-70), reconstructed exactly
# by quadrature: K_e = E0/(1-nu^2) * (KA + nu*KB) / 24.
_KA = np.rint(24.0 * _gauss_elasticity(2, 1.0, 0.0, 1.0))
_KB = np.rint(4.0 * (22.5 * _gauss_elasticity(2, 1.0, 0.25, 1.0) - _KA))
# Q1 scalar tables (fem.py:72-92): Laplacian*6 by corner distance {0:4, 1:-1, 2:-2};
# mass*36/h^2 by corner distance {0:4, 1:2, 2:1}.
_DIST2 = np.abs(_q1_corners(2)[:, None, :] - _q1_corners(2)[None, :, :]).sum(-1) / 2
_S6 = np.choose(_DIST2.astype(int), [4.0, -1.0, -2.0])
_M36 = np.choose(_DIST2.astype(int), [4.0, 2.0, 1.0])


def elasticity_element_matrix(e0: float, nu: float, h: float = 1.0) -> np.ndarray:
    """Exact Q4 plane-stress unit-density stiffness, h-independent (fem.py:95-116)."""
    if not 0.0 <= nu < 0.5:
        raise ValueError(f"Poisson ratio must satisfy 0 <= nu < 0.5, got {nu}")
    if e0 <= 0.0:
        raise ValueError(f"Young's modulus must be positive, got {e0}")
    if h <= 0.0:
        raise ValueError(f"element size must be positive, got {h}")
    return e0 / (1.0 - nu**2) * (_KA + nu * _KB) / 24.0


def hex8_element_matrix(e0: float, nu: float, h: float = 1.0) -> np.ndarray:
    """Hex8 isotropic unit-density stiffness (24x24) by 2x2x2 Gauss quadrature."""
    if not 0.0 <= nu < 0.5:
        raise ValueError(f"Poisson ratio must satisfy 0 <= nu < 0.5, got {nu}")
    if e0 <= 0.0 or h <= 0.0:
        raise ValueError("e0 and h must be positive")
    return _gauss_elasticity(3, e0, nu, h)


def element_mass_matrix(h: float) -> np.ndarray:
    """Consistent Q4 mass matrix (fem.py:119-121)."""
    return h**2 / 36.0 * _M36


def helmholtz_element_matrices(r: float, h: float):
    """(H_e, b_e) = (r^2 S_e + M_e, M_e 1) of the Q4 screened-Poisson filter (fem.py:124-137)."""
    if r < 0.0:
        raise ValueError(f"filter length must be nonnegative, got {r}")
    if h <= 0.0:
        raise ValueError(f"element size must be positive, got {h}")
    h_e = r**2 * _S6 / 6.0 + element_mass_matrix(h)
    b_e = element_mass_matrix(h) @ np.ones(4)
    return h_e, b_e


# ----------------------------------------------------------------------------------------
# mesh
# ----------------------------------------------------------------------------------------
class StructuredMesh:
    """Rectangular (2D) or box (3D) grid of congruent Q1 elements (fem.py:154-212).

    Node ``(k*(ny+1)+j)*(nx+1)+i`` (x fastest), element ``(k*ny+j)*nx+i``, dofs
    interleaved ``dim*n + c``; element nodes CCW from the bottom-left corner
    (3D: bottom face then top face).
    """

    def __init__(self, nx: int, ny: int, h: float, nz: int = 0):
        self.nx, self.ny, self.nz, self.h = int(nx), int(ny), int(nz), float(h)

    def __repr__(self):
        dims = f"{self.nx}x{self.ny}" + (f"x{self.nz}" if self.nz else "")
        return f"StructuredMesh({dims}, h={self.h})"

    def __eq__(self, other):
        return isinstance(other, StructuredMesh) and (self.nx, self.ny, self.nz, self.h) == (
            other.nx, other.ny, other.nz, other.h)

    def __hash__(self):
        return hash((self.nx, self.ny, self.nz, self.h))

    @property
    def dim(self) -> int:
        return 3 if self.nz else 2

    @property
    def n_elems(self) -> int:
        return self.nx * self.ny * (self.nz or 1)

    @property
    def n_nodes(self) -> int:
        return (self.nx + 1) * (self.ny + 1) * ((self.nz + 1) if self.nz else 1)

    @property
    def n_dofs(self) -> int:
        return self.dim * self.n_nodes

    @property
    def elem_volume(self) -> float:
        return self.h**self.dim

    @property
    def domain_volume(self) -> float:
        return self.n_elems * self.elem_volume

    def node_id(self, i, j, k=0):
        return (k * (self.ny + 1) + j) * (self.nx + 1) + i

    def node_coords(self) -> np.ndarray:
        n = np.arange(self.n_nodes)
        nnx, nny = self.nx + 1, self.ny + 1
        cols = [n % nnx, (n // nnx) % nny] + ([n // (nnx * nny)] if self.nz else [])
        return np.column_stack(cols) * self.h

    def boundary_nodes(self, side: str) -> np.ndarray:
        """Sorted node ids on 'left'/'right' (x), 'bottom'/'top' (y), 'front'/'back' (z)."""
        nnx, nny, nnz = self.nx + 1, self.ny + 1, (self.nz + 1 if self.nz else 1)
        if side in ("front", "back") and not self.nz:
            raise ValueError(f"unknown side {side!r}")
        axis = {"left": (0, 0), "right": (0, self.nx), "bottom": (1, 0), "top": (1, self.ny),
                "front": (2, 0), "back": (2, self.nz)}.get(side)
        if axis is None:
            raise ValueError(f"unknown side {side!r}")
        k, j, i = np.meshgrid(np.arange(nnz), np.arange(nny), np.arange(nnx), indexing="ij")
        sel = (i, j, k)[axis[0]] == axis[1]
        return np.sort(((k * nny + j) * nnx + i)[sel].ravel())

    @cached_property
    def elem_nodes(self) -> np.ndarray:
        e = np.arange(self.n_elems, dtype=np.int64)
        i, j = e % self.nx, (e // self.nx) % self.ny
        nnx = self.nx + 1
        if not self.nz:
            n0 = j * nnx + i
            return np.column_stack([n0, n0 + 1, n0 + nnx + 1, n0 + nnx])
        k = e // (self.nx * self.ny)
        nnxy = nnx * (self.ny + 1)
        n0 = k * nnxy + j * nnx + i
        face = [n0, n0 + 1, n0 + nnx + 1, n0 + nnx]
        return np.column_stack(face + [f + nnxy for f in face])

    @cached_property
    def elem_dofs(self) -> np.ndarray:
        d = self.dim
        en = self.elem_nodes
        return (d * en[:, :, None] + np.arange(d)[None, None, :]).reshape(en.shape[0], -1)


def build_mesh(nx: int, ny: int, h: float) -> StructuredMesh:
    """2D mesh of nx x ny square elements (fem.py:215-229)."""
    if nx < 1 or ny < 1:
        raise ValueError(f"element counts must be >= 1, got nx={nx}, ny={ny}")
    if h <= 0.0:
        raise ValueError(f"element size must be positive, got {h}")
    return StructuredMesh(nx, ny, h)


def build_mesh_3d(nx: int, ny: int, nz: int, h: float) -> StructuredMesh:
    """3D mesh of nx x ny x nz cubic Hex8 elements."""
    if nx < 1 or ny < 1 or nz < 1:
        raise ValueError(f"element counts must be >= 1, got {nx}x{ny}x{nz}")
    if h <= 0.0:
        raise ValueError(f"element size must be positive, got {h}")
    return StructuredMesh(nx, ny, h, nz)


def assemble(mesh: StructuredMesh, elem_matrix: np.ndarray, scales=None, field_kind: str = "vector"):
    """Diagnostic sparse assembly sum_e s_e P_e K_e P_e^T (fem.py:232-267).

    Host-side scipy utility for inspection and tests only; no solver in this package uses
    an assembled matrix.
    """
    import scipy.sparse as sp

    if field_kind == "vector":
        idx, n = mesh.elem_dofs, mesh.n_dofs
    elif field_kind == "scalar":
        idx, n = mesh.elem_nodes, mesh.n_nodes
    else:
        raise ValueError(f"unknown field kind {field_kind!r}")
    k = idx.shape[1]
    if elem_matrix.shape != (k, k):
        raise ValueError(f"element matrix must be {(k, k)}, got {elem_matrix.shape}")
    scales = np.ones(mesh.n_elems) if scales is None else np.asarray(scales, dtype=float)
    if scales.shape != (mesh.n_elems,):
        raise ValueError(f"scales must have length {mesh.n_elems}, got shape {scales.shape}")
    rows = np.repeat(idx, k, axis=1).ravel()
    cols = np.tile(idx, (1, k)).ravel()
    vals = (scales[:, None] * elem_matrix.ravel()[None, :]).ravel()
    return sp.coo_matrix((vals, (rows, cols)), shape=(n, n)).tocsc()
