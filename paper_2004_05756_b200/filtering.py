"""Helmholtz PDE density filter on the GPU (drop-in for reference filtering.py:47-114).

``H phi = b(psi)`` (pure Neumann, H = sum_e r^2 S_e + M_e) is solved matrix-free by a
Jacobi-preconditioned CG inside one CUDA graph; the element density is the nodal
average.  ``apply_adjoint`` applies the exact transpose (one more solve).  Inputs may
be numpy arrays (results come back as numpy, like the reference) or CUDA tensors
(results stay on the device).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .fem import StructuredMesh

__all__ = ["HelmholtzFilter", "ConeFilter", "FilterResult", "LENGTH_SCALE_FACTOR"]

# R = 2 sqrt(3) r  (filtering.py:29-32)
LENGTH_SCALE_FACTOR = 1.0 / (2.0 * np.sqrt(3.0))


class FilterResult:
    """Nodal solution and element-averaged density (filtering.py:37-44)."""

    __slots__ = ("phi", "rho")

    def __init__(self, phi, rho):
        self.phi = phi
        self.rho = rho


class HelmholtzFilter:
    """Design-density filter of radius ``R`` on a structured mesh (2D Q4 or 3D Hex8).

    ``rtol`` is the relative residual at which the inner pCG stops.  The reference factorises H
    once and solves directly, so the default (None) solves to round-off: target 1e-15, a true
    residual stagnating at its floor accepted (tb_filter_apply round-off mode).  Filtered
    densities then agree with the direct solve to ~1e-16, which finite differences of J need.
    """

    def __init__(self, mesh: StructuredMesh, radius: float, rtol: float | None = None, device=None):
        if radius < 0.0:
            raise ValueError(f"filter radius must be nonnegative, got {radius}")
        self.mesh = mesh
        self.radius = float(radius)
        self.r = LENGTH_SCALE_FACTOR * self.radius
        self.rtol = -1e-15 if rtol is None else float(rtol)  # negative: round-off mode (C ABI)
        dim, nz = _lib.mesh_dims(mesh)
        self.nodes_per_elem = 2**dim
        # b_e = M_e 1 = (h^d / 2^d) per node (filtering.py:60-61, 75-76)
        self.b_e = np.full(self.nodes_per_elem, mesh.elem_volume / self.nodes_per_elem)
        self.device = _lib.require_cuda(device)
        self.last_iters = 0
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().tb_filter_create(dim, mesh.nx, mesh.ny, nz, mesh.h, self.radius,
                                               self.device.index, ctypes.byref(h)), "HelmholtzFilter")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib._lib is not None:
            _lib._lib.tb_filter_destroy(h)
            self._h = None

    def _check(self, x, name):
        n = self.mesh.n_elems
        if tuple(x.shape) != (n,):
            raise ValueError(f"{name} must have length {n}, got shape {tuple(x.shape)}")

    def load_vector(self, psi):
        """b(psi) = (h^d/2^d) sum_{e∋n} psi_e (filtering.py:73-76)."""
        t = _lib.torch()
        native = _lib.is_torch(psi)
        psi_d = _lib.to_dev(psi, self.device)
        self._check(psi_d, "psi")
        b = t.empty(self.mesh.n_nodes, dtype=t.float64, device=self.device)
        _lib.check(_lib.lib().tb_filter_load_vector(self._h, _lib.ptr(psi_d), _lib.ptr(b),
                                                    _lib.stream_ptr(self.device)), "load_vector")
        return _lib.to_user(b, native)

    def apply_device(self, psi_d, want_phi=True):
        """Device-tensor path: returns (phi or None, rho) as CUDA tensors."""
        t = _lib.torch()
        self._check(psi_d, "psi")
        rho = t.empty(self.mesh.n_elems, dtype=t.float64, device=self.device)
        phi = t.empty(self.mesh.n_nodes, dtype=t.float64, device=self.device) if want_phi else None
        it = ctypes.c_int(0)
        _lib.check(_lib.lib().tb_filter_apply(self._h, _lib.ptr(psi_d), _lib.ptr(phi), _lib.ptr(rho), self.rtol,
                                              ctypes.byref(it), _lib.stream_ptr(self.device)), "filter apply")
        self.last_iters = it.value
        return phi, rho

    def apply(self, psi) -> FilterResult:
        """Filter a raw density field (filtering.py:78-97)."""
        native = _lib.is_torch(psi)
        psi_d = _lib.to_dev(psi, self.device)
        phi, rho = self.apply_device(psi_d)
        return FilterResult(phi=_lib.to_user(phi, native), rho=_lib.to_user(rho, native))

    def apply_adjoint_device(self, v_d):
        t = _lib.torch()
        self._check(v_d, "v")
        w = t.empty(self.mesh.n_elems, dtype=t.float64, device=self.device)
        it = ctypes.c_int(0)
        _lib.check(_lib.lib().tb_filter_adjoint(self._h, _lib.ptr(v_d), _lib.ptr(w), self.rtol, ctypes.byref(it),
                                                _lib.stream_ptr(self.device)), "filter adjoint")
        self.last_iters = it.value
        return w

    def apply_adjoint(self, v):
        """Exact transpose of the psi -> rho map (filtering.py:99-114)."""
        native = _lib.is_torch(v)
        return _lib.to_user(self.apply_adjoint_device(_lib.to_dev(v, self.device)), native)


class ConeFilter:
    """Classical cone ("linear hat") density filter of radius ``R``.

    rho_e = sum_j w(e, j) psi_j / sum_j w(e, j),  w(e, j) = max(0, R - |c_e - c_j|), over the
    elements of the grid (normalised at the boundary).  An alternative to HelmholtzFilter for
    BASELINE's "linear density filter" wording; the reference has no such filter, so its
    parity is against oracle/filters.py.  Drop-in for HdmSolver: same ``apply`` /
    ``apply_adjoint`` (and device variants); ``phi`` is None (no nodal field).
    """

    def __init__(self, mesh: StructuredMesh, radius: float, device=None):
        if radius < 0.0:
            raise ValueError(f"filter radius must be nonnegative, got {radius}")
        self.mesh = mesh
        self.radius = float(radius)
        self.device = _lib.require_cuda(device)
        self.last_iters = 0
        h = ctypes.c_void_p()
        dim, nz = _lib.mesh_dims(mesh)
        _lib.check(_lib.lib().tb_cone_create(dim, mesh.nx, mesh.ny, nz, mesh.h, self.radius,
                                             self.device.index, ctypes.byref(h)), "ConeFilter")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib._lib is not None:
            _lib._lib.tb_cone_destroy(h)
            self._h = None

    def _check(self, x, name):
        n = self.mesh.n_elems
        if tuple(x.shape) != (n,):
            raise ValueError(f"{name} must have length {n}, got shape {tuple(x.shape)}")

    def apply_device(self, psi_d, want_phi=True):
        """Device-tensor path: returns (None, rho)."""
        del want_phi
        t = _lib.torch()
        self._check(psi_d, "psi")
        rho = t.empty(self.mesh.n_elems, dtype=t.float64, device=self.device)
        _lib.check(_lib.lib().tb_cone_apply(self._h, _lib.ptr(psi_d), _lib.ptr(rho), _lib.stream_ptr(self.device)),
                   "cone filter apply")
        return None, rho

    def apply(self, psi) -> FilterResult:
        native = _lib.is_torch(psi)
        _, rho = self.apply_device(_lib.to_dev(psi, self.device).contiguous())
        return FilterResult(phi=None, rho=_lib.to_user(rho, native))

    def apply_adjoint_device(self, v_d):
        t = _lib.torch()
        self._check(v_d, "v")
        w = t.empty(self.mesh.n_elems, dtype=t.float64, device=self.device)
        _lib.check(_lib.lib().tb_cone_adjoint(self._h, _lib.ptr(v_d), _lib.ptr(w), _lib.stream_ptr(self.device)),
                   "cone filter adjoint")
        return w

    def apply_adjoint(self, v):
        """Exact transpose of the psi -> rho map."""
        native = _lib.is_torch(v)
        return _lib.to_user(self.apply_adjoint_device(_lib.to_dev(v, self.device).contiguous()), native)
