"""Full-order SIMP evaluation on the GPU (drop-in for reference hdm.py).

Chain (hdm.py:1-8): psi -> rho (Helmholtz filter, clamp) -> K(rho) u = f (matrix-free
Jacobi-pCG on sm_100a instead of SuperLU) -> J = f^T u -> per-element sensitivity ->
filter adjoint.  Public names, signatures, counters and exceptions follow the reference:
``MaterialModel``, ``Objective``, ``ComplianceObjective``, ``HdmSolution``, ``HdmSolver``,
``StaleSolutionError``, ``psi_digest``.

Two calling modes share one device path:
* compat  — numpy inputs, numpy outputs (one D2H copy per returned array), like the reference;
* native  — CUDA tensors in, CUDA tensors out, no host copies on the hot path.
"""

from __future__ import annotations

import ctypes
import hashlib
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import _lib
from .fem import StructuredMesh, assemble
from .filtering import HelmholtzFilter
from .stats import RunStats

__all__ = [
    "MaterialModel",
    "Objective",
    "ComplianceObjective",
    "HdmSolution",
    "HdmSolver",
    "StaleSolutionError",
    "psi_digest",
]


_HOST_POOL = None


def _host_pool():
    """Worker threads for the host-side byte work of the numpy API (design snapshot, staleness
    comparison): numpy releases the GIL for the copies and the solver's ctypes calls release it
    while the device works, so the bytes are handled during the solve instead of after it."""
    global _HOST_POOL
    if _HOST_POOL is None:
        _HOST_POOL = ThreadPoolExecutor(max_workers=2, thread_name_prefix="tb-host")
    return _HOST_POOL


def _same_bytes(psi, snap):
    arr = np.ascontiguousarray(psi, dtype=float)
    return arr.shape == snap.shape and np.array_equal(arr.view(np.uint64), snap.view(np.uint64))


ROUNDOFF_RTOL = -1e-12  # tb_pcg_solve round-off mode: target 1e-12, stagnation <= 1e-7 accepted


class StaleSolutionError(RuntimeError):
    """A solution object was paired with a design it was not computed from (hdm.py:32-33)."""


def psi_digest(psi) -> str:
    """SHA-256 of the fp64 bytes of psi (hdm.py:36-37)."""
    if _lib.is_torch(psi):
        psi = psi.detach().to("cpu", dtype=_lib.torch().float64).numpy()
    return hashlib.sha256(np.ascontiguousarray(psi, dtype=float).tobytes()).hexdigest()


@dataclass(frozen=True)
class MaterialModel:
    """alpha(rho) = rho_l + (1-rho_l) rho^p (hdm.py:40-55).  The device kernels evaluate the
    same law; these host methods serve callers that inspect it."""

    rho_l: float = 1e-3
    p: float = 3.0

    def alpha(self, rho):
        return self.rho_l + (1.0 - self.rho_l) * rho**self.p

    def dalpha(self, rho):
        return (1.0 - self.rho_l) * self.p * rho ** (self.p - 1.0)


class Objective:
    """Objective interface j(u, rho) with analytic partials (hdm.py:58-77)."""

    is_compliance = False
    is_linear_in_u = False

    def value(self, u, rho) -> float:
        raise NotImplementedError

    def du(self, u, rho):
        raise NotImplementedError

    def drho(self, u, rho):
        raise NotImplementedError


class ComplianceObjective(Objective):
    """j = f^T u (hdm.py:80-96); evaluated on the device by the solvers."""

    is_compliance = True
    is_linear_in_u = True

    def __init__(self, f):
        self.f = f if _lib.is_torch(f) else np.asarray(f, dtype=float)
        self._f_dev = None

    def device_f(self, device):
        if self._f_dev is None or self._f_dev.device != device:
            self._f_dev = _lib.to_dev(self.f, device)
        return self._f_dev

    def value(self, u, rho):
        if _lib.is_torch(u):
            return float((self.device_f(u.device) * u).sum())
        return float(np.asarray(self.f) @ u)

    def du(self, u, rho):
        return self.f

    def drho(self, u, rho):
        if _lib.is_torch(rho):
            return _lib.torch().zeros_like(rho)
        return np.zeros(rho.shape[0])


class HdmSolution:
    """One converged full-order evaluation (hdm.py:99-109).

    ``factorization`` is kept for signature compatibility and holds None: the matrix-free
    solver has no factor (the reference stores but never reads it, hdm.py:109,196).
    ``iterations`` / ``relres`` report the pCG run.
    """

    def __init__(self, psi_hash, rho, u, lam, j, clamp_width, factorization=None, psi_ref=None,
                 iterations=0, relres=0.0):
        self._psi_hash = psi_hash
        self._psi_ref = psi_ref
        self.rho, self.u, self.lam, self.j = rho, u, lam, j
        self.clamp_width = clamp_width
        self.factorization = factorization
        self.iterations, self.relres = iterations, relres
        # numpy mode: the device copies the host arrays were made from, reused by gradient()
        # while solution.rho/u/lam are still those very objects (no re-upload)
        self._dev = None

    @property
    def psi_hash(self) -> str:
        if self._psi_hash is None:  # native mode: hash on first request only
            self._psi_hash = psi_digest(self._psi_ref[0])
        return self._psi_hash

    def __repr__(self):
        return f"HdmSolution(j={self.j!r}, clamp_width={self.clamp_width!r}, iterations={self.iterations})"


class HdmSolver:
    """Full-order objective and adjoint gradient on one GPU (hdm.py:112-233).

    Extra keyword arguments: ``rtol`` (pCG true-residual tolerance; the default None solves to
    round-off like the reference's direct solve -- target 1e-12, a true residual that stagnates
    at its attainable floor accepted up to 1e-7 -- which the reference's finite-difference gradient tests need; the
    BASELINE configs pass their own strict rtol: 1e-10 for cfg 1-2, 1e-8 for cfg 3-5),
    ``maxit``, ``device`` and ``preconditioner`` ("jacobi", the BASELINE design, or "mg":
    geometric multigrid with Galerkin coarse operators).  The default (None) is
    "mg" in round-off mode when the grid coarsens (Jacobi-pCG stalls near a 1e-9 relative
    residual on ill-conditioned designs, above the reference's trust-region centre checks) and
    "jacobi" otherwise.
    """

    def __init__(self, mesh: StructuredMesh, k_e, filt: HelmholtzFilter, f, fixed_dofs,
                 material: MaterialModel | None = None, stats: RunStats | None = None,
                 rtol: float | None = None, maxit: int = 200000, device=None, preconditioner: str | None = None):
        self.mesh = mesh
        self.k_e = np.asarray(k_e, dtype=float)
        self.filter = filt
        self.fixed_dofs = np.asarray(fixed_dofs, dtype=np.int64)
        self.material = material or MaterialModel()
        self.stats = stats or RunStats()
        # rtol None: round-off mode, passed to the C ABI as a negative tolerance
        self.rtol = ROUNDOFF_RTOL if rtol is None else float(rtol)
        self.maxit = int(maxit)
        f = np.asarray(f.detach().cpu().numpy() if _lib.is_torch(f) else f, dtype=float).copy()
        f[self.fixed_dofs] = 0.0  # loads on constrained dofs go into reactions (hdm.py:136-137)
        self.f = f
        free_mask = np.ones(mesh.n_dofs, dtype=bool)
        free_mask[self.fixed_dofs] = False
        self.free_mask = free_mask
        dim, nz = _lib.mesh_dims(mesh)
        nde = (2**dim) * dim
        if self.k_e.shape != (nde, nde):
            raise ValueError(f"element matrix must be {(nde, nde)}, got {self.k_e.shape}")
        self.device = filt.device if device is None else _lib.require_cuda(device)
        fixed_u8 = np.ascontiguousarray((~free_mask).astype(np.uint8))
        ke = np.ascontiguousarray(self.k_e)
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().tb_plan_create(
            dim, mesh.nx, mesh.ny, nz, mesh.h, ke.ctypes.data_as(ctypes.c_void_p),
            self.material.rho_l, self.material.p, fixed_u8.ctypes.data_as(ctypes.c_void_p),
            self.device.index, ctypes.byref(h)), "HdmSolver")
        self._plan = h
        if preconditioner not in (None, "jacobi", "mg"):
            raise ValueError(f"preconditioner must be 'jacobi' or 'mg', got {preconditioner!r}")
        if preconditioner is None:
            # default: the drop-in's round-off mode (rtol None, standing in for the reference's
            # direct solve) takes multigrid where the grid coarsens -- Jacobi-pCG stalls near a
            # 1e-9 relative residual on ill-conditioned SIMP designs, above what the reference's
            # trust-region centre checks demand (trustregion.py:360-375); an explicit rtol (the
            # BASELINE configurations) keeps the north_star's Jacobi-pCG
            preconditioner = "jacobi"
            if rtol is None and _lib.lib().tb_plan_set_preconditioner(h, 1) == 0:
                preconditioner = "mg"
        elif preconditioner == "mg":
            _lib.check(_lib.lib().tb_plan_set_preconditioner(h, 1), "multigrid set-up")
        self.preconditioner = preconditioner
        self._f_d = _lib.to_dev(self.f, self.device)
        self._fixed_d = _lib.to_dev(fixed_u8, self.device, dtype=_lib.torch().uint8)
        self.last_iterations = 0
        self.last_relres = 0.0

    def __del__(self):
        h = getattr(self, "_plan", None)
        if h is not None and h.value and _lib._lib is not None:
            _lib._lib.tb_plan_destroy(h)
            self._plan = None

    # ------------------------------------------------------------------ device helpers
    def _stream(self):
        return _lib.stream_ptr(self.device)

    def _empty(self, n):
        t = _lib.torch()
        return t.empty(n, dtype=t.float64, device=self.device)

    def filtered_density_device(self, psi_d):
        """(rho, clamp_width) on the device; counts one filter solve (hdm.py:144-154)."""
        _, rho_raw = self.filter.apply_device(psi_d, want_phi=False)
        self.stats.filter_solves += 1
        rho = self._empty(self.mesh.n_elems)
        cw = ctypes.c_double(0.0)
        _lib.check(_lib.lib().tb_clamp_density(self._plan, _lib.ptr(rho_raw), _lib.ptr(rho), ctypes.byref(cw),
                                               self._stream()), "clamp")
        return rho, float(cw.value)

    def pcg_device(self, rho_d, b_d, rtol=None):
        """Solve Z K(rho) Z x = Z b on the device (replaces PatternAssembler.factorize + solve)."""
        x = self._empty(self.mesh.n_dofs)
        it, rr = ctypes.c_int(0), ctypes.c_double(0.0)
        _lib.check(_lib.lib().tb_pcg_solve(self._plan, _lib.ptr(rho_d), _lib.ptr(b_d), _lib.ptr(x),
                                           self.rtol if rtol is None else rtol, self.maxit, ctypes.byref(it),
                                           ctypes.byref(rr), self._stream()), "pCG solve")
        self.last_iterations, self.last_relres = it.value, rr.value
        return x

    def last_kernel_time(self):
        """(ms, launches): device time spanned by the persistent multigrid-pCG launches of the last
        solve (2D, preconditioner "mg"); (0.0, 0) when it ran the graph path (tb_pcg_kernel_time)."""
        ms, n = ctypes.c_float(0.0), ctypes.c_int(0)
        _lib.check(_lib.lib().tb_pcg_kernel_time(self._plan, ctypes.byref(ms), ctypes.byref(n)), "kernel time")
        return float(ms.value), int(n.value)

    def dot_device(self, a_d, b_d) -> float:
        out = ctypes.c_double(0.0)
        _lib.check(_lib.lib().tb_dot(self._plan, _lib.ptr(a_d), _lib.ptr(b_d), a_d.numel(), ctypes.byref(out),
                                     self._stream()), "dot")
        return float(out.value)

    def sensitivity_device(self, rho_d, u_d, lam_d, drho_d=None):
        s = self._empty(self.mesh.n_elems)
        _lib.check(_lib.lib().tb_element_sensitivity(self._plan, _lib.ptr(rho_d), _lib.ptr(u_d), _lib.ptr(lam_d),
                                                     _lib.ptr(drho_d), _lib.ptr(s), self._stream()),
                   "element_sensitivity")
        return s

    def apply_device(self, rho_d, v_d, mask_rows=True):
        y = self._empty(self.mesh.n_dofs)
        _lib.check(_lib.lib().tb_apply_stiffness(self._plan, _lib.ptr(rho_d), _lib.ptr(v_d), _lib.ptr(y),
                                                 1 if mask_rows else 0, self._stream()), "apply_stiffness")
        return y

    def _user(self, x_d, native):
        return _lib.to_user(x_d, native)

    # ------------------------------------------------------------------ reference API
    def filtered_density(self, psi):
        native = _lib.is_torch(psi)
        rho, cw = self.filtered_density_device(_lib.to_dev(psi, self.device))
        return self._user(rho, native), cw

    def _check_density(self, rho) -> None:
        lo, hi = self.material.rho_l, 1.0
        rmin, rmax = (float(rho.min()), float(rho.max()))
        if rmin < lo - 1e-12 or rmax > hi + 1e-12:
            raise ValueError(f"density out of admissible range [{lo}, {hi}]: min={rmin}, max={rmax}")

    def assemble_stiffness(self, rho):
        """Sparse K(rho) for diagnostics (hdm.py:164-168); host scipy, not used by any solver."""
        rho = np.asarray(rho.detach().cpu().numpy() if _lib.is_torch(rho) else rho, dtype=float)
        self._check_density(rho)
        return assemble(self.mesh, self.k_e, self.material.alpha(rho), "vector")

    def solve(self, psi, objective: Objective) -> HdmSolution:
        """Filter, solve and evaluate the objective at psi (hdm.py:170-197)."""
        native = _lib.is_torch(psi)
        psi_d = _lib.to_dev(psi, self.device)
        if tuple(psi_d.shape) != (self.mesh.n_elems,):
            raise ValueError(f"psi must have length {self.mesh.n_elems}, got shape {tuple(psi_d.shape)}")
        # numpy design: its byte snapshot (for gradient's staleness check) is taken by a worker
        # thread while the device filters and solves
        snap_job = None if native else _host_pool().submit(np.array, psi, dtype=float, copy=True)
        rho_d, clamp_width = self.filtered_density_device(psi_d)
        rho_host = None if native else _lib.to_host_async(rho_d)  # lands while the solve runs
        # the clamp guarantees [rho_l, 1]; NaN input surfaces as a pCG breakdown
        self.stats.factorizations += 1
        u_d = self.pcg_device(rho_d, self._f_d)
        iters, relres = self.last_iterations, self.last_relres
        self.stats.hdm_solves += 1
        rho_u = rho_d if native else _lib.finish_host(rho_host)
        u_u = self._user(u_d, native)
        if objective.is_compliance:
            lam_u = u_u
            if isinstance(objective, ComplianceObjective):
                j = self.dot_device(objective.device_f(self.device), u_d)
            else:
                j = float(objective.value(u_u, rho_u))
        else:
            g_d = _lib.to_dev(objective.du(u_u, rho_u), self.device)
            lam_u = self._user(self.pcg_device(rho_d, g_d), native)
            self.stats.hdm_adjoint_solves += 1
            j = float(objective.value(u_u, rho_u))
        if native:
            keep = psi_d.clone() if psi_d is psi else psi_d  # snapshot of the design's bytes
            return HdmSolution(None, rho_u, u_u, lam_u, j, clamp_width, None, psi_ref=(keep, psi, psi._version),
                               iterations=iters, relres=relres)
        # numpy design: keep a byte snapshot; psi_hash (SHA-256, hdm.py:36-37) is computed on
        # first request and gradient() compares bytes directly (same strictness, no hashing)
        snap = snap_job.result()
        sol = HdmSolution(None, rho_u, u_u, lam_u, j, clamp_width, None, psi_ref=(snap, None, None),
                          iterations=iters, relres=relres)
        sol._dev = ((rho_u, u_u, lam_u), (rho_d, u_d, u_d if lam_u is u_u else None))
        return sol

    def gradient(self, psi, solution: HdmSolution, objective: Objective):
        """Adjoint gradient of J at psi; requires a matching solution (hdm.py:199-209)."""
        native = _lib.is_torch(psi)
        ref = solution._psi_ref
        if native and ref is not None and _lib.is_torch(ref[0]):
            snap, src, version = ref
            if psi is src and psi._version == version:
                same = True  # the very tensor the solution was computed from, never modified since
            else:
                same = tuple(snap.shape) == tuple(psi.shape) and bool(
                    _lib.torch().equal(snap, psi.to(snap.device, snap.dtype)))
        elif not native and ref is not None and isinstance(ref[0], np.ndarray):
            # compared by a worker thread while the device computes the gradient; a mismatch
            # raises before anything is returned (the gradient does not touch RunStats)
            same = _host_pool().submit(_same_bytes, psi, ref[0])
        else:
            same = psi_digest(psi) == solution.psi_hash
        if same is False:
            raise StaleSolutionError("solution was computed at a different design than psi")
        dev = solution._dev
        if (dev is not None and dev[1][2] is not None and solution.rho is dev[0][0] and solution.u is dev[0][1]
                and solution.lam is dev[0][2] and objective.is_compliance):
            s_d = self.sensitivity_device(dev[1][0], dev[1][1], dev[1][2])  # device copies, no re-upload
        else:
            s_d = self._sensitivity(solution.rho, solution.u, solution.lam, objective)
        g_d = self.filter.apply_adjoint_device(s_d)
        if not isinstance(same, bool) and not same.result():
            raise StaleSolutionError("solution was computed at a different design than psi")
        return self._user(g_d, native)

    def _sensitivity(self, rho, u, lam, objective):
        rho_d = _lib.to_dev(rho, self.device)
        u_d = _lib.to_dev(u, self.device)
        lam_d = u_d if lam is u else _lib.to_dev(lam, self.device)
        drho_d = None
        if not objective.is_compliance:
            drho_d = _lib.to_dev(objective.drho(u, rho), self.device)
        return self.sensitivity_device(rho_d, u_d, lam_d, drho_d)

    def element_sensitivity(self, rho, u, lam, objective: Objective):
        """dj/drho_e - alpha'(rho_e) u_e^T K_e lam_e (hdm.py:211-222)."""
        return self._user(self._sensitivity(rho, u, lam, objective), _lib.is_torch(u))

    def apply_stiffness(self, rho, v):
        """Matrix-free K(rho) v with fixed rows zeroed (hdm.py:224-233)."""
        native = _lib.is_torch(v)
        return self._user(self.apply_device(_lib.to_dev(rho, self.device), _lib.to_dev(v, self.device)), native)
