"""Trust-region subproblem on the device.

The reference's inner loop, ``TrustRegionDriver.solve_subproblem`` (trustregion.py:304-351)
with ``_evaluate_model`` (trustregion.py:298-302) and ``tr_constraint`` (trustregion.py:285-296),
runs up to ``max_inner`` (50) MMA steps per trust-region iteration.  Each step takes one
reduced-model evaluation: Helmholtz filter, ``RomModel.solve(compute_gradient=True)`` (which
adds a sensitivity and a filter-adjoint solve), and the residual-norm constraint.

Here every vector of that loop stays in device memory: the MMA step is one cooperative kernel
(``mma.py``), the filter is the matrix-free Helmholtz pCG, and the reduced solve, sensitivity
and residual norm are the ROM kernels.  Only the scalars the loop branches on (J, the residual
norm, the curvature quotient) come back to the host, as in the reference.  The driver around it
(radius update, acceptance, basis rebuild) stays out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .hdm import HdmSolver, Objective
from .mma import MmaConfig, MmaOptimizer
from .rom import ReducedBasis, RomModel

__all__ = ["SubproblemResult", "TrustRegionSubproblem"]


@dataclass
class SubproblemResult:
    """Outcome of one inner sweep (trustregion.py:238-252): candidate point and bookkeeping.
    Arrays are numpy when the centre was numpy, device tensors when it was a device tensor."""

    candidate: object
    model_value: float
    theta: float
    steps: int = 0
    rom_solves: int = 0
    curvature: float = 0.0
    first_iterate: object = None


class TrustRegionSubproblem:
    """The reduced-model subproblem of ``TrustRegionDriver`` with the same constraint kinds
    ("res": ROM residual norm, "dist": ||psi - psi_k||), bounds [0, 1] (trustregion.py:280-281)
    and MMA settings (``TrConfig.max_inner``, ``TrConfig.mma``)."""

    def __init__(self, solver: HdmSolver, rom: RomModel, objective: Objective, volume_weights, volume_cap: float,
                 constraint: str = "res", max_inner: int = 50, mma: MmaConfig | None = None):
        if constraint not in ("res", "dist"):
            raise ValueError(f"unknown constraint kind {constraint!r}")
        self.solver, self.rom, self.objective = solver, rom, objective
        self.device = solver.device
        self.w = _lib.to_dev(volume_weights, self.device).contiguous()
        self.cap = float(volume_cap)
        self.constraint = constraint
        self.max_inner = int(max_inner)
        self.mma = mma or MmaConfig()
        t = _lib.torch()
        n = solver.mesh.n_elems
        self.lower = t.zeros(n, dtype=t.float64, device=self.device)
        self.upper = t.ones(n, dtype=t.float64, device=self.device)

    def tr_constraint(self, psi, center_psi, residual_norm: float | None) -> float:
        """trustregion.py:285-296 (exponent 1)."""
        if self.constraint == "dist":
            t = _lib.torch()
            d = _lib.to_dev(psi, self.device) - _lib.to_dev(center_psi, self.device)
            return float(t.linalg.vector_norm(d))
        if residual_norm is None:
            raise ValueError("residual-based constraint needs a reduced solve")
        return float(residual_norm)

    def evaluate_model(self, basis: ReducedBasis, psi_d):
        """Reduced objective, gradient and residual at an iterate (trustregion.py:298-302)."""
        rho_d, _ = self.solver.filtered_density_device(psi_d)
        return self.rom.solve(basis, rho_d, self.objective, compute_gradient=True)

    def solve_subproblem(self, basis: ReducedBasis, psi_k, delta: float, j_center: float,
                         grad_center) -> SubproblemResult:
        """Inner MMA sweep on the reduced objective, stopped at the trust boundary
        (trustregion.py:304-351): returns the best in-region iterate (or the centre), the
        first iterate, the number of in-region steps and the largest curvature quotient."""
        t = _lib.torch()
        native = _lib.is_torch(psi_k)
        xk = _lib.to_dev(psi_k, self.device).contiguous()
        g_m = _lib.to_dev(grad_center, self.device).contiguous()
        opt = MmaOptimizer(self.lower, self.upper, self.w, self.cap, self.mma, device=self.device)
        x, j_m = xk, float(j_center)
        res = SubproblemResult(candidate=xk, model_value=float(j_center), theta=0.0)
        move_cap = delta / np.sqrt(xk.shape[0]) if self.constraint == "dist" else None
        for i in range(self.max_inner):
            x_new = opt.step(x, j_m, g_m, move_cap=move_cap)
            sol = self.evaluate_model(basis, x_new)
            res.rom_solves += 1
            if i == 0:
                res.first_iterate = x_new
            dx = x_new - x
            dx_norm = float(t.linalg.vector_norm(dx))
            if sol.grad is not None and dx_norm > 0.0:
                q = abs(float(t.dot(sol.grad - g_m, dx))) / dx_norm**2
                res.curvature = max(res.curvature, q)
            theta = self.tr_constraint(x_new, xk, sol.residual_norm)
            if theta > delta:
                break
            res.steps += 1
            # keep the best in-region model value (MMA may transiently raise the model)
            if sol.j < res.model_value:
                res.candidate, res.model_value, res.theta = x_new, sol.j, theta
            x, j_m, g_m = x_new, sol.j, sol.grad
        if not native:
            res.candidate = _lib.to_user(res.candidate, False)
            if res.first_iterate is not None:
                res.first_iterate = _lib.to_user(res.first_iterate, False)
        return res
