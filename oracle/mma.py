"""CPU restatement of the reference MMA step (romtopt/mma.py:41-175).

TEST INFRASTRUCTURE ONLY: used by tests/ as the checker of the device MmaOptimizer, never by
the product path.  Pinned against tests/golden/golden_mma.npz (the reference's own
MmaOptimizer run on tests/mma_cases.py).
"""

from __future__ import annotations

import numpy as np

DEFAULTS = dict(asy_init=0.5, asy_incr=1.2, asy_decr=0.7, asy_min_frac=0.01, asy_max_frac=10.0, move=0.2,
                albefa=0.1, raa0=1e-5, bisect_rtol=1e-12, bisect_max_iter=200)  # mma.py:25-38


class MmaOracle:
    """min F over [lower, upper] with w . x <= cap, one separable convex model per step."""

    def __init__(self, lower, upper, w, cap, **cfg):
        self.lo = np.asarray(lower, float)
        self.hi = np.asarray(upper, float)
        self.w = np.asarray(w, float)
        self.cap = float(cap)
        self.c = dict(DEFAULTS, **cfg)
        self.span = self.hi - self.lo
        self.k = 0
        self.hist = []  # previous iterates, newest last (at most two kept)
        self.asy = None  # (low, upp) of the previous step

    def _asymptotes(self, x):
        """mma.py:71-89: reset for the first two steps, else widen/narrow by oscillation."""
        c, s = self.c, self.span
        if self.k <= 2 or len(self.hist) < 2:
            low, upp = x - c["asy_init"] * s, x + c["asy_init"] * s
        else:
            x1, x2 = self.hist[-1], self.hist[-2]
            osc = (x - x1) * (x1 - x2)
            f = np.where(osc > 0, c["asy_incr"], np.where(osc < 0, c["asy_decr"], 1.0))
            low = x - f * (x1 - self.asy[0])
            upp = x + f * (self.asy[1] - x1)
        low = np.minimum(np.maximum(low, x - c["asy_max_frac"] * s), x - c["asy_min_frac"] * s)
        upp = np.minimum(np.maximum(upp, x + c["asy_min_frac"] * s), x + c["asy_max_frac"] * s)
        return low, upp

    def step(self, x, grad, move_cap=None):
        x = np.asarray(x, float)
        g = np.asarray(grad, float)
        if not np.all(np.isfinite(g)):  # mma.py:112-119
            raise ValueError("gradient must be finite")
        if np.any(x < self.lo - 1e-12) or np.any(x > self.hi + 1e-12):
            raise ValueError("iterate outside box bounds")
        if self.w @ x > self.cap * (1.0 + 1e-9) + 1e-12:
            raise ValueError("iterate violates the volume constraint")
        c = self.c
        self.k += 1
        low, upp = self._asymptotes(x)
        mv = c["move"] * self.span  # mma.py:122-131
        if move_cap is not None:
            mv = np.minimum(mv, move_cap)
        a = np.maximum(np.maximum(self.lo, low + c["albefa"] * (x - low)), x - mv)
        b = np.minimum(np.minimum(self.hi, upp - c["albefa"] * (upp - x)), x + mv)
        gp, gm = np.maximum(g, 0.0), np.maximum(-g, 0.0)  # mma.py:133-141
        r0 = c["raa0"] / self.span
        p0 = (upp - x) ** 2 * (1.001 * gp + 0.001 * gm + r0)
        q0 = (x - low) ** 2 * (0.001 * gp + 1.001 * gm + r0)
        p1 = (upp - x) ** 2 * self.w
        sq = np.sqrt(q0)

        def primal(lam):  # mma.py:143-146: closed-form minimiser for a given multiplier
            sp = np.sqrt(p0 + lam * p1)
            return np.clip((low * sp + upp * sq) / (sp + sq), a, b)

        tol = c["bisect_rtol"] * max(abs(self.cap), 1.0)  # mma.py:148-170
        xn = primal(0.0)
        if not self.w @ xn <= self.cap + tol:
            lam_lo, lam_hi = 0.0, 1.0
            while self.w @ primal(lam_hi) > self.cap:
                lam_lo, lam_hi = lam_hi, lam_hi * 10.0
                if lam_hi > 1e40:
                    raise RuntimeError("volume multiplier bracket failed")
            xn = primal(lam_hi)
            for _ in range(c["bisect_max_iter"]):
                mid = 0.5 * (lam_lo + lam_hi)
                xm = primal(mid)
                if self.w @ xm > self.cap:
                    lam_lo = mid
                else:
                    lam_hi, xn = mid, xm
                if abs(self.w @ xn - self.cap) <= tol:
                    break
        self.hist = (self.hist + [x.copy()])[-2:]
        self.asy = (low, upp)
        return xn
