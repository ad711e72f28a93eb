"""Method of Moving Asymptotes on the device (reference ``romtopt/mma.py``).

``MmaOptimizer`` keeps the reference signature and semantics (mma.py:41-175): box bounds plus
one linear volume bound, Svanberg-style asymptote memory, the exact separable subproblem solved
by bracketing and bisecting the volume multiplier.  The asymptote memory lives in device
memory, and one ``step`` is one cooperative kernel (``tb_mma_step``).  The per-element
expressions round exactly as numpy's; only the dot products ``w @ x`` sum in a different order.

It is the trust-region subproblem engine (trustregion.py:320): the inner
loop ``x -> MMA step -> reduced model`` stays on the GPU, see ``subproblem.py``.

numpy in -> numpy out (reference behaviour); CUDA tensors in -> CUDA tensors out.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _lib

__all__ = ["MmaConfig", "MmaOptimizer"]


@dataclass(frozen=True)
class MmaConfig:
    """Standard moving-asymptote parameters (mma.py:25-38, same defaults)."""

    asy_init: float = 0.5
    asy_incr: float = 1.2
    asy_decr: float = 0.7
    asy_min_frac: float = 0.01
    asy_max_frac: float = 10.0
    move: float = 0.2
    albefa: float = 0.1
    raa0: float = 1e-5
    bisect_rtol: float = 1e-12
    bisect_max_iter: int = 200

    def _c(self) -> _lib.MmaConfigC:
        return _lib.MmaConfigC(self.asy_init, self.asy_incr, self.asy_decr, self.asy_min_frac, self.asy_max_frac,
                               self.move, self.albefa, self.raa0, self.bisect_rtol, int(self.bisect_max_iter))


class MmaOptimizer:
    """Sequential MMA state for min F(x) over [lower, upper] with w @ x <= V (mma.py:41-69).

    Mutates its asymptote memory on every :meth:`step`; a fresh instance gives a deterministic
    replay.  ``low``/``upp``/``xold1``/``xold2`` mirror the reference attributes (numpy views
    of the device state, ``None`` before they exist).
    """

    def __init__(self, lower, upper, volume_weights, volume_cap: float, config: MmaConfig | None = None,
                 device=None):
        t = _lib.torch()
        if device is None:
            device = next((a.device for a in (lower, upper, volume_weights) if _lib.is_torch(a)), None)
        self.device = _lib.require_cuda(device)
        lo = _lib.to_dev(lower, self.device).contiguous()
        up = _lib.to_dev(upper, self.device).contiguous()
        w = _lib.to_dev(volume_weights, self.device).contiguous()
        if lo.ndim != 1 or lo.shape != up.shape or lo.shape != w.shape:
            raise ValueError("lower, upper and volume_weights must be 1-D arrays of the same length")
        if bool(t.any(lo >= up)):
            raise ValueError("lower bounds must be strictly below upper bounds")
        if bool(t.any(w <= 0.0)):
            raise ValueError("volume weights must be positive")
        self._lower, self._upper, self._w = lo, up, w
        self.volume_cap = float(volume_cap)
        self.cfg = config or MmaConfig()
        self._cfg_c = self.cfg._c()
        self.n = int(lo.shape[0])
        self.range = up - lo
        self.it = 0
        z = lambda: t.zeros(self.n, dtype=t.float64, device=self.device)  # noqa: E731
        self._xold1, self._xold2, self._low, self._upp = z(), z(), z(), z()
        self._has1 = self._has2 = self._has_asy = False
        nbytes = int(_lib.lib().tb_mma_workspace_bytes(self.n))
        self._ws = t.zeros(nbytes, dtype=t.uint8, device=self.device)

    # reference attribute names (None until set, mma.py:65-69)
    @property
    def lower(self):
        return self._lower.cpu().numpy()

    @property
    def upper(self):
        return self._upper.cpu().numpy()

    @property
    def w(self):
        return self._w.cpu().numpy()

    @property
    def xold1(self):
        return self._xold1.cpu().numpy() if self._has1 else None

    @property
    def xold2(self):
        return self._xold2.cpu().numpy() if self._has2 else None

    @property
    def low(self):
        return self._low.cpu().numpy() if self._has_asy else None

    @property
    def upp(self):
        return self._upp.cpu().numpy() if self._has_asy else None

    def step(self, x, f_val: float, grad, move_cap: float | None = None):
        """One MMA update from the feasible point ``x`` with gradient ``grad`` (mma.py:91-175).

        Returns the exact minimizer of the convex separable approximation over the
        move-limited box intersected with the volume constraint.  Raises ValueError for a
        non-finite gradient, an iterate outside the box or violating the volume bound (state
        untouched), RuntimeError if the volume multiplier cannot be bracketed.
        """
        del f_val
        t = _lib.torch()
        native = _lib.is_torch(x)
        xd = _lib.to_dev(x, self.device).contiguous()
        gd = _lib.to_dev(grad, self.device).contiguous()
        if xd.shape != (self.n,) or gd.shape != (self.n,):
            raise ValueError(f"x and grad must have shape ({self.n},)")
        out = t.empty(self.n, dtype=t.float64, device=self.device)
        it = self.it + 1
        rc = _lib.lib().tb_mma_step(
            self.n, _lib.ptr(xd), _lib.ptr(gd), _lib.ptr(self._lower), _lib.ptr(self._upper), _lib.ptr(self._w),
            self.volume_cap, -1.0 if move_cap is None else float(move_cap), it, int(self._has1), int(self._has2),
            ctypes.byref(self._cfg_c), _lib.ptr(self._xold1), _lib.ptr(self._xold2), _lib.ptr(self._low),
            _lib.ptr(self._upp), _lib.ptr(self._ws), _lib.ptr(out), _lib.stream_ptr(self.device))
        _lib.check(rc, "MMA step")
        self.it = it
        self._has2 = self._has1
        self._has1 = True
        self._has_asy = True
        return out if native else out.cpu().numpy()
