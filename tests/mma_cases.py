"""Seeded MMA problems shared by tests/golden/make_golden.py (which runs the reference
MmaOptimizer on them) and the tests (which replay them on the oracle and the device)."""

import numpy as np


def mma_cases():
    """(name, lower, upper, w, cap, x0, grads, move_caps) for each trajectory."""
    cases = []
    rng = np.random.default_rng(11)
    n = 6
    w = 0.5 + rng.random(n)
    cap = 0.6 * w.sum()
    x0 = np.full(n, 0.5)
    x0 = x0 * min(1.0, cap / (w @ x0))
    cases.append(("six", np.zeros(n), np.ones(n), w, cap, x0, rng.standard_normal((6, n)), [None] * 6))
    # compliance-like (negative) gradients: the volume bound is active and bisected every step
    n = 2000
    w = np.ones(n)
    cap = 0.4 * n
    x0 = np.full(n, 0.4)
    base = -np.abs(np.sin(np.linspace(0.0, 7.0, n))) - 0.05
    grads = np.stack([base * (1.0 + 0.3 * rng.standard_normal(n)) for _ in range(6)])
    cases.append(("active", np.zeros(n), np.ones(n), w, cap, x0, grads, [None, None, 0.05, None, 0.02, None]))
    # non-uniform weights and bounds, mixed-sign gradients (volume inactive on some steps)
    n = 500
    lower = 0.01 * rng.random(n)
    upper = 0.9 + 0.1 * rng.random(n)
    w = 0.2 + rng.random(n)
    cap = 0.5 * w @ upper
    x0 = lower + 0.45 * (upper - lower)
    cases.append(("mixed", lower, upper, w, cap, x0, rng.standard_normal((6, n)), [None] * 6))
    return cases
