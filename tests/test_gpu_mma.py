"""Device MMA step against the reference MmaOptimizer trajectories and the
reference's own unit tests (pkg/tests/test_mma.py), run through the CUDA path."""

import numpy as np
import pytest
import torch

import paper_2004_05756_b200 as tb
from conftest import golden
from mma_cases import mma_cases
from oracle.mma import MmaOracle

pytestmark = pytest.mark.gpu


def two_var(move=0.5):
    return tb.MmaOptimizer(np.zeros(2), np.ones(2), np.ones(2), 1.0, tb.MmaConfig(move=move))


def test_trajectories_match_reference(cuda):
    """Bit-identical per-element arithmetic; only w.x sums differ in order, so iterates agree
    with the reference to the bisection tolerance."""
    G = golden("golden_mma.npz")
    for name, lower, upper, w, cap, x0, grads, caps in mma_cases():
        opt = tb.MmaOptimizer(lower, upper, w, cap)
        ora = MmaOracle(lower, upper, w, cap)
        x, xo = x0, x0
        for k, (g, mc) in enumerate(zip(grads, caps)):
            x = opt.step(x, 0.0, g, move_cap=mc)
            xo = ora.step(xo, g, move_cap=mc)
            ref = G[f"{name}_xs"][k]
            assert np.abs(x - ref).max() <= 1e-9, (name, k, np.abs(x - ref).max())
            assert np.abs(x - xo).max() <= 1e-9
            assert w @ x <= cap * (1 + 1e-12) + 1e-12
        assert np.abs(opt.low - G[f"{name}_low"]).max() <= 1e-9
        assert np.abs(opt.upp - G[f"{name}_upp"]).max() <= 1e-9


def test_inactive_volume_is_bit_exact(cuda):
    """When the volume bound is slack the step has no reduction-dependent branch: x_new is
    bit-identical to the reference."""
    G = golden("golden_mma.npz")
    name, lower, upper, w, cap, x0, grads, caps = mma_cases()[2]
    opt, ora = tb.MmaOptimizer(lower, upper, w, cap), MmaOracle(lower, upper, w, cap)
    x = opt.step(x0, 0.0, grads[0])
    xo = ora.step(x0, grads[0])
    if w @ xo < cap - 1e-6:
        assert np.array_equal(x, xo)
        assert np.array_equal(x, G[f"{name}_xs"][0])


def test_zero_gradient_keeps_iterate(cuda):
    opt = two_var()
    x = np.array([0.3, 0.6])
    assert np.abs(opt.step(x, 1.0, np.zeros(2)) - x).max() < 1e-13


def test_two_variable_descent_hits_volume_or_box(cuda):
    opt = two_var(move=0.5)
    x = np.array([0.5, 0.5])
    x_new = opt.step(x, 1.0, np.ones(2))
    assert np.all(x_new <= x)
    assert x_new @ np.ones(2) <= 1.0 + 1e-12
    assert np.all(x_new < 0.25)


def test_negative_gradient_drives_volume_active(cuda):
    opt = two_var(move=0.5)
    x_new = opt.step(np.array([0.4, 0.4]), -1.0, np.array([-1.0, -1.0]))
    assert abs(x_new @ np.ones(2) - 1.0) <= 1e-10
    assert abs(x_new[0] - x_new[1]) < 1e-12


def test_asymmetric_gradient_kkt(cuda):
    opt = two_var(move=0.9)
    x_new = opt.step(np.array([0.5, 0.5]), 0.0, np.array([-2.0, -1.0]))
    assert abs(x_new.sum() - 1.0) <= 1e-10
    assert x_new[0] > x_new[1]


def test_rejects_bad_inputs_and_keeps_state(cuda):
    opt = two_var()
    with pytest.raises(ValueError, match="box"):
        opt.step(np.array([1.2, 0.0]), 0.0, np.zeros(2))
    with pytest.raises(ValueError, match="volume"):
        opt.step(np.array([0.9, 0.9]), 0.0, np.zeros(2))
    with pytest.raises(ValueError, match="finite"):
        opt.step(np.array([0.2, 0.2]), 0.0, np.array([np.nan, 0.0]))
    assert opt.it == 0 and opt.xold1 is None and opt.low is None
    with pytest.raises(ValueError):
        tb.MmaOptimizer(np.zeros(2), np.ones(2), np.array([1.0, -1.0]), 1.0)
    with pytest.raises(ValueError):
        tb.MmaOptimizer(np.ones(2), np.ones(2), np.ones(2), 1.0)


def test_move_cap_limits_step(cuda):
    opt = two_var(move=0.5)
    x = np.array([0.5, 0.5])
    x_new = opt.step(x, 0.0, np.array([5.0, -5.0]), move_cap=0.01)
    assert np.abs(x_new - x).max() <= 0.01 + 1e-14


@pytest.mark.parametrize("seed", range(12))
def test_feasibility_random_steps(cuda, seed):
    rng = np.random.default_rng(seed)
    n = 6
    w = 0.5 + rng.random(n)
    cap = 0.6 * w.sum()
    opt = tb.MmaOptimizer(np.zeros(n), np.ones(n), w, cap)
    x = np.full(n, 0.5)
    x = x * min(1.0, cap / (w @ x))
    for _ in range(4):
        x = opt.step(x, 0.0, rng.standard_normal(n))
        assert np.all(x >= -1e-14) and np.all(x <= 1.0 + 1e-14)
        assert w @ x <= cap + 1e-10
        assert np.all(opt.low < x - 1e-12) and np.all(opt.upp > x + 1e-12)


def test_device_tensors_in_device_tensors_out(cuda):
    n = 300000  # cfg-2 sized design vector: many CTAs, one cooperative launch per step
    rng = np.random.default_rng(5)
    w = torch.ones(n, dtype=torch.float64, device=cuda)
    lo, up = torch.zeros_like(w), torch.ones_like(w)
    opt = tb.MmaOptimizer(lo, up, w, 0.3 * n)
    x = torch.full((n,), 0.3, dtype=torch.float64, device=cuda)
    ora = MmaOracle(np.zeros(n), np.ones(n), np.ones(n), 0.3 * n)
    xo = np.full(n, 0.3)
    for _ in range(3):
        g = -np.abs(rng.standard_normal(n)) - 0.01
        x = opt.step(x, 0.0, torch.as_tensor(g, device=cuda))
        xo = ora.step(xo, g)
        assert x.is_cuda
        assert np.abs(x.cpu().numpy() - xo).max() <= 1e-9
        assert float(w @ x) <= 0.3 * n * (1 + 1e-12)
