"""Parity at the bench's full grid size (BASELINE configs[1]: 256^3) and
above, where the small-case tests cannot reach: the chunk / wave model picks
the production launch shapes (10 z-chunks of 26 planes, 2.9 waves of CTAs)
only on big grids.

* 256^3 superposed gradient vs the C oracle (bit-exact, fewer time steps
  than the bench so the oracle finishes in seconds);
* 512^3: two-step passes vs single steps, bit-exact (size-independent
  property: both are exact restatements of the same update);
* 256^3 fp64 time reversal: forward then backward replay returns to the zero
  initial state (SPEC acceptance 2 at full size)."""

import numpy as np
import pytest

from helpers import bits_equal
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def W():
    import paper_2509_15744_b200 as W

    from paper_2509_15744_b200 import _native

    _native.load(require_device=True)
    return W


def _bench_like(W, n, n_steps, seed=0):
    rng = np.random.default_rng(seed)
    shape = (n, n, n)
    dx = 1e-4
    dt = 0.45 * dx / 6000.0 / np.sqrt(3)
    gamma = rng.uniform(0.3, 1.0, size=shape)
    grid = W.build_grid(shape, dx)
    mat = W.MaterialModel.rho_scaled(gamma, grid, rho0=2700.0, c0=6000.0)
    src = W.SourceSpec(node=(3, n // 2, n // 2), amplitude=1e12, frequency=0.05 / dt, cycles=2)
    lin = np.unique(np.round(np.linspace(2, n - 3, 33)).astype(int))
    sens = [(n - 4, int(j), int(k)) for j in lin for k in lin]
    meas = rng.normal(scale=1e-10, size=(1, len(sens), n_steps))
    problem = W.FwiProblem(grid=grid, time=W.TimeConfig(n_steps, dt), material=mat,
                           sources=[src], sensors=W.SensorArray(nodes=sens), measured=meas)
    omat = O.Material("rho_scaled", gamma, dx, rho0=2700.0, c0=6000.0)
    support = np.array([grid.flat_index(s) for s in sens], dtype=np.int64)
    shots = [(O.Source(src.node, 1e12, 0.05 / dt, 2), O.FwiShot(support, meas[0], dt))]
    return problem, mat, omat, dt, shots


@pytest.mark.parametrize("prec", ["single", "double"])
def test_bench_grid_gradient_matches_oracle(W, prec):
    from paper_2509_15744_b200 import engine

    n_steps = 24
    problem, mat, omat, dt, shots = _bench_like(W, 256, n_steps)
    ctx = engine.get_context(problem.grid, W.precision_dtype(prec))
    ctx.set_two_step(2)                      # two-step passes for fp64 too
    ctx.reset_stats()
    try:
        res = W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=1e13, precision=prec))
        assert ctx.stats()["pair_launches"] > 0
    finally:
        ctx.set_two_step(1)
    cost, grad, _ = O.gradient_superposed(omat, dt, n_steps, shots, 1e13, prec)
    assert bits_equal(res.gradient, grad)
    assert abs(res.cost - cost) <= 1e-13 * abs(cost)


def test_two_step_equals_single_step_512(W):
    from paper_2509_15744_b200 import engine

    problem, mat, _, _, _ = _bench_like(W, 512, 12, seed=1)
    cfg = W.SuperpositionConfig(k=1e13, precision="single")
    ctx = engine.get_context(problem.grid, np.float32)
    try:
        ctx.set_two_step(0)
        single = W.gradient_superposed(problem, mat, cfg)
        ctx.set_two_step(1)
        ctx.reset_stats()
        paired = W.gradient_superposed(problem, mat, cfg)
        assert ctx.stats()["pair_launches"] > 0
    finally:
        ctx.set_two_step(1)
        engine.release_contexts()
    assert bits_equal(paired.gradient, single.gradient)
    assert paired.cost == single.cost


def test_time_reversal_roundtrip_256(W):
    n, n_steps = 256, 120
    dx = 1e-4
    dt = 0.5 * dx / 6000.0
    grid = W.build_grid((n, n, n), dx)
    mat = W.MaterialModel.rho_scaled(np.ones((n, n, n)), grid, rho0=2700.0, c0=6000.0)
    src = W.SourceSpec(node=(n // 2, n // 2, n // 2), amplitude=1e12, frequency=0.05 / dt,
                       cycles=2)
    time = W.TimeConfig(n_steps, dt)
    fwd = W.run_forward(mat, time, [src])
    idx = np.array([grid.flat_index(src.node)])
    back = W.run_backward(mat, time, fwd.window,
                          lambda k: (idx, np.array([W.burst_amplitude(k * dt, src)])))
    assert np.max(np.abs(back.u_cur)) <= 1e-10 * fwd.peak_abs
