"""Subprocess body for test_two_step_long_chunks (env WB_T2_NZ set by the test)."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(HERE), HERE, os.path.join(HERE, "golden")]
import numpy as np  # noqa: E402

import paper_2509_15744_b200 as W  # noqa: E402
from helpers import bits_equal  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2509_15744_b200 import engine  # noqa: E402

shape, n_steps, prec = (45, 16, 64), 41, sys.argv[1]
rng = np.random.default_rng(8)
dx = 1e-4
gamma = rng.uniform(0.3, 1.0, size=shape)
grid = W.build_grid(shape, dx)
mat = W.MaterialModel.rho_scaled(gamma, grid, rho0=2700.0, c0=6000.0)
dt = 0.45 * dx / 6000.0 / np.sqrt(3)
src = W.SourceSpec(node=(20, 7, 40), amplitude=1e12, frequency=0.05 / dt, cycles=2)
sens = [(i, j, k) for i in (0, 22, 44) for j in (0, 8, 15) for k in (0, 63)]
meas = rng.normal(scale=1e-10, size=(1, len(sens), n_steps))
problem = W.FwiProblem(grid=grid, time=W.TimeConfig(n_steps, dt), material=mat, sources=[src],
                       sensors=W.SensorArray(nodes=sens), measured=meas)
ctx = engine.get_context(grid, W.precision_dtype(prec))
ctx.set_two_step(2)
ctx.reset_stats()
res = W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=1e13, precision=prec))
assert ctx.stats()["pair_launches"] > 0
omat = O.Material("rho_scaled", gamma, dx, rho0=2700.0, c0=6000.0)
support = np.array([grid.flat_index(n) for n in sens], dtype=np.int64)
shots = [(O.Source(src.node, 1e12, 0.05 / dt, 2), O.FwiShot(support, meas[0], dt))]
cost, grad, _ = O.gradient_superposed(omat, dt, n_steps, shots, 1e13, prec)
assert bits_equal(res.gradient, grad), "gradient differs"
assert abs(res.cost - cost) <= 1e-13 * abs(cost)
print("ok")
