"""Dev: one superposed gradient on an n0 x n1 x n2 FWI grid (for ncu per-pass timing)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "profiles"))
import numpy as np  # noqa: E402

import paper_2509_15744_b200 as W  # noqa: E402

shape = tuple(int(a) for a in sys.argv[1:4])
dx, c0 = 1e-4, 6000.0
grid = W.build_grid(shape, dx)
mat = W.MaterialModel.rho_scaled(np.ones(shape), grid, rho0=2700.0, c0=c0)
n = shape
src = W.SourceSpec(node=(3, n[1] // 2, n[2] // 2), amplitude=1e12, frequency=5e6, cycles=2)
sens = [(n[0] - 4, j, k) for j in range(8, n[1] - 8, 8) for k in range(8, n[2] - 8, 8)]
N = 24
meas = np.random.default_rng(0).normal(scale=1e-9, size=(1, len(sens), N))
problem = W.FwiProblem(grid=grid, time=W.TimeConfig(N, 0.5 * dx / c0), material=mat,
                       sources=[src], sensors=W.SensorArray(nodes=sens), measured=meas)
W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=1e13, precision="single"))
