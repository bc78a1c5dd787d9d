"""Dev repro: one gradient_superposed on a given shape with the two-step path
on and off (python profiles/dev/two_step_repro.py 64 128 [--single])."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2509_15744_b200 as W  # noqa: E402
from paper_2509_15744_b200 import engine  # noqa: E402

shape = tuple(int(a) for a in sys.argv[1:] if a.isdigit())
two = "--single" not in sys.argv
rng = np.random.default_rng(1)
dx = 1e-4
dt = 0.45 * dx / 6000.0 / np.sqrt(len(shape))
gamma = rng.uniform(0.3, 1.0, size=shape)
grid = W.build_grid(shape, dx)
mat = W.MaterialModel.rho_scaled(gamma, grid, rho0=2700.0, c0=6000.0)
src = W.SourceSpec(node=tuple(s // 3 for s in shape), amplitude=1e12, frequency=4e6, cycles=2)
sens = [tuple((s * (q + 1)) // 4 for s in shape) for q in range(3)]
n_steps = 20
measured = rng.normal(scale=1e-10, size=(1, len(sens), n_steps))
problem = W.FwiProblem(grid=grid, time=W.TimeConfig(n_steps, dt), material=mat, sources=[src],
                       sensors=W.SensorArray(nodes=sens), measured=measured)
ctx = engine.get_context(grid, np.float32)
ctx.set_two_step(two)
for what in ("fwd", "grad"):
    if what == "fwd":
        r = W.run_forward(mat, problem.time, [src], None, dtype=np.float32)
        print("fwd ok", float(np.abs(r.window.u_cur).max()), flush=True)
    else:
        r = W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=1e13, precision="single"))
        print("grad ok", r.cost, ctx.stats(), flush=True)
