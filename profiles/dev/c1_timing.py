"""Dev: SURVEY C1 — 2D FWI 256^2, N = 3200 (fwi_desk-like), fp32 and fp64:
device time of one superposed gradient (launch-bound regime)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2509_15744_b200 as W  # noqa: E402
from paper_2509_15744_b200 import gradients as G  # noqa: E402

n, N = 256, 3200
dx = 0.02 / 255
dt = 7.5e-9
grid = W.build_grid((n, n), dx)
mat = W.MaterialModel.rho_scaled(np.ones((n, n)), grid, rho0=2700.0, c0=6000.0)
src = W.SourceSpec(node=(128, 3), amplitude=1e12, frequency=1e6, cycles=2)
sens = [(i, n - 4) for i in range(3, n - 3, 4)]
meas = np.random.default_rng(0).normal(scale=1e-9, size=(1, len(sens), N))
problem = W.FwiProblem(grid=grid, time=W.TimeConfig(N, dt), material=mat, sources=[src],
                       sensors=W.SensorArray(nodes=sens), measured=meas)
for prec in ("single", "double"):
    plan = G.SuperposedPlan(problem, mat, W.SuperpositionConfig(k=1e13, precision=prec)).upload()
    plan.run()
    ctx = plan.ctx
    ctx.synchronize()
    ctx.reset_stats()
    ctx.timer_mark(0)
    for _ in range(5):
        plan.run()
    ctx.timer_mark(1)
    ms = ctx.timer_elapsed_ms(0, 1) / 5
    upd = 2 * (N - 1) * n * n
    st = ctx.stats()
    print(f"C1 {prec}: {ms:.2f} ms/gradient, {upd / ms / 1e6:.1f} Gcell-upd/s, "
          f"{st['step_launches'] // 5} step launches ({st['pair_launches'] // 5} two-step)",
          flush=True)
