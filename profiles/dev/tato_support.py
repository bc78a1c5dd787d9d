"""Dev: TATO 192^3 forward sweep time with / without the objective support."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "profiles"))
import numpy as np  # noqa: E402

import configs  # noqa: E402
from paper_2509_15744_b200 import engine  # noqa: E402

N = 200
problem, mat = configs.tato((192, 192, 192), N)
ctx = engine.get_context(problem.grid, np.float32)
ctx.set_material(mat, problem.time.dt)
src = problem.source
amp = engine.source_amplitude_table([src], problem.time.dt, N)
sf = [problem.grid.flat_index(src.node)]
sup = np.flatnonzero(problem.objective_mask)
for label in ("support", "none", "support"):
    if label == "support":
        ctx.set_support(sup)
    else:
        ctx.clear_support()
    for rep in range(2):
        ctx.reset_window()
        ctx.zero_accumulator()
        ctx.synchronize()
        ctx.timer_mark(0)
        ctx.sweep_forward(N, sf, amp, accumulate=True, dt=problem.time.dt, scale=0.0)
        ctx.timer_mark(1)
    print(label, len(sup) if label == "support" else 0, round(ctx.timer_elapsed_ms(0, 1), 3), "ms",
          flush=True)
