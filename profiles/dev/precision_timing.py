"""Dev: device time of one gradient_superposed (256^3, N steps) per precision,
with the two-step pass on and off.  python profiles/dev/precision_timing.py [N]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2509_15744_b200 as W  # noqa: E402
from paper_2509_15744_b200 import gradients as G  # noqa: E402

n_steps = int(sys.argv[1]) if len(sys.argv) > 1 else 128
wl = bench.workload(256, n_steps)
problem, model = bench.build_problem(W, wl, synth_only=-1)
for prec in ("single", "double"):
    for two in (True, False):
        plan = G.SuperposedPlan(problem, model, W.SuperpositionConfig(k=wl["k"], precision=prec))
        plan.upload()
        plan.ctx.set_two_step(two)
        plan.run()
        plan.ctx.synchronize()
        plan.ctx.timer_mark(0)
        for _ in range(3):
            plan.run()
        plan.ctx.timer_mark(1)
        ms = plan.ctx.timer_elapsed_ms(0, 1) / 3
        upd = 2 * (n_steps - 1) * problem.grid.n_nodes
        print(f"{prec:6s} two_step={two!s:5s} {ms:8.2f} ms  {upd / ms / 1e6:7.1f} Gcell-upd/s",
              flush=True)
        plan.ctx.set_two_step(True)
