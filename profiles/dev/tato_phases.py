"""Dev: forward / misfit / backward sweep times of one superposed gradient
(C3 TATO 192^3 N = 600 vs the FWI 192^3 bench-like problem)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "profiles")]

import configs  # noqa: E402
import paper_2509_15744_b200 as W  # noqa: E402
from paper_2509_15744_b200 import gradients as G  # noqa: E402

for name, (problem, mat) in (("tato192", configs.tato((192,) * 3, 600)),
                             ("fwi192", configs.fwi((192,) * 3, 600))):
    plan = G.SuperposedPlan(problem, mat, W.SuperpositionConfig(k=1e13, precision="single")).upload()
    for _ in range(3):
        plan.run()
    ctx = plan.ctx
    n_steps, dt = problem.time.n_steps, problem.time.dt
    shot, src_flat, amp, scale, (kind, c, adj_coef, meas) = plan.shots[0]
    for rep in range(2):
        ctx.zero_accumulator()
        ctx.reset_window()
        ctx.synchronize()
        ctx.timer_mark(0)
        ctx.sweep_forward(n_steps, [src_flat], amp, accumulate=True, dt=dt, scale=scale)
        ctx.timer_mark(1)
        ctx.shot_misfit(n_steps, kind, None, c, adj_coef, True, 1e13)
        ctx.timer_mark(2)
        ctx.sweep_backward(n_steps, src_flat, amp[0], inject=True, accumulate=True, dt=dt)
        ctx.timer_mark(3)
        ctx.synchronize()
        print(name, "n_sup", ctx.n_sup, "fwd", round(ctx.timer_elapsed_ms(0, 1), 2), "misfit",
              round(ctx.timer_elapsed_ms(1, 2), 2), "bwd", round(ctx.timer_elapsed_ms(2, 3), 2), "ms",
              flush=True)
