"""fp64 superposed-gradient rate at one grid (dev A/B of single-step knobs).

    WB_T1_CHUNK=... python profiles/dev/f64_rate.py [--grid 256] [--n-steps 256]
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "profiles"))

import configs  # noqa: E402
import paper_2509_15744_b200 as W  # noqa: E402
from paper_2509_15744_b200 import gradients as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--grid", type=int, default=256)
ap.add_argument("--n-steps", type=int, default=256)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--two-step", type=int, default=1, help="0: single steps, 1: two-step passes")
args = ap.parse_args()
n = args.grid
problem, mat = configs.fwi((n, n, n), args.n_steps)
plan = G.SuperposedPlan(problem, mat, W.SuperpositionConfig(k=1e13, precision="double")).upload()
plan.ctx.set_two_step(args.two_step)
plan.run()
plan.ctx.synchronize()
t0 = time.perf_counter()
for _ in range(args.reps):
    plan.run()
plan.ctx.synchronize()
ms = (time.perf_counter() - t0) / args.reps * 1e3
upd = 2 * (args.n_steps - 1) * problem.grid.n_nodes
print(json.dumps({"grid": n, "n_steps": args.n_steps, "chunk": os.environ.get("WB_T1_CHUNK", "model"),
                  "two_step": args.two_step,
                  "ms": round(ms, 2), "gcell_upd_s": round(upd / ms / 1e6, 1)}))
