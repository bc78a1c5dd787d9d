"""Phases of the material upload at 256^3 (dev): raw pinned H2D rate of the
fp64 gamma, wo_set_material, and the rest of SuperposedPlan.upload."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_15744_b200 as W  # noqa: E402
from paper_2509_15744_b200 import engine, gradients as G  # noqa: E402

wl = bench.workload(256, 64)
problem, model = bench.build_problem(W, wl)
gp = torch.empty(problem.grid.shape, dtype=torch.float64, pin_memory=True)
gp.numpy()[...] = model.gamma
dev = torch.empty_like(gp, device="cuda")
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev.copy_(gp, non_blocking=True)
    torch.cuda.synchronize()
    print(f"torch pinned H2D {gp.numel() * 8 / 1e6:.0f} MB: {1e3 * (time.perf_counter() - t0):.2f} ms")
mat = model.with_gamma(gp.numpy())
ctx = engine.get_context(problem.grid, "float32")
for _ in range(4):
    t0 = time.perf_counter()
    ctx.set_material(mat, problem.time.dt)
    t1 = time.perf_counter()
    plan = G.SuperposedPlan(problem, mat, W.SuperpositionConfig(k=wl["k"], precision="single"))
    plan.upload()
    t2 = time.perf_counter()
    print(f"set_material {1e3 * (t1 - t0):.2f} ms, plan.upload {1e3 * (t2 - t1):.2f} ms "
          f"fast_div={ctx.fast_div_active()}")
