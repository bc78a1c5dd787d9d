"""Time the phases of one public-API gradient_superposed call (dev tool)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2509_15744_b200 as W  # noqa: E402
from paper_2509_15744_b200 import gradients as G  # noqa: E402


def main():
    wl = bench.workload(256, int(sys.argv[1]) if len(sys.argv) > 1 else 1024)
    problem, model = bench.build_problem(W, wl)
    cfg = W.SuperpositionConfig(k=wl["k"], precision="single")
    if "--pinned" in sys.argv:
        import torch

        gp = torch.empty(problem.grid.shape, dtype=torch.float64, pin_memory=True).numpy()
        gp[...] = model.gamma
        model = model.with_gamma(gp)
        mp = torch.empty(problem.measured.shape, dtype=torch.float64, pin_memory=True).numpy()
        mp[...] = problem.measured
        problem.measured = mp
    for rep in range(int(os.environ.get("REPS", "8"))):
        t0 = time.perf_counter()
        plan = G.SuperposedPlan(problem, model, cfg)
        t1 = time.perf_counter()
        plan.upload()
        t2 = time.perf_counter()
        plan.run()
        t3 = time.perf_counter()
        plan.download()
        t4 = time.perf_counter()
        print(f"rep {rep}: init {1e3*(t1-t0):.1f} upload {1e3*(t2-t1):.1f} run {1e3*(t3-t2):.1f} "
              f"download {1e3*(t4-t3):.1f} ms  fast_div={plan.ctx.fast_div_active()}", flush=True)
    ctx = plan.ctx
    for phase in range(2):
        ctx.reset_stats()
        ctx.set_profiling(True)
        t0 = time.perf_counter()
        plan.run()
        t1 = time.perf_counter()
        ctx.set_profiling(False)
        st = ctx.stats()
        print(f"run {1e3*(t1-t0):.1f} ms, step kernels {st['step_kernel_ms']:.1f} ms over "
              f"{st['step_launches']} launches", flush=True)


if __name__ == "__main__":
    main()
