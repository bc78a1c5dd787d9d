"""One C1 fp32 superposed gradient after warm-up, bracketed by
cudaProfilerStart/Stop (dev: `ncu --profile-from-start off` target)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "profiles")]

import torch  # noqa: E402

import configs  # noqa: E402
import paper_2509_15744_b200 as W  # noqa: E402
from paper_2509_15744_b200 import gradients as G  # noqa: E402

torch.cuda.init()
problem, mat = configs.fwi((256, 256), 3200)
plan = G.SuperposedPlan(problem, mat, W.SuperpositionConfig(k=1e13, precision="single")).upload()
for _ in range(3):
    plan.run()
plan.ctx.synchronize()
torch.cuda.profiler.start()
plan.run()
plan.ctx.synchronize()
torch.cuda.profiler.stop()
