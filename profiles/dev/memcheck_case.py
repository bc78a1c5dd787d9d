"""Small superposed gradients through every step-kernel family (dev):
two-step TMA (fp32 3D), single-step TMA (fp64 3D), 2D, and slabs with peer
ghost stores.  Exits non-zero unless two-step == single-step and slabs ==
one context, bitwise.  Written as a compute-sanitizer case; the sanitizer is
closed on this GPU pool, so it runs plain (PDL build: all equal)."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "profiles"))

import configs  # noqa: E402
import paper_2509_15744_b200 as W  # noqa: E402
from paper_2509_15744_b200 import gradients as G  # noqa: E402
from paper_2509_15744_b200.distributed import gradient_superposed_slabs  # noqa: E402

ok = True
for shape, prec in (((48, 48, 128), "single"), ((40, 40, 64), "double"), ((96, 128), "single")):
    problem, mat = configs.fwi(shape, 40)
    cfg = W.SuperpositionConfig(k=1e13, precision=prec)
    res = []
    for two in (1, 0):
        plan = G.SuperposedPlan(problem, mat, cfg).upload()
        plan.ctx.set_two_step(two)
        plan.run()
        res.append(plan.download().copy())
        plan.ctx.set_two_step(1)
    same = res[0].view(np.uint8).tobytes() == res[1].view(np.uint8).tobytes()
    print(shape, prec, "two-step == single-step:", same, flush=True)
    ok &= same
problem, mat = configs.fwi((48, 48, 128), 40)
cfg = W.SuperpositionConfig(k=1e13, precision="single")
g1 = W.gradient_superposed(problem, mat, cfg).gradient
gs = gradient_superposed_slabs(problem, mat, cfg, 3, halo="peer").gradient
same = g1.view(np.uint8).tobytes() == gs.view(np.uint8).tobytes()
print("slabs (peer stores) == one context:", same, flush=True)
ok &= same
sys.exit(0 if ok else 1)
