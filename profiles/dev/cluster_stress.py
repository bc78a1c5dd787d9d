"""Stress the register-resident cluster sweep for races: repeated superposed
gradients on several 2D shapes (fp32 / fp64) must be bit-identical to the
step-kernel path every time (dev: python profiles/dev/cluster_stress.py [reps])."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "profiles")]

import configs  # noqa: E402
import paper_2509_15744_b200 as W  # noqa: E402
from paper_2509_15744_b200 import engine  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
bad = 0
for shape, n in (((256, 256), 800), ((97, 97), 300), ((200, 200), 300), ((33, 33), 300)):
    problem, mat = configs.fwi(shape, n)
    for prec in ("single", "double"):
        cfg = W.SuperpositionConfig(k=1e13, precision=prec)
        ctx = engine.get_context(problem.grid, W.precision_dtype(prec))
        ctx.set_cluster(False)
        ref = W.gradient_superposed(problem, mat, cfg)
        ctx.set_cluster(None)
        diffs = 0
        for _ in range(reps):
            r = W.gradient_superposed(problem, mat, cfg)
            diffs += (r.gradient.tobytes() != ref.gradient.tobytes()) or (r.cost != ref.cost)
        bad += diffs
        print(shape, prec, "mismatches", diffs, "of", reps, flush=True)
print("TOTAL mismatches", bad)
