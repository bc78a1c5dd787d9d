"""Short gradient_superposed run used for ncu captures of the fused step kernel.

    python profiles/profile_step.py [--grid 256] [--n-steps 32] [--precision single]
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2509_15744_b200 as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--n-steps", type=int, default=32)
    ap.add_argument("--precision", default="single")
    args = ap.parse_args()
    wl = bench.workload(args.grid, args.n_steps)
    problem, model = bench.build_problem(W, wl, synth_only=-1)
    problem.measured = np.zeros_like(problem.measured)
    cfg = W.SuperpositionConfig(k=wl["k"], precision=args.precision)
    res = W.gradient_superposed(problem, model, cfg)
    print("ok", res.cost, float(np.abs(res.gradient).max()))


if __name__ == "__main__":
    main()
