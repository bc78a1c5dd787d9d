"""Cost of the slab decomposition on ONE GPU (BASELINE C5 mechanics).

    python profiles/dev/slab_timing.py [--grid 512] [--n-steps 64] [--parts 2]

Times one superposed gradient (fp32, rho-scaled 3D FWI, one shot) as
  mono2   one context, two-step passes (the bench path)
  mono1   one context, single-step kernel only (what a slab runs)
  slabsO  `parts` slab contexts on this GPU, loopback halo, split
          boundary/interior steps (the overlapped NCCL schedule)
  slabsW  the same with whole steps then the exchange
  slabsP  peer ghost stores + device flags (no exchange): whole sweeps with
          two-step passes (interleaved pass by pass: same device)
Host wall clock around a synchronised run (slabs use one stream each).
On one GPU the slabs run one after the other, so slabsO/slabsW vs mono1 is
the price of the decomposition itself (split launches, ghost planes, the
per-step host loop), not a scaling number.
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
from paper_2509_15744_b200.distributed import SlabGradient, slab_ranges  # noqa: E402


def timed(run, sync, reps):
    run()
    sync()
    t0 = time.perf_counter()
    for _ in range(reps):
        run()
    sync()
    return (time.perf_counter() - t0) / reps * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=512)
    ap.add_argument("--n-steps", type=int, default=64)
    ap.add_argument("--parts", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    n = args.grid
    problem, mat = configs.fwi((n, n, n), args.n_steps)
    cfg = W.SuperpositionConfig(k=1e13, precision="single")
    upd = 2 * (args.n_steps - 1) * problem.grid.n_nodes
    rows = {}
    for name, two in (("mono2", 1), ("mono1", 0)):
        plan = G.SuperposedPlan(problem, mat, cfg).upload()
        plan.ctx.set_two_step(two)
        ms = timed(plan.run, plan.ctx.synchronize, args.reps)
        rows[name] = ms
        plan.ctx.set_two_step(1)        # pooled context: restore the default
    for name, overlap, halo in (("slabsO", True, "loopback"), ("slabsW", False, "loopback"),
                                ("slabsP", True, "peer")):
        sg = SlabGradient(problem, mat, cfg, slab_ranges(n, args.parts), overlap=overlap,
                          halo=halo).upload()

        def sync(sg=sg):
            for c in sg.ctxs:
                c.synchronize()

        rows[name] = timed(sg.run, sync, args.reps)
        sg.close()
    out = {"grid": n, "n_steps": args.n_steps, "parts": args.parts,
           "ms": {k: round(v, 2) for k, v in rows.items()},
           "gcell_upd_s": {k: round(upd / v / 1e6, 1) for k, v in rows.items()},
           "slab_overhead_vs_mono1": {k: round(rows[k] / rows["mono1"] - 1, 3)
                                      for k in ("slabsO", "slabsW", "slabsP")}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
