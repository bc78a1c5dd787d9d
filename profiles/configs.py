"""Throughput of the hot path on the BASELINE / SURVEY §8(d) configurations
(one B200, device-resident; not bench lines — the headline is bench.py's C2).

    python profiles/configs.py [--out profiles/r1/configs.json]

C1  2D FWI 256², N = 3200 (launch/latency-bound; SURVEY: report as such)
C2  3D FWI 256³, N = 1024 (the bench workload)
C3  TATO 512² (N = 2000) and 192³ (N = 600), acoustic flavour
C4  3D FWI 1024³, 4 shots, N = 128 (timed sample of the 2048-step run)
Each line: Gcell-updates/s of one superposed gradient evaluation
(2 (N-1) C S cell-updates / CUDA-event time), fp32 and fp64.
"""

import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2509_15744_b200 as W  # noqa: E402
from paper_2509_15744_b200 import gradients as G  # noqa: E402


def fwi(shape, n_steps, n_sources=1):
    n = shape[0]
    dx = 1e-4 if len(shape) == 3 else 0.02 / 255
    c0 = 6000.0
    dt = 0.5 * dx / c0 if len(shape) == 3 else 7.5e-9
    grid = W.build_grid(shape, dx)
    mat = W.MaterialModel.rho_scaled(np.ones(shape), grid, rho0=2700.0, c0=c0)
    if len(shape) == 3:
        srcs = [W.SourceSpec(node=(3, n // 3 + 17 * s, n // 2), amplitude=1e12, frequency=5e6,
                             cycles=2) for s in range(n_sources)]
        sens = [(n - 4, j, k) for j in range(n // 8, n - n // 8, max(n // 32, 1))
                for k in range(n // 8, n - n // 8, max(n // 32, 1))]
    else:
        srcs = [W.SourceSpec(node=(n // 2, 3), amplitude=1e12, frequency=1e6, cycles=2)]
        sens = [(i, n - 4) for i in range(3, n - 3, 4)]
    meas = np.random.default_rng(0).normal(scale=1e-9, size=(len(srcs), len(sens), n_steps))
    return W.FwiProblem(grid=grid, time=W.TimeConfig(n_steps, dt), material=mat, sources=srcs,
                        sensors=W.SensorArray(nodes=sens), measured=meas), mat


def tato(shape, n_steps):
    rho1, kappa1, rho2, kappa2 = 1.204, 1.419e5, 2643.0, 6.87e8
    dx = 0.01
    dt = 0.5 * dx / math.sqrt(kappa2 / rho2)
    grid = W.build_grid(shape, dx)
    design = np.zeros(shape, dtype=bool)
    objective = np.zeros(shape, dtype=bool)
    sl = tuple(slice(s // 3, 2 * s // 3) for s in shape)
    design[sl] = True
    ob = tuple(slice(3 * s // 4, 3 * s // 4 + max(s // 16, 2)) for s in shape)
    objective[ob] = True
    node = tuple([s // 8 for s in shape])
    problem = W.TatoProblem(grid=grid, time=W.TimeConfig(n_steps, dt),
                            source=W.SourceSpec(node=node, amplitude=1.0, frequency=650.0,
                                                cycles=2),
                            design_mask=design, objective_mask=objective, rho1=rho1,
                            kappa1=kappa1, rho2=rho2, kappa2=kappa2, r_f=1.5, eta=0.5,
                            mode="suppress")
    g = np.where(design, np.random.default_rng(1).uniform(size=shape), 0.0)
    return problem, problem.material(g)


def rate(problem, mat, prec, reps=3):
    plan = G.SuperposedPlan(problem, mat, W.SuperpositionConfig(k=1e13, precision=prec)).upload()
    for _ in range(3):   # a repeated evaluation captures its sweep graphs
        plan.run()
    ctx = plan.ctx
    ctx.synchronize()
    ctx.reset_stats()
    ctx.timer_mark(0)
    for _ in range(reps):
        plan.run()
    ctx.timer_mark(1)
    ms = ctx.timer_elapsed_ms(0, 1) / reps
    n_shots = len(list(problem.shots()))
    upd = 2 * (problem.time.n_steps - 1) * problem.grid.n_nodes * n_shots
    st = ctx.stats()
    return {"ms_per_gradient": ms, "gcell_upd_s": upd / ms / 1e6,
            "two_step_passes": st["pair_launches"] // reps,
            "step_launches": st["step_launches"] // reps}


def rate_reference(problem, mat, prec, reps=2):
    """gradient_reference (gradients.py:329-391, the C1 comparator): forward
    with the full history on the device, fused adjoint + mixed-kernel steps."""
    import time

    W.gradient_reference(problem, mat, precision=prec)          # warm
    t0 = time.perf_counter()
    for _ in range(reps):
        W.gradient_reference(problem, mat, precision=prec)
    ms = (time.perf_counter() - t0) / reps * 1e3
    n_shots = len(list(problem.shots()))
    upd = 2 * (problem.time.n_steps - 1) * problem.grid.n_nodes * n_shots
    return {"ms_per_gradient": ms, "gcell_upd_s": upd / ms / 1e6, "engine": "reference",
            "timing": "host wall clock around gradient_reference (incl. the gradient D2H)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--only", default=None, help="comma-separated config prefixes, e.g. C1,C3")
    args = ap.parse_args()
    rows = []
    cases = [
        ("C1 2D FWI 256^2, N=3200", lambda: fwi((256, 256), 3200)),
        ("C2 3D FWI 256^3, N=1024", lambda: fwi((256, 256, 256), 1024)),
        ("C3 TATO 2D 512^2, N=2000", lambda: tato((512, 512), 2000)),
        ("C3 TATO 3D 192^3, N=600", lambda: tato((192, 192, 192), 600)),
        ("C4 3D FWI 1024^3, 4 shots, N=128 sample", lambda: fwi((1024, 1024, 1024), 128, 4)),
    ]
    if args.only:
        keep = tuple(args.only.split(","))
        cases = [c for c in cases if c[0].startswith(keep)]
    for name, make in cases:
        problem, mat = make()
        for prec in ("single", "double"):
            if "1024" in name and prec == "double":
                reps = 1
            else:
                reps = 3
            r = rate(problem, mat, prec, reps)
            r.update({"config": name, "precision": prec})
            rows.append(r)
            print(json.dumps(r), flush=True)
            if name.startswith("C1"):
                r = rate_reference(problem, mat, prec)
                r.update({"config": name + " gradient_reference", "precision": prec})
                rows.append(r)
                print(json.dumps(r), flush=True)
        W.release_contexts() if hasattr(W, "release_contexts") else None
    if args.out:
        with open(args.out, "w") as fh:
            json.dump({"peaks": bench.measured_peaks()[0], "rows": rows}, fh, indent=1)


if __name__ == "__main__":
    main()
