"""Headline benchmark: superposed forward+adjoint sensitivity throughput.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]

Metric (BASELINE.json): Gcell-updates/s of gradient_superposed, 3D, fp32.
One bench "step" = one full gradient_superposed evaluation of the C2
workload: 3D rho-scaled FWI on a 256^3 grid, one source,
N = 1024 time steps, a 33x33 sensor plane, k = 1e13.  It performs
2*(N-1)*C cell-updates (forward sweep + superposed backward sweep).

* value  — device-resident: inputs already in HBM (SuperposedPlan.run()),
           timed with CUDA events on the library stream, max over ranks.
* e2e    — the public API call gradient_superposed(problem, material, cfg)
           with host (pinned) inputs: gamma/measured H2D and the gradient
           D2H inside the timed region.
* roofline — the dominant step kernel: SURVEY 8(d)'s 24 algorithmic bytes
           per fp32 cell-update x the cell-updates of one launch (a two-step
           pass does 2C) / its mean launch duration, from CUDA events around
           every 8th step launch of the timed region (bracketing every launch
           cost ~3.5% of it), against MEASURED_PEAKS.json; the bytes the
           two-step kernel really streams (10 fields per cell and pass) are
           reported beside it.
* cpu_baseline / --impl reference — the CPU oracle port (oracle/, a
           restatement of the reference's Numba loops pinned bit-exact to
           it) on the host cores, on a bounded sample of the same workload.

N > 1 (torchrun): shot-parallel weak scaling — each rank evaluates its own
shot of the same 256^3 model and the per-shot accumulators are summed with
one NCCL all-reduce per evaluation (shot-parallel mode).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gcell-updates/s fwd+adjoint sensitivity (3D, 1/2/4/8 B200); % HBM roofline"
UNIT = "Gcell-updates/s"
ITEMSIZE = {"single": 4, "double": 8}
PROFILE_EVERY = 8      # CUDA-event bracket on every 8th step launch of the timed region


def workload(n=256, n_steps=1024):
    return dict(name=f"fwi3d_{n}^3_superposed", shape=(n, n, n), dx=1e-4, c0=6000.0,
                rho0=2700.0, eps=1e-5, n_steps=n_steps, freq=5e6, cycles=2, amp=1e12,
                k=1e13, precision="single", sphere_r=20)


def build_problem(W, wl, n_sources=1, synth_only=None):
    shape = wl["shape"]
    n0, n1, n2 = shape
    dx, c0 = wl["dx"], wl["c0"]
    dt = 0.5 * dx / c0                       # Courant 0.5 < 1/sqrt(3)
    grid = W.build_grid(shape, dx)
    time_cfg = W.TimeConfig(wl["n_steps"], dt)
    model = W.MaterialModel.rho_scaled(np.ones(shape), grid, rho0=wl["rho0"], c0=c0,
                                       eps=wl["eps"])
    # sources on the axis-0 = 3 face (shot 0: face centre; one shot per GPU)
    offs = [(0, 0), (-40, -40), (40, 40), (-40, 40), (40, -40), (0, -60), (0, 60), (-60, 0)]
    sources = [W.SourceSpec(node=(3, n1 // 2 + offs[s % 8][0], n2 // 2 + offs[s % 8][1]),
                            amplitude=wl["amp"], frequency=wl["freq"], cycles=wl["cycles"])
               for s in range(n_sources)]
    lin = np.unique(np.round(np.linspace(2, n1 - 3, 33)).astype(int))
    sensors = W.SensorArray(nodes=[(n0 - 4, j, k) for j in lin for k in lin])
    truth = np.ones(shape)
    idx = np.ogrid[:n0, :n1, :n2]
    r2 = sum((idx[a] - shape[a] // 2) ** 2 for a in range(3))
    truth[r2 <= wl["sphere_r"] ** 2] = wl["eps"]
    problem = W.FwiProblem(grid=grid, time=time_cfg, material=model, sources=sources,
                           sensors=sensors)
    # measured traces of the truth (refine=1); a rank only needs its own shot's
    measured = np.zeros((n_sources, len(sensors), wl["n_steps"]))
    for s in range(n_sources):
        if synth_only is None or s == synth_only:
            sub = W.FwiProblem(grid=grid, time=time_cfg, material=model, sources=[sources[s]],
                               sensors=sensors)
            measured[s] = W.synthesize_measurements(model.with_gamma(truth), sub, refine=1)[0]
    problem.measured = measured
    return problem, model


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device=0):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.device), "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.th.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


def ncu_traffic(kernel_key):
    """dram bytes per launch of the fused step kernel from the committed ncu
    capture (profiles/ncu_step_kernel.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_step_kernel.json")) as fh:
            data = json.load(fh)
        return data.get(kernel_key, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def cpu_oracle_rate(wl, problem, model, n_sample, threads=None):
    """Oracle port (oracle/oracle.py + wave_oracle.c, OpenMP) on a bounded
    sample: the full 256^3 grid, the same shot and k, N = n_sample steps."""
    from oracle import oracle as O

    if threads:
        os.environ["OMP_NUM_THREADS"] = str(threads)
    c = problem.grid.n_nodes
    dt = problem.time.dt
    src = problem.sources[0]
    mat = O.Material("rho_scaled", np.asarray(model.gamma, dtype=np.float64), problem.grid.dx,
                     rho0=model.rho0, c0=model.c0)
    support = problem.sensors.flat_indices(problem.grid)
    shots = [(O.Source(src.node, src.amplitude, src.frequency, src.cycles),
              O.FwiShot(support, problem.measured[0][:, :n_sample], dt))]
    t0 = time.perf_counter()
    O.gradient_superposed(mat, dt, n_sample, shots, wl["k"], wl["precision"])
    el = time.perf_counter() - t0
    return 2 * (n_sample - 1) * c / el / 1e9, el, O.num_threads()


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def run_reference_arm(args):
    rank, world, _ = dist_setup()
    if rank != 0:
        return
    import paper_2509_15744_b200 as W

    wl = workload()
    # host-only: the measured traces are zeros (the misfit then uses r = u;
    # the CPU work per step is identical), so this arm never touches a GPU
    problem, model = build_problem(W, wl, synth_only=-1)
    n_sample = args.ref_sample_steps
    for _ in range(args.warmup):
        cpu_oracle_rate(wl, problem, model, min(n_sample, 4))
    rates, els = [], []
    threads = None
    for _ in range(args.steps):
        r, el, threads = cpu_oracle_rate(wl, problem, model, n_sample)
        rates.append(r)
        els.append(el)
    value = float(np.mean(rates))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(els)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": wl["name"], "grid": list(wl["shape"]),
                   "n_steps_sampled": n_sample, "shots": 1, "precision": "single",
                   "l2": "inputs larger than L2 (268 MB working set)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{wl['name']} grid, 1 shot, N={n_sample} steps "
                                   f"({2 * (n_sample - 1)} cell-update sweeps) per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_native(args):
    rank, world, local = dist_setup()
    import torch

    import paper_2509_15744_b200 as W
    from paper_2509_15744_b200 import gradients as G

    from paper_2509_15744_b200.distributed import ShotParallelGradient

    wl = workload(args.grid, args.n_steps)
    problem, model = build_problem(W, wl, n_sources=world, synth_only=rank)
    grid, n_steps = problem.grid, problem.time.n_steps
    C = grid.n_nodes
    cfg = W.SuperpositionConfig(k=wl["k"], precision=wl["precision"])
    updates = 2 * (n_steps - 1) * C          # per rank per evaluation (one shot)

    # ---------------- device-resident hot path ----------------------------
    if world > 1:
        plan = ShotParallelGradient(problem, model, cfg, rank, world).upload()
        ctx = plan.plan.ctx
    else:
        plan = G.SuperposedPlan(problem, model, cfg).upload()
        ctx = plan.ctx
    for _ in range(args.warmup):
        plan.run()
    barrier(world)
    ctx.synchronize()
    ctx.reset_stats()
    # per-launch CUDA events on a sample of the step launches (every 8th):
    # bracketing every launch cost ~3.5% of the timed region
    ctx.set_profiling(PROFILE_EVERY)
    with ClockSampler(local) as clocks:
        # cudaProfilerStart/Stop: `ncu --profile-from-start off` sees only
        # the timed region (profiles/capture_round.sh); no-ops otherwise
        torch.cuda.profiler.start()
        ctx.timer_mark(0)
        for _ in range(args.steps):
            plan.run()
        ctx.timer_mark(1)
        ms = ctx.timer_elapsed_ms(0, 1)
        torch.cuda.profiler.stop()
    ctx.set_profiling(False)
    stats = ctx.stats()
    barrier(world)
    ms = max_over_ranks(ms, world)
    ms_per_step = ms / args.steps
    value = world * updates / (ms_per_step * 1e-3) / 1e9

    # ---------------- roofline of the fused step kernels -------------------
    # 24 algorithmic bytes per fp32 cell-update (read u^n,
    # u^{n-1}, gamma, acc; write u^{n+1}, acc), also for temporal blocking.
    # A two-step pass (step2_kernel_tma) performs 2C cell-updates; it actually
    # streams 10 fields per cell (u^{n-1}, u^n, acc, coef, 3 face arrays in;
    # u^{n+1}, u^{n+2}, acc out) = "streamed_bytes_per_launch".  achieved =
    # algorithmic bytes of all step launches / their summed CUDA-event time.
    peaks, peak_kind = measured_peaks()
    item = ITEMSIZE[wl["precision"]]
    pairs = stats.get("pair_launches", 0)
    singles = stats["step_launches"] - pairs
    two = pairs >= singles
    # dominant kernel: mean duration of its sampled launches
    n_prof = stats["profiled_pair_n"] if two else stats["profiled_single_n"]
    ms_prof = stats["profiled_pair_ms"] if two else stats["profiled_single_ms"]
    k_ms = ms_prof / max(n_prof, 1)
    upd_per_launch = (2 if two else 1) * C
    achieved = 6 * item * upd_per_launch / (k_ms * 1e-3) / 1e9
    streamed = (10 if two else 6) * item * C / (k_ms * 1e-3) / 1e9
    peak = float(peaks["hbm_gbs"])
    kname = "step2_kernel" if two else "step_kernel"
    traffic = ncu_traffic(f"{kname}_{wl['precision']}_{args.grid}")

    # ---------------- end to end through the public API --------------------
    gamma_pinned = torch.empty(grid.shape, dtype=torch.float64, pin_memory=True).numpy()
    gamma_pinned[...] = model.gamma
    meas_pinned = torch.empty(problem.measured.shape, dtype=torch.float64,
                              pin_memory=True).numpy()
    meas_pinned[...] = problem.measured
    problem.measured = meas_pinned
    material = model.with_gamma(gamma_pinned)
    def api_call():
        if world == 1:
            return W.gradient_superposed(problem, material, cfg).gradient
        sp = ShotParallelGradient(problem, material, cfg, rank, world).upload()
        sp.run()
        return sp.download()

    import gc

    api_call()                                             # warm the API path
    api_call()
    gc.collect()
    gc.disable()                                           # no collector pauses in the timing
    barrier(world)
    t0 = time.perf_counter()
    per_call = []
    for _ in range(args.steps):
        tc = time.perf_counter()
        api_call()
        per_call.append(time.perf_counter() - tc)
    e2e_s = max_over_ranks((time.perf_counter() - t0) / args.steps, world)
    gc.enable()
    print(f"e2e per call (s): {[round(x, 4) for x in per_call]}", file=sys.stderr)
    e2e_value = world * updates / e2e_s / 1e9
    n_sup = len(problem.sensors)
    h2d = C * 8 + n_sup * n_steps * 8
    d2h = C * 4 + 8 + 2 * (n_steps + 2) * 8

    # ---------------- CPU oracle beside it (rank 0, N=1) ------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        r, el, threads = cpu_oracle_rate(wl, problem, model, args.cpu_sample_steps)
        cpu = {"value": r, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{wl['name']} grid, 1 shot, N={args.cpu_sample_steps} steps "
                         f"({2 * (args.cpu_sample_steps - 1)} sweeps), {el:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": wl["name"], "grid": list(wl["shape"]), "n_steps": n_steps,
                       "shots_per_gpu": 1, "precision": wl["precision"], "k": wl["k"],
                       "parallelism": "shot-parallel" if world > 1 else "single",
                       "cell_updates_per_step": world * updates,
                       "l2": "inputs larger than L2 (4 x 67 MB fields = 268 MB > 126 MB)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": ("wb::step2_kernel_tma (two fused steps per pass)" if two
                                    else "wb::step_kernel_tma4 (fused step)"),
                         "algorithmic_bytes_per_cell_update": 6 * item,
                         "algorithmic_bytes_per_launch": 6 * item * C * (2 if two else 1),
                         "streamed_bytes_per_launch": (10 if two else 6) * item * C,
                         "streamed_gbs": streamed, "streamed_frac": streamed / peak,
                         "pair_launches": pairs, "single_launches": singles,
                         "mean_launch_ms": k_ms, "profiled_launches": n_prof,
                         "profiled_every": PROFILE_EVERY,
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3},
            "gpu_launches": int(stats["launches"]),
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["native", "reference"], default="native")
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--n-steps", type=int, default=1024)
    # CPU samples: ~12 s for cpu_baseline; ~5 s per step of the reference arm
    # (so its default 10 steps finish in about a minute)
    ap.add_argument("--cpu-sample-steps", type=int, default=160)
    ap.add_argument("--ref-sample-steps", type=int, default=100)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_native(args)


if __name__ == "__main__":
    main()
