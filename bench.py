"""Headline benchmark: superposed forward+adjoint sensitivity throughput.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]
                    [--workload auto|c2|c5] [--scaling weak|strong] [--halo ipc|nccl]

Metric (BASELINE.json): Gcell-updates/s of gradient_superposed, 3D, fp32.

N = 1 (default): one bench "step" = one full gradient_superposed evaluation
of the C2 workload: 3D rho-scaled FWI on a 256^3 grid, one
source, N = 1024 time steps, a 33x33 sensor plane, k = 1e13.  It performs
2*(N-1)*C cell-updates (forward sweep + superposed backward sweep).

* value  — device-resident: inputs already in HBM (SuperposedPlan.run()),
           timed with CUDA events on the library stream, max over ranks;
           the timed evaluations run exactly as a user's.
* e2e    — the public API call gradient_superposed(problem, material, cfg)
           with host (pinned) inputs: gamma/measured H2D and the gradient
           D2H inside the timed region.
* roofline — the dominant step kernel (step2_kernel_tma, two time steps per
           pass): its time per step = ms_per_step x its share of the step's
           GPU time in the committed ncu launch list of this command
           (profiles/launch_share.json); achieved = SURVEY 8(d)'s 24 B per
           fp32 cell-update x the 2C cell-updates of one launch / its launch
           time; traffic / physical_frac from the committed ncu capture
           (profiles/ncu_step_kernel.json); peak = MEASURED_PEAKS.json.
* cpu_baseline / --impl reference — the reference ITSELF (baseline/_ref:
           the unmodified waveopt package, Python + Numba) on the host cores,
           one process and one per core, on a bounded sample of the same
           workload; the pinned C/OpenMP oracle port (oracle/) is reported
           beside it and replaces it when baseline/_ref is absent.

N > 1 (torchrun) or --workload c5: SURVEY C5 — one slab of 256 x 2048^2
cells per GPU (weak scaling; --scaling strong: global 2048^3), N = 200
steps, peer ghost stores through CUDA IPC (SlabGradient.for_rank, halo
"ipc"; --halo nccl: send/recv exchanges), two-step passes on the slabs.
--workload c2 with N > 1: shot-parallel (one 256^3 shot per GPU, one NCCL
all-reduce of the accumulator per evaluation).
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
PROFILE_EVERY = 8      # diagnostic: CUDA events around every 8th launch of one extra evaluation


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


NCU_TRAFFIC_SRC = "profiles/ncu_step_kernel.json"


def ncu_traffic(kernel_key):
    """dram bytes per launch of the fused step kernel from the committed ncu
    capture (profiles/ncu_step_kernel.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_step_kernel.json")) as fh:
            data = json.load(fh)
        return data.get(kernel_key, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def launch_share(kernel, workload=None):
    """Share of the bench step's GPU time taken by `kernel` in the committed
    ncu launch list of this bench command (profiles/launch_share[_c5].json,
    written by profiles/launch_shares.py); (1.0, "assumed") without one."""
    name = "launch_share.json" if workload is None else f"launch_share_{workload}.json"
    try:
        with open(os.path.join(ROOT, "profiles", name)) as fh:
            data = json.load(fh)
        top = max(data["kernels"].items(), key=lambda kv: kv[1]["share"])
        if kernel in top[0]:   # the list was taken on the same engine
            return float(top[1]["share"]), data.get("source", "profiles/launch_share.json")
        return 1.0, f"assumed 1.0 (the committed {name} is of another engine)"
    except (OSError, ValueError, KeyError):
        pass
    return 1.0, "assumed 1.0 (no committed launch list)"


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


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def load_reference_package():
    """The UNMODIFIED reference package (waveopt: Python + Numba), installed
    under baseline/_ref with `pip install --target` (travels to
    the GPU box with the repo snapshot).  None when absent or not importable
    (then the CPU legs fall back to the pinned C/OpenMP oracle port)."""
    if not os.path.isdir(os.path.join(REF_DIR, "waveopt")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_bench_ref")
    os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
    sys.dont_write_bytecode = True
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import waveopt
    except Exception as e:   # e.g. numba missing on the host
        print(f"reference package not importable: {e}", file=sys.stderr)
        return None
    return waveopt


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


class ReferenceCPU:
    """The reference's own gradient_superposed (gradients.py:284-326, Numba
    kernels, single-threaded per process — kernels.py:1-6) on the host cores,
    BASELINE.md §2: one process, and `cores` concurrent processes with one
    shot each (aggregate rate).  Same workload as the GPU arm (grid, source,
    sensors, sphere-void truth, k, fp32) on a bounded sample of N steps;
    measured traces synthesized by the reference itself (refine = 1) for that
    N.  Numba compile is excluded (warm-up on a small grid); processes are
    forked from the prepared parent, so the problem is shared copy-on-write."""

    def __init__(self, R, wl, n_sample):
        self.R, self.wl, self.n = R, dict(wl), int(n_sample)
        self.wl["n_steps"] = self.n
        self.problem, self.model = build_problem(R, self.wl)
        self.cfg = R.SuperpositionConfig(k=self.wl["k"], precision=self.wl["precision"])
        small = workload(16, 4)
        small["precision"] = self.wl["precision"]
        p, m = build_problem(R, small)
        R.gradient_superposed(p, m, self.cfg)          # JIT warm-up
        self.updates = 2 * (self.n - 1) * self.problem.grid.n_nodes

    def one(self):
        t0 = time.perf_counter()
        self.R.gradient_superposed(self.problem, self.model, self.cfg)
        return time.perf_counter() - t0

    def concurrent(self, procs):
        """Wall time of `procs` forked processes each evaluating the gradient."""
        import multiprocessing as mp

        ctx = mp.get_context("fork")
        t0 = time.perf_counter()
        ps = [ctx.Process(target=self.one) for _ in range(procs)]
        for p in ps:
            p.start()
        for p in ps:
            p.join()
        el = time.perf_counter() - t0
        if any(p.exitcode != 0 for p in ps):
            raise RuntimeError("a reference CPU process failed")
        return el

    def describe(self, procs):
        return (f"{self.wl['name']} grid, 1 shot per process, N={self.n} steps "
                f"({2 * (self.n - 1)} cell-update sweeps), fp32 ({self.wl['precision']}); "
                f"{procs} concurrent processes; CPU {cpu_model()}")


# WB_BENCH_SHARED_GPU=1: every rank on GPU 0 with a gloo process group — a
# functional dry run of the multi-GPU code path on a one-GPU box (the ranks
# share the GPU, so the numbers are not a scaling measurement)
SHARED_GPU = os.environ.get("WB_BENCH_SHARED_GPU", "0") == "1"


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if SHARED_GPU:
        local = 0
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        if SHARED_GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cpu" if SHARED_GPU else "cuda")
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
    wl = workload()
    R = load_reference_package()
    if R is None:
        return run_port_arm(args, wl)
    n_sample = args.ref_sample_steps
    ref = ReferenceCPU(R, wl, n_sample)
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    procs = host_cores()
    one_s = ref.one()                                  # 1 process (1 core)
    for _ in range(args.warmup):
        ref.concurrent(procs)
    els = [ref.concurrent(procs) for _ in range(args.steps)]
    el = float(np.mean(els))
    value = procs * ref.updates / el / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": wl["name"], "grid": list(wl["shape"]),
                   "n_steps_sampled": n_sample, "shots": procs, "precision": "single",
                   "l2": "inputs larger than L2 (268 MB working set per process)",
                   "note": ("per-cell-update rate of the reference on the 256^3 grid (the "
                            "C5 slabs need >= 43 GB per CPU process: extrapolated, SURVEY "
                            "8(d))" if world_env > 1 else "same grid as the GPU arm")},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "reference",
                         "sample": ref.describe(procs),
                         "value_1process": ref.updates / one_s / 1e9,
                         "package": "baseline/_ref waveopt 0.1.0 (unmodified reference)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_port_arm(args, wl):
    """Fallback CPU arm: the pinned C/OpenMP oracle port (oracle/)."""
    import paper_2509_15744_b200 as W

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
                                   f"({2 * (n_sample - 1)} cell-update sweeps) per step; "
                                   f"CPU {cpu_model()}"},
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
    # the timed region runs exactly as a user's evaluation (no per-launch
    # events: they break the programmatic-dependent-launch overlap)
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
    stats = ctx.stats()
    # diagnostic only (not the roofline): CUDA events around every 8th step
    # launch of one more evaluation
    ctx.reset_stats()
    ctx.set_profiling(PROFILE_EVERY)
    plan.run()
    ctx.set_profiling(False)
    pstats = ctx.stats()
    barrier(world)
    ms = max_over_ranks(ms, world)
    ms_per_step = ms / args.steps
    value = world * updates / (ms_per_step * 1e-3) / 1e9

    # ---------------- roofline of the fused step kernels -------------------
    # 24 algorithmic bytes per fp32 cell-update (read u^n,
    # u^{n-1}, gamma, acc; write u^{n+1}, acc), also for temporal blocking.
    # A two-step pass (step2_kernel_tma) performs 2C cell-updates; it actually
    # streams 10 fields per cell (u^{n-1}, u^n, acc, coef, 3 face arrays in;
    # u^{n+1}, u^{n+2}, acc out) = "streamed_bytes_per_launch".
    # The dominant kernel's time per step = ms_per_step (CUDA events around
    # the timed region) x its share of the step's GPU time in the committed
    # ncu launch list of this bench command (profiles/launch_share.json);
    # achieved = its algorithmic bytes per launch / (that time / launches).
    peaks, peak_kind = measured_peaks()
    item = ITEMSIZE[wl["precision"]]
    pairs = stats.get("pair_launches", 0)
    singles = stats["step_launches"] - pairs
    two = pairs >= singles
    kname = "step2_kernel" if two else "step_kernel"
    share, share_src = launch_share("step2_kernel_tma" if two else "step_kernel_tma4")
    n_dom = (pairs if two else singles) / args.steps          # launches per step
    k_ms = ms_per_step * share / max(n_dom, 1)
    upd_per_launch = (2 if two else 1) * C
    achieved = 6 * item * upd_per_launch / (k_ms * 1e-3) / 1e9
    streamed = (10 if two else 6) * item * C / (k_ms * 1e-3) / 1e9
    peak = float(peaks["hbm_gbs"])
    traffic = ncu_traffic(f"{kname}_{wl['precision']}_{args.grid}")
    n_ev = pstats["profiled_pair_n"] if two else pstats["profiled_single_n"]
    ms_ev = pstats["profiled_pair_ms"] if two else pstats["profiled_single_ms"]
    ev_ms = ms_ev / max(n_ev, 1)
    # physical DRAM rate of the whole step: ncu dram bytes of the dominant
    # kernel per launch x its launches per step / ms_per_step
    physical = traffic * n_dom / (ms_per_step * 1e-3) / 1e9 if traffic else None

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
    # the same call from plain pageable numpy arrays (the usual waveopt
    # caller): two evaluations, reported beside the pinned e2e
    pageable = None
    if world == 1:
        problem.measured = np.array(meas_pinned)
        mat_pg = model.with_gamma(np.array(gamma_pinned))
        W.gradient_superposed(problem, mat_pg, cfg)
        t0 = time.perf_counter()
        for _ in range(2):
            W.gradient_superposed(problem, mat_pg, cfg)
        pageable = updates / ((time.perf_counter() - t0) / 2) / 1e9
        problem.measured = meas_pinned
    n_sup = len(problem.sensors)
    h2d = C * 8 + n_sup * n_steps * 8
    d2h = C * 4 + 8 + 2 * (n_steps + 2) * 8

    # ---------------- CPU oracle beside it (rank 0, N=1) ------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        n_cpu = args.cpu_sample_steps
        r, el, threads = cpu_oracle_rate(wl, problem, model, n_cpu)
        port = {"value": r, "cores": threads, "kind": "port",
                "sample": f"C/OpenMP oracle port, same grid / shot / k, N={n_cpu}, {el:.1f} s"}
        R = load_reference_package()
        if R is not None:   # the reference itself (Numba), BASELINE.md §2
            ref = ReferenceCPU(R, wl, n_cpu)
            procs = host_cores()
            one_s = ref.one()
            el_all = ref.concurrent(procs)
            cpu = {"value": procs * ref.updates / el_all / 1e9, "unit": UNIT, "cores": procs,
                   "kind": "reference", "sample": ref.describe(procs),
                   "value_1process": ref.updates / one_s / 1e9, "port": port}
        else:
            cpu = dict(port, unit=UNIT)
            cpu["sample"] += f"; CPU {cpu_model()}"

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
                       "l2": "inputs larger than L2 (a two-step pass streams 10 x 67 MB fields = 671 MB > 126 MB)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": ("wb::step2_kernel_tma (two fused steps per pass)" if two
                                    else "wb::step_kernel_tma4 (fused step)"),
                         "algorithmic_bytes_per_cell_update": 6 * item,
                         "algorithmic_bytes_per_launch": 6 * item * C * (2 if two else 1),
                         "streamed_bytes_per_launch": (10 if two else 6) * item * C,
                         "streamed_gbs": streamed, "streamed_frac": streamed / peak,
                         "physical_gbs": physical,
                         "physical_frac": physical / peak if physical else None,
                         "pair_launches": pairs, "single_launches": singles,
                         "launch_ms": k_ms, "share": share, "share_source": share_src,
                         "kernel_ms_per_step": ms_per_step * share,
                         "event_sampled_launch_ms": ev_ms,
                         "event_sampled_note": f"CUDA events around every {PROFILE_EVERY}th "
                                               "launch of an extra evaluation (diagnostic: "
                                               "events break the PDL overlap)",
                         "traffic_source": NCU_TRAFFIC_SRC,
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3,
                    "host_buffers": "pinned", "value_pageable": pageable},
            "gpu_launches": int(stats["launches"]),
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)


def c5_workload(world, scaling, n_steps):
    """3D FWI on 2048 x 2048 planes, slab-decomposed along
    axis 0, one slab per GPU.  weak: 256 planes per GPU (1.07e9 cells),
    global (256 P) x 2048^2; strong: global 2048^3."""
    n0 = 256 * world if scaling == "weak" else 2048
    return dict(name=f"fwi3d_c5_{n0}x2048^2_slabs", shape=(n0, 2048, 2048), dx=1e-4,
                c0=6000.0, rho0=2700.0, eps=1e-5, n_steps=n_steps, freq=5e6, cycles=2,
                amp=1e12, k=1e13, precision="single", truth_gamma=0.9)


def build_c5_problem(W, wl):
    """Model gamma = 1 and truth gamma = 0.9 everywhere (a 10% density
    contrast), as constant broadcast views: no process materialises the
    global grid, each slab uploads its own planes.  Source at the axis-0 = 3
    face centre, 33 x 33 sensors on the plane n0-4."""
    shape = wl["shape"]
    n0, n1, n2 = shape
    dx, c0 = wl["dx"], wl["c0"]
    grid = W.build_grid(shape, dx)
    model = W.MaterialModel.rho_scaled(np.broadcast_to(np.float64(1.0), shape), grid,
                                       rho0=wl["rho0"], c0=c0, eps=wl["eps"])
    truth = model.with_gamma(np.broadcast_to(np.float64(wl["truth_gamma"]), shape))
    src = W.SourceSpec(node=(3, n1 // 2, n2 // 2), amplitude=wl["amp"], frequency=wl["freq"],
                       cycles=wl["cycles"])
    lin = np.unique(np.round(np.linspace(2, n1 - 3, 33)).astype(int))
    sensors = W.SensorArray(nodes=[(n0 - 4, j, k) for j in lin for k in lin])
    problem = W.FwiProblem(grid=grid, time=W.TimeConfig(wl["n_steps"], 0.5 * dx / c0),
                           material=model, sources=[src], sensors=sensors,
                           measured=np.zeros((1, len(sensors), wl["n_steps"])))
    return problem, model, truth


def run_native_slab(args):
    """C5: one slab per rank (SlabGradient.for_rank), peer ghost stores
    through CUDA IPC (or NCCL send/recv with --halo nccl), two-step passes."""
    rank, world, local = dist_setup()
    import torch

    import paper_2509_15744_b200 as W
    from paper_2509_15744_b200.distributed import SlabGradient

    wl = c5_workload(world, args.scaling, args.c5_steps)
    problem, model, truth = build_c5_problem(W, wl)
    cfg = W.SuperpositionConfig(k=wl["k"], precision=wl["precision"])
    sg = SlabGradient.for_rank(problem, model, cfg, rank, world, device=local, halo=args.halo)
    sg.upload()
    sg.set_measured(sg.record_traces(truth))   # owned sensors' truth traces (refine = 1)
    ctx = sg.ctxs[0]
    C = ctx.grid.n_nodes
    n_steps = wl["n_steps"]
    updates = 2 * (n_steps - 1) * C                       # per rank per evaluation

    for _ in range(args.warmup):
        sg.run()
    barrier(world)
    ctx.synchronize()
    ctx.reset_stats()
    with ClockSampler(local) as clocks:
        torch.cuda.profiler.start()
        ctx.timer_mark(0)
        for _ in range(args.steps):
            sg.run()
        ctx.timer_mark(1)
        ms = ctx.timer_elapsed_ms(0, 1)
        torch.cuda.profiler.stop()
    stats = ctx.stats()
    barrier(world)
    ms = max_over_ranks(ms, world)
    ms_per_step = ms / args.steps
    value = world * updates / (ms_per_step * 1e-3) / 1e9

    peaks, peak_kind = measured_peaks()
    peak = float(peaks["hbm_gbs"])
    item = ITEMSIZE[wl["precision"]]
    pairs = stats.get("pair_launches", 0)
    singles = stats["step_launches"] - pairs
    two = pairs >= singles
    share, share_src = launch_share("step2_kernel_tma" if two else "step_kernel_tma4", "c5")
    n_dom = (pairs if two else singles) / args.steps
    k_ms = ms_per_step * share / max(n_dom, 1)
    achieved = 6 * item * (2 if two else 1) * C / (k_ms * 1e-3) / 1e9
    traffic = ncu_traffic(f"{'step2_kernel' if two else 'step_kernel'}_single_c5")

    # end to end: this rank's gamma planes H2D from pinned host memory, the
    # evaluation, this rank's gradient planes D2H into pinned host memory
    lo, hi = ctx.alloc_range
    pinned_gb = ((hi - lo) * 8 + ctx.grid.shape[0] * 4) * wl["shape"][1] * wl["shape"][2] / 1e9
    e2e = None
    if pinned_gb <= 48:   # the 2048^3 one-GPU point would need ~100 GB of pinned host memory
        g_loc = torch.empty((hi - lo,) + tuple(wl["shape"][1:]), dtype=torch.float64,
                            pin_memory=True).numpy()
        g_loc[...] = 1.0
        out = torch.empty(ctx.grid.shape, dtype=torch.float32, pin_memory=True).numpy()

        def api_call():
            sg.upload(gamma_local=[g_loc])
            sg.run()
            return ctx.get_accumulator(out)

        api_call()
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            api_call()
        e2e_s = max_over_ranks((time.perf_counter() - t0) / args.steps, world)
        e2e = {"value": world * updates / e2e_s / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": g_loc.nbytes, "d2h_bytes_per_step": out.nbytes,
               "ms_per_step": e2e_s * 1e3}
    else:
        e2e = {"value": None, "unit": UNIT,
               "note": f"skipped: {pinned_gb:.0f} GB of pinned host buffers per rank"}
    memory_mode = "four_fields (single steps)" if pairs == 0 else "fast (two-step passes)"
    dev_bytes = ctx.device_bytes()
    sg.close()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": wl["name"], "config": "C5 (SURVEY 8d)",
                       "grid": list(wl["shape"]), "slab_planes_per_gpu": wl["shape"][0] // world,
                       "n_steps": n_steps, "shots": 1, "precision": wl["precision"],
                       "k": wl["k"], "parallelism": "slab", "halo": args.halo,
                       "two_step_slabs": bool(sg.two_step and pairs > 0),
                       "cell_updates_per_step": world * updates,
                       "truth": "homogeneous gamma 0.9 vs model 1.0 (traces synthesized on "
                                "the slabs, refine = 1)",
                       "weak_scaling_n1": ("the same per-GPU work on one GPU: python bench.py "
                                           "--workload c5 (profiles/r2/bench_c5_1gpu_r2e.json); "
                                           "the default N = 1 line is C2 256^3"),
                       "l2": "inputs larger than L2 (4.3 GB per field per GPU)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": ("wb::step2_kernel_tma (two fused steps per pass)" if two
                                    else "wb::step_kernel_tma4 (fused step)"),
                         "algorithmic_bytes_per_cell_update": 6 * item,
                         "algorithmic_bytes_per_launch": 6 * item * C * (2 if two else 1),
                         "launch_ms": k_ms, "share": share, "share_source": share_src,
                         "pair_launches": pairs, "single_launches": singles,
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})"},
            "e2e": e2e,
            "memory_mode": memory_mode,
            "device_bytes_per_gpu": dev_bytes,
            "gpu_launches": int(stats["launches"]),
            "clocks": clocks.summary(),
            "cpu_baseline": None,
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
    # CPU samples (steps of the 256^3 sweep): the Numba reference runs
    # ~0.09 Gcell-upd/s per process at N <= 24 on these hosts, so N = 16 is
    # ~5-8 s per process and the reference arm's 25 default steps (one
    # concurrent evaluation per core each) finish in a few minutes
    ap.add_argument("--cpu-sample-steps", type=int, default=16)
    ap.add_argument("--ref-sample-steps", type=int, default=16)
    ap.add_argument("--no-cpu", action="store_true")
    # workload: c2 (256^3, one GPU; shot-parallel across GPUs) or c5 (2048^2
    # planes, one slab per GPU); auto = c2 on one GPU, c5 on several
    ap.add_argument("--workload", choices=["auto", "c2", "c5"], default="auto")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--halo", choices=["ipc", "nccl"], default="ipc")
    ap.add_argument("--c5-steps", type=int, default=200)
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    workload_name = args.workload if args.workload != "auto" else ("c5" if world > 1 else "c2")
    if args.impl == "reference":
        run_reference_arm(args)
    elif workload_name == "c5":
        run_native_slab(args)
    else:
        run_native(args)


if __name__ == "__main__":
    main()
