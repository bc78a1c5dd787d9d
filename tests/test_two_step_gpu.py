"""GPU parity of the two-steps-per-pass kernel (csrc/step2_kernel.cuh).

Grids of whole 64 x 8 tiles run the sweeps as two-step passes (plus one
single step at an odd range end).  Every result must be bit-identical to the
single-step kernels and to the oracle (oracle/oracle.py): gradients, costs,
traces, final windows and the stability report.  Sources and sensors sit on
tile edges and on the plane-chunk boundaries, where the recomputed ring and
the chunk overlap planes are exercised."""

import numpy as np
import pytest

from helpers import bits_equal
from oracle import oracle as O

pytestmark = pytest.mark.gpu

COST_RTOL = 1e-13
RHO1, KAPPA1, RHO2, KAPPA2 = 1.204, 1.419e5, 2643.0, 6.87e8


@pytest.fixture(scope="module")
def W():
    import paper_2509_15744_b200 as W

    from paper_2509_15744_b200 import _native

    _native.load(require_device=True)
    return W


def _materials(W, flavor, gamma, grid, dx):
    if flavor == "rho_scaled":
        return (W.MaterialModel.rho_scaled(gamma, grid, rho0=2700.0, c0=6000.0),
                O.Material("rho_scaled", gamma, dx, rho0=2700.0, c0=6000.0), 6000.0)
    return (W.MaterialModel.acoustic(gamma, grid, RHO1, KAPPA1, RHO2, KAPPA2),
            O.Material("acoustic", gamma, dx, rho1=RHO1, kappa1=KAPPA1, rho2=RHO2,
                       kappa2=KAPPA2), float(np.sqrt(KAPPA2 / RHO2)))


def _problem(W, shape, flavor, n_steps, seed):
    rng = np.random.default_rng(seed)
    dx = 1e-4 if flavor == "rho_scaled" else 1e-2
    lo = 0.2 if flavor == "rho_scaled" else 0.0
    gamma = rng.uniform(lo, 1.0, size=shape)
    grid = W.build_grid(shape, dx)
    mat, omat, c_max = _materials(W, flavor, gamma, grid, dx)
    dt = 0.45 * dx / c_max / np.sqrt(len(shape))
    freq = 0.05 / dt
    nd = len(shape)
    # two shots: one on a chunk boundary plane / tile corner, one interior
    nodes = [tuple([min(8, shape[0] - 1)] + [63 if s > 64 else s // 2 for s in shape[1:]])
             if nd == 3 else (min(8, shape[0] - 1), 63),
             tuple(s // 3 for s in shape)]
    amp = 1e12 if flavor == "rho_scaled" else 1.0
    srcs = [W.SourceSpec(node=n, amplitude=amp, frequency=freq, cycles=2) for n in nodes]
    def edge(n, cuts):   # tile / chunk edges inside an axis of n nodes
        return sorted({min(c, n - 1) for c in cuts} | {0, n - 1})

    ks = edge(shape[-1], (63, 64))
    if nd == 3:
        sens = [(i, j, k) for i in sorted({shape[0] - 1, max(shape[0] - 8, 0)})
                for j in edge(shape[1], (7, 8)) for k in ks]
    else:
        sens = [(i, k) for i in edge(shape[0], (7, 8)) for k in ks]
    sens = list(dict.fromkeys(sens))
    measured = rng.normal(scale=1e-10 if flavor == "rho_scaled" else 1e-3,
                          size=(len(srcs), len(sens), n_steps))
    problem = W.FwiProblem(grid=grid, time=W.TimeConfig(n_steps, dt), material=mat,
                           sources=srcs, sensors=W.SensorArray(nodes=sens), measured=measured)
    support = np.array([grid.flat_index(n) for n in sens], dtype=np.int64)
    shots = [(O.Source(s.node, amp, freq, 2), O.FwiShot(support, measured[q], dt))
             for q, s in enumerate(srcs)]
    return problem, mat, omat, dt, shots


SHAPES = [(40, 8, 64), (9, 24, 128), (64, 128), (3, 16, 192), (70, 48, 128), (10, 16, 96)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("flavor", ["rho_scaled", "acoustic"])
@pytest.mark.parametrize("prec", ["single", "double"])
@pytest.mark.parametrize("n_steps", [60, 61])
def test_two_step_gradient_bitexact(W, shape, flavor, prec, n_steps):
    from paper_2509_15744_b200 import engine

    problem, mat, omat, dt, shots = _problem(W, shape, flavor, n_steps, sum(shape) + n_steps)
    cfg = W.SuperpositionConfig(k=1e13 if flavor == "rho_scaled" else 1e3, precision=prec)
    ctx = engine.get_context(problem.grid, W.precision_dtype(prec))
    ctx.set_cluster(False)   # the step kernels themselves (small 2D fp32 grids default to the cluster engine)
    out = {}
    for two in (True, False):
        ctx.set_two_step(2 if two else 0)   # 2: fp64 grids too
        ctx.reset_stats()
        out[two] = W.gradient_superposed(problem, mat, cfg)
        pairs = ctx.stats()["pair_launches"]
        if two:
            assert pairs > 0, "two-step path did not run"
        if not two:
            assert pairs == 0
    ctx.set_two_step(1)
    ctx.set_cluster(None)
    assert bits_equal(out[True].gradient, out[False].gradient)
    cost, grad, _ = O.gradient_superposed(omat, dt, n_steps, shots, cfg.k, prec)
    assert bits_equal(out[True].gradient, grad)
    assert abs(out[True].cost - cost) <= COST_RTOL * abs(cost)


@pytest.mark.parametrize("shape", [(40, 8, 64), (64, 128)])
@pytest.mark.parametrize("dn", ["f32", "f64"])
def test_two_step_forward_traces_and_window(W, shape, dn):
    """Trace gather (no accumulation) and the final window after an odd number
    of steps match the oracle's run_forward."""
    from paper_2509_15744_b200 import engine

    dtype = np.float32 if dn == "f32" else np.float64
    problem, mat, omat, dt, shots = _problem(W, shape, "rho_scaled", 73, 3)
    ctx = engine.get_context(problem.grid, dtype)
    ctx.set_two_step(2)
    ctx.set_cluster(False)
    try:
        ctx.reset_stats()
        res = W.run_forward(mat, problem.time, problem.sources,
                            W.SensorArray(nodes=problem.sensors.nodes), dtype=dtype)
        assert ctx.stats()["pair_launches"] > 0
    finally:
        ctx.set_two_step(1)
        ctx.set_cluster(None)
    sup = np.array([problem.grid.flat_index(n) for n in problem.sensors.nodes], dtype=np.int64)
    osrc = [s for s, _ in shots]
    u_prev, u_cur, traces, _, peak = O.run_forward(omat, dt, 73, osrc, sensor_idx=sup,
                                                   dtype=dtype)
    assert bits_equal(res.window.u_prev, u_prev)
    assert bits_equal(res.window.u_cur, u_cur)
    assert bits_equal(res.traces, traces)
    assert res.peak_abs == peak


@pytest.mark.parametrize("courant", [1.2, 0.75])
def test_two_step_instability_step(W, courant):
    """The blow-up step and max reported from a two-step sweep equal the
    oracle's (the check can land on either half of a pass)."""
    shape, dx = (16, 16, 64), 1e-4
    dt = courant * dx / 6000.0
    grid = W.build_grid(shape, dx)
    gamma = np.ones(shape)
    mat = W.MaterialModel.rho_scaled(gamma, grid, rho0=2700.0, c0=6000.0)
    src = W.SourceSpec(node=(8, 8, 32), amplitude=1e12, frequency=3e6, cycles=2)
    n_steps = 400
    with pytest.raises(W.SolverInstabilityError) as ei:
        W.run_forward(mat, W.TimeConfig(n_steps, dt), [src], None)
    omat = O.Material("rho_scaled", gamma, dx, rho0=2700.0, c0=6000.0)
    with pytest.raises(O.OracleInstability) as eo:
        O.run_forward(omat, dt, n_steps, [O.Source((8, 8, 32), 1e12, 3e6, 2)])
    assert ei.value.step == eo.value.step
    assert ei.value.max_abs == eo.value.max_abs or (
        np.isnan(ei.value.max_abs) and np.isnan(eo.value.max_abs))


# ------------------------------------------------ k batching
def test_calibrate_k_batched_equals_unbatched(W, golden):
    """One forward sweep per precision for every decade gives the same rows
    as one gradient_superposed per decade (and the reference's rows)."""
    import cases
    from helpers import product_tato_problem

    g = golden("tato2d")
    c = cases.tato2d_case()
    problem = product_tato_problem(W, c)
    mat = problem.material(g["g_bar"])
    fast = W.calibrate_k(problem, mat, k_start=1e18)
    slow = W.calibrate_k(problem, mat, k_start=1e18, batch=False)
    assert fast.rows == slow.rows
    assert fast.k == slow.k == float(g["cal_k"])
    assert fast.diverged_at == slow.diverged_at


@pytest.mark.parametrize("shape", [(40, 8, 64), (33, 64)])
@pytest.mark.parametrize("prec", ["single", "double"])
def test_kbatch_bitexact_per_k(W, shape, prec):
    from paper_2509_15744_b200 import gradients as G

    problem, mat, omat, dt, shots = _problem(W, shape, "rho_scaled", 60, 7)
    problem = W.FwiProblem(grid=problem.grid, time=problem.time, material=mat,
                           sources=problem.sources[:1], sensors=problem.sensors,
                           measured=problem.measured[:1])
    batch = G.KBatch(problem, mat, prec)
    try:
        for k in (1e15, 1e13, 1e11):
            got = batch.gradient(k)
            ref = W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=k, precision=prec))
            assert bits_equal(got.gradient, ref.gradient), k
            assert got.cost == ref.cost
        # interleave an unrelated evaluation on the same context, then batch again
        other = mat.with_gamma(np.asarray(mat.gamma) * 0.9)
        W.gradient_superposed(problem, other, W.SuperpositionConfig(k=1e13, precision=prec))
        got = batch.gradient(1e12)
        ref = W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=1e12, precision=prec))
        assert bits_equal(got.gradient, ref.gradient)
    finally:
        batch.close()


def test_ksweep_batched_rows(W):
    from paper_2509_15744_b200 import gradients as G

    problem, mat, _, _, _ = _problem(W, (24, 16, 64), "rho_scaled", 50, 9)
    problem = W.FwiProblem(grid=problem.grid, time=problem.time, material=mat,
                           sources=problem.sources[:1], sensors=problem.sensors,
                           measured=problem.measured[:1])
    ks = [1e14, 1e12]
    rows, ref = W.ksweep(problem, mat, ks)
    for (k, e32, e64) in rows:
        g32 = W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=k, precision="single"))
        g64 = W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=k, precision="double"))
        assert e32 == G.rel_mse(g32.gradient, ref)
        assert e64 == G.rel_mse(g64.gradient, ref)


# ------------------------------------------------ device field dumps (8f-4)
@pytest.mark.parametrize("shape", [(40, 8, 64), (33, 64), (37, 45, 19)])
@pytest.mark.parametrize("prec", ["single", "double"])
def test_device_dump_equals_host_dump(W, tmp_path, shape, prec):
    from paper_2509_15744_b200 import engine
    from paper_2509_15744_b200 import io as WIO

    problem, mat, _, _, _ = _problem(W, shape, "rho_scaled", 30, 4)
    res = W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=1e13, precision=prec))
    ctx = engine.get_context(problem.grid, W.precision_dtype(prec))
    flat = ctx.get_field("acc", first_axis_fastest=True)
    assert bits_equal(flat, np.ravel(res.gradient, order="F"))
    a = WIO.dump_device_field(tmp_path / "dev", ctx, "acc", dt=problem.time.dt, step_index=30)
    b = WIO.dump_field(tmp_path / "host", res.gradient, problem.grid, dt=problem.time.dt,
                       step_index=30)
    assert a.read_bytes() == b.read_bytes()
    assert a.with_suffix(".json").read_text() == b.with_suffix(".json").read_text()
    gam = ctx.get_field("gamma", first_axis_fastest=True)
    dt = np.float32 if prec == "single" else np.float64
    assert bits_equal(gam, np.ravel(np.asarray(mat.gamma).astype(dt), order="F"))


# ------------------------------------------------ randomised parity sweep
@pytest.mark.parametrize("seed", range(12))
def test_two_step_random_cases(W, seed):
    """Random tile-multiple grids, step counts, flavours, precisions and
    source / sensor placements: gradient and cost bit-exact vs the oracle."""
    rng = np.random.default_rng(1000 + seed)
    nd = 3 if seed % 4 else 2
    if nd == 3:
        shape = (int(rng.integers(2, 30)), 8 * int(rng.integers(1, 5)),
                 int(rng.choice([64, 96, 128, 192])))
    else:
        shape = (8 * int(rng.integers(1, 9)), int(rng.choice([64, 128, 192])))
    flavor = "rho_scaled" if seed % 3 else "acoustic"
    prec = "single" if seed % 2 == 0 else "double"
    n_steps = int(rng.integers(20, 70))
    dx = 1e-4 if flavor == "rho_scaled" else 1e-2
    gamma = rng.uniform(0.2 if flavor == "rho_scaled" else 0.0, 1.0, size=shape)
    grid = W.build_grid(shape, dx)
    mat, omat, c_max = _materials(W, flavor, gamma, grid, dx)
    dt = 0.4 * dx / c_max / np.sqrt(nd)
    amp = 1e12 if flavor == "rho_scaled" else 1.0
    node = tuple(int(rng.integers(0, s)) for s in shape)
    src = W.SourceSpec(node=node, amplitude=amp, frequency=0.05 / dt, cycles=2)
    sens = list(dict.fromkeys(tuple(int(rng.integers(0, s)) for s in shape) for _ in range(7)))
    meas = rng.normal(scale=1e-10 if flavor == "rho_scaled" else 1e-3,
                      size=(1, len(sens), n_steps))
    problem = W.FwiProblem(grid=grid, time=W.TimeConfig(n_steps, dt), material=mat, sources=[src],
                           sensors=W.SensorArray(nodes=sens), measured=meas)
    from paper_2509_15744_b200 import engine

    ctx = engine.get_context(grid, W.precision_dtype(prec))
    ctx.set_two_step(2)
    ctx.set_cluster(False)
    try:
        ctx.reset_stats()
        k = 1e13 if flavor == "rho_scaled" else 1e3
        res = W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=k, precision=prec))
        assert ctx.stats()["pair_launches"] > 0
    finally:
        ctx.set_two_step(1)
        ctx.set_cluster(None)
    support = np.array([grid.flat_index(n) for n in sens], dtype=np.int64)
    shots = [(O.Source(node, amp, 0.05 / dt, 2), O.FwiShot(support, meas[0], dt))]
    cost, grad, _ = O.gradient_superposed(omat, dt, n_steps, shots, k, prec)
    assert bits_equal(res.gradient, grad)
    assert abs(res.cost - cost) <= COST_RTOL * abs(cost)


# ------------------------------------------------ sweep graphs (WO_OPT_GRAPHS)
@pytest.mark.parametrize("shape", [(40, 8, 64), (64, 128), (33, 64)])
@pytest.mark.parametrize("cluster", [False, None])
def test_sweep_graph_replay_matches_direct_launches(W, shape, cluster):
    """Repeated evaluations replay captured sweep graphs; a new gamma (same
    scalars: data, graph kept), new measured data, a new k and a new source
    frequency (new key: recapture) must all give the direct-launch bits."""
    from paper_2509_15744_b200 import engine

    problem, mat, _, _, _ = _problem(W, shape, "rho_scaled", 40, 11)
    problem = W.FwiProblem(grid=problem.grid, time=problem.time, material=mat,
                           sources=problem.sources[:1], sensors=problem.sensors,
                           measured=problem.measured[:1])
    ctx = engine.get_context(problem.grid, np.float32)
    ctx.set_cluster(cluster)   # None: the default (2D: the cluster engine, no graphs)
    cfg = W.SuperpositionConfig(k=1e13, precision="single")

    def both(prob, m, c):
        ctx.set_graphs(False)
        ref = W.gradient_superposed(prob, m, c)
        ctx.set_graphs(True)
        got = [W.gradient_superposed(prob, m, c) for _ in range(3)]   # capture, replay
        for g in got:
            assert bits_equal(g.gradient, ref.gradient)
            assert g.cost == ref.cost

    both(problem, mat, cfg)
    rng = np.random.default_rng(3)
    mat2 = mat.with_gamma(np.asarray(mat.gamma) * rng.uniform(0.8, 1.0, size=problem.grid.shape))
    both(problem, mat2, cfg)
    problem.measured = problem.measured * 1.5
    both(problem, mat2, cfg)
    both(problem, mat2, W.SuperpositionConfig(k=1e11, precision="single"))
    s0 = problem.sources[0]
    p3 = W.FwiProblem(grid=problem.grid, time=problem.time, material=mat2,
                      sources=[W.SourceSpec(node=s0.node, amplitude=s0.amplitude,
                                            frequency=s0.frequency * 1.3, cycles=2)],
                      sensors=problem.sensors, measured=problem.measured)
    both(p3, mat2, cfg)
    ctx.set_cluster(None)


@pytest.mark.parametrize("knob", [("WB_T2_NZ", "1"), ("WB_T2_NZ", "2"), ("WB_T2_NZ", "3"),
                                  ("WB_T2_LAYERS", "20x1,5x3,10x1"),
                                  ("WB_T2_LAYERS", "1x1,2x1,42x1")])
@pytest.mark.parametrize("prec", ["single", "double"])
def test_two_step_long_chunks(W, knob, prec):
    """Chunks of 15-45 planes per CTA (several TMA-ring wraps, the mbarrier
    parities, the chunk-end plane through the ring) and uneven z layers down
    to one plane: the size model picks such chunks only on large grids, so
    force them (WB_T2_NZ / WB_T2_LAYERS, read once per process) in a
    subprocess."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, **{knob[0]: knob[1]})
    out = subprocess.run([sys.executable, os.path.join(here, "_long_chunk_case.py"), prec],
                         env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stdout + out.stderr


@pytest.mark.parametrize("shape", [(256, 256), (101, 101), (33, 29), (40, 200), (97, 64),
                                   (200, 200), (70, 96)])   # partial last CTAs
@pytest.mark.parametrize("prec", ["single", "double"])
def test_cluster_sweep_engine_bitwise(W, shape, prec):
    """Small 2D grids: the cluster-resident whole-sweep engine (one launch per
    sweep, fields in distributed shared memory) gives the step kernels' bits
    (and the oracle's) for the superposed gradient, FWI with a source near a
    CTA row boundary and sensors on several CTAs."""
    from oracle import oracle as O
    from paper_2509_15744_b200 import engine

    rng = np.random.default_rng(sum(shape))
    dx, n_steps = 2e-4, 121
    dt = 0.5 * dx / 6000.0
    grid = W.build_grid(shape, dx)
    gamma = rng.uniform(0.3, 1.0, size=shape)
    mat = W.MaterialModel.rho_scaled(gamma, grid, rho0=2700.0, c0=6000.0)
    src = W.SourceSpec(node=(shape[0] // 2 + 1, shape[1] // 3), amplitude=1e12, frequency=1.5e6,
                       cycles=2)
    nodes = sorted({(i, j) for i in (0, shape[0] // 4, shape[0] - 1)
                    for j in (0, shape[1] // 2, shape[1] - 1)}
                   # a sensor in the source's packed pair: the forward sweep
                   # only gathers there, the backward sweep injects both
                   | {(src.node[0], src.node[1] ^ 1)})
    meas = rng.normal(scale=1e-9, size=(1, len(nodes), n_steps))
    problem = W.FwiProblem(grid=grid, time=W.TimeConfig(n_steps, dt), material=mat,
                           sources=[src], sensors=W.SensorArray(nodes=nodes), measured=meas)
    cfg = W.SuperpositionConfig(k=1e14, precision=prec)
    ctx = engine.get_context(grid, W.precision_dtype(prec))
    try:
        ctx.set_cluster(True)
        ctx.reset_stats()
        on = W.gradient_superposed(problem, mat, cfg)
        launches_on = ctx.stats()["step_launches"]
        again = W.gradient_superposed(problem, mat, cfg)   # shared memory left by a backward sweep
        assert bits_equal(again.gradient, on.gradient) and again.cost == on.cost
        ctx.set_cluster(False)
        off = W.gradient_superposed(problem, mat, cfg)
    finally:
        ctx.set_cluster(None)
    assert launches_on == 2        # one launch per sweep
    assert bits_equal(on.gradient, off.gradient)
    assert on.cost == off.cost
    omat = O.Material("rho_scaled", gamma, dx, rho0=2700.0, c0=6000.0)
    support = np.array([grid.flat_index(n) for n in nodes], dtype=np.int64)
    shots = [(O.Source(src.node, 1e12, 1.5e6, 2), O.FwiShot(support, meas[0], dt))]
    _, grad, _ = O.gradient_superposed(omat, dt, n_steps, shots, 1e14, prec)
    assert bits_equal(on.gradient, grad)


@pytest.mark.parametrize("seed", range(24))
def test_cluster_sweep_random_shapes(W, seed):
    """Random 2D shapes that fit one cluster (odd widths, partial last CTAs,
    a handful of rows), random source / sensors: the cluster sweep equals the
    step kernels bit for bit, fp32 and fp64."""
    from paper_2509_15744_b200 import engine

    rng = np.random.default_rng(500 + seed)
    while True:   # one cluster: 16 CTAs, threads of 2 (fp64) / 4 (fp32) rows x 4 cells
        shape = (int(rng.integers(3, 300)), int(rng.integers(3, 300)))
        rows = -(-shape[0] // 16)
        if all(-(-shape[1] // 4) * (-(-rows // rt) * rt) <= 1024 for rt in (2, 4)):
            break
    dx, n_steps = 2e-4, int(rng.integers(20, 90))
    dt = 0.5 * dx / 6000.0
    grid = W.build_grid(shape, dx)
    gamma = rng.uniform(0.3, 1.0, size=shape)
    mat = W.MaterialModel.rho_scaled(gamma, grid, rho0=2700.0, c0=6000.0)
    src = W.SourceSpec(node=tuple(int(rng.integers(0, n)) for n in shape), amplitude=1e12,
                       frequency=3e6, cycles=2)
    nodes = sorted({tuple(int(rng.integers(0, n)) for n in shape) for _ in range(12)})
    meas = rng.normal(scale=1e-9, size=(1, len(nodes), n_steps))
    problem = W.FwiProblem(grid=grid, time=W.TimeConfig(n_steps, dt), material=mat,
                           sources=[src], sensors=W.SensorArray(nodes=nodes), measured=meas)
    for prec in ("single", "double"):
        cfg = W.SuperpositionConfig(k=1e14, precision=prec)
        ctx = engine.get_context(grid, W.precision_dtype(prec))
        try:
            ctx.set_cluster(True)
            ctx.reset_stats()
            on = W.gradient_superposed(problem, mat, cfg)
            launches = ctx.stats()["step_launches"]
            ctx.set_cluster(False)
            off = W.gradient_superposed(problem, mat, cfg)
        finally:
            ctx.set_cluster(None)
        assert launches == 2, shape
        assert bits_equal(on.gradient, off.gradient), (shape, prec)
        assert on.cost == off.cost, (shape, prec)
