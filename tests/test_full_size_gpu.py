"""Parity at the bench's full grid size (BASELINE configs[1]: 256^3) and
above, where the small-case tests cannot reach: the chunk / wave model picks
the production launch shapes (10 z-chunks of 26 planes, 2.9 waves of CTAs)
only on big grids.

* 256^3 superposed gradient vs the C oracle (bit-exact, fewer time steps
  than the bench so the oracle finishes in seconds);
* 512^3: two-step passes vs single steps, bit-exact (size-independent
  property: both are exact restatements of the same update);
* 256^3 fp64 time reversal: forward then backward replay returns to the zero
  initial state (SPEC acceptance 2 at full size)."""

import numpy as np
import pytest

from helpers import bits_equal
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def W():
    import paper_2509_15744_b200 as W

    from paper_2509_15744_b200 import _native

    _native.load(require_device=True)
    return W


def _bench_like(W, n, n_steps, seed=0):
    rng = np.random.default_rng(seed)
    shape = (n, n, n)
    dx = 1e-4
    dt = 0.45 * dx / 6000.0 / np.sqrt(3)
    gamma = rng.uniform(0.3, 1.0, size=shape)
    grid = W.build_grid(shape, dx)
    mat = W.MaterialModel.rho_scaled(gamma, grid, rho0=2700.0, c0=6000.0)
    src = W.SourceSpec(node=(3, n // 2, n // 2), amplitude=1e12, frequency=0.05 / dt, cycles=2)
    lin = np.unique(np.round(np.linspace(2, n - 3, 33)).astype(int))
    sens = [(n - 4, int(j), int(k)) for j in lin for k in lin]
    meas = rng.normal(scale=1e-10, size=(1, len(sens), n_steps))
    problem = W.FwiProblem(grid=grid, time=W.TimeConfig(n_steps, dt), material=mat,
                           sources=[src], sensors=W.SensorArray(nodes=sens), measured=meas)
    omat = O.Material("rho_scaled", gamma, dx, rho0=2700.0, c0=6000.0)
    support = np.array([grid.flat_index(s) for s in sens], dtype=np.int64)
    shots = [(O.Source(src.node, 1e12, 0.05 / dt, 2), O.FwiShot(support, meas[0], dt))]
    return problem, mat, omat, dt, shots


@pytest.mark.parametrize("prec", ["single", "double"])
def test_bench_grid_gradient_matches_oracle(W, prec):
    from paper_2509_15744_b200 import engine

    n_steps = 24
    problem, mat, omat, dt, shots = _bench_like(W, 256, n_steps)
    ctx = engine.get_context(problem.grid, W.precision_dtype(prec))
    ctx.set_two_step(2)                      # two-step passes for fp64 too
    ctx.reset_stats()
    try:
        res = W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=1e13, precision=prec))
        assert ctx.stats()["pair_launches"] > 0
    finally:
        ctx.set_two_step(1)
    cost, grad, _ = O.gradient_superposed(omat, dt, n_steps, shots, 1e13, prec)
    assert bits_equal(res.gradient, grad)
    assert abs(res.cost - cost) <= 1e-13 * abs(cost)


def test_two_step_equals_single_step_512(W):
    from paper_2509_15744_b200 import engine

    problem, mat, _, _, _ = _bench_like(W, 512, 12, seed=1)
    cfg = W.SuperpositionConfig(k=1e13, precision="single")
    ctx = engine.get_context(problem.grid, np.float32)
    try:
        ctx.set_two_step(0)
        single = W.gradient_superposed(problem, mat, cfg)
        ctx.set_two_step(1)
        ctx.reset_stats()
        paired = W.gradient_superposed(problem, mat, cfg)
        assert ctx.stats()["pair_launches"] > 0
    finally:
        ctx.set_two_step(1)
        engine.release_contexts()
    assert bits_equal(paired.gradient, single.gradient)
    assert paired.cost == single.cost


def test_time_reversal_roundtrip_256(W):
    n, n_steps = 256, 120
    dx = 1e-4
    dt = 0.5 * dx / 6000.0
    grid = W.build_grid((n, n, n), dx)
    mat = W.MaterialModel.rho_scaled(np.ones((n, n, n)), grid, rho0=2700.0, c0=6000.0)
    src = W.SourceSpec(node=(n // 2, n // 2, n // 2), amplitude=1e12, frequency=0.05 / dt,
                       cycles=2)
    time = W.TimeConfig(n_steps, dt)
    fwd = W.run_forward(mat, time, [src])
    idx = np.array([grid.flat_index(src.node)])
    back = W.run_backward(mat, time, fwd.window,
                          lambda k: (idx, np.array([W.burst_amplitude(k * dt, src)])))
    assert np.max(np.abs(back.u_cur)) <= 1e-10 * fwd.peak_abs


# ------------------------------------------------ BASELINE config sizes
def _host_ram_gb():
    try:
        import psutil

        return psutil.virtual_memory().available / 1e9
    except Exception:
        return 0.0


@pytest.mark.parametrize("prec", ["single", "double"])
def test_bench_workload_production_n_matches_oracle(W, prec):
    """The bench workload itself (bench.py: C2 256^3, sphere-void truth traces
    synthesized on the GPU, 33 x 33 sensors, k = 1e13) at N = 200 steps — the
    production launch sequence (511-pass sweeps shortened to 99 passes + the
    odd step) — bit-exact against the C oracle on the same inputs."""
    import bench

    wl = bench.workload(256, 200)
    wl["precision"] = prec
    problem, model = bench.build_problem(W, wl)
    cfg = W.SuperpositionConfig(k=wl["k"], precision=prec)
    res = W.gradient_superposed(problem, model, cfg)
    dt = problem.time.dt
    src = problem.sources[0]
    omat = O.Material("rho_scaled", np.asarray(model.gamma, dtype=np.float64), wl["dx"],
                      rho0=wl["rho0"], c0=wl["c0"])
    shots = [(O.Source(src.node, src.amplitude, src.frequency, src.cycles),
              O.FwiShot(problem.sensors.flat_indices(problem.grid), problem.measured[0], dt))]
    cost, grad, _ = O.gradient_superposed(omat, dt, wl["n_steps"], shots, wl["k"], prec)
    assert bits_equal(res.gradient, grad)
    assert abs(res.cost - cost) <= 1e-13 * abs(cost)


@pytest.mark.parametrize("prec", ["single", "double"])
def test_c1_2d_256_n3200_matches_oracle(W, prec):
    """C1: 2D rho-scaled FWI on 256^2, dx = 0.02/255,
    dt = 7.5e-9, N = 3200, source (128, 3), sensor ring (inset 3, stride 4),
    disk-void truth traces, bit-exact against the oracle."""
    import cases

    shape, n_steps = (256, 256), 3200
    dx, dt = 0.02 / 255, 7.5e-9
    grid = W.build_grid(shape, dx)
    model = W.MaterialModel.rho_scaled(np.ones(shape), grid, rho0=2700.0, c0=6000.0, eps=1e-5)
    src = W.SourceSpec(node=(128, 3), amplitude=1e12, frequency=1e6, cycles=2)
    nodes = cases.ring_nodes(shape, 3, 4)
    sens = W.SensorArray(nodes=nodes)
    problem = W.FwiProblem(grid=grid, time=W.TimeConfig(n_steps, dt), material=model,
                           sources=[src], sensors=sens)
    truth = cases.disk_gamma(shape, [((150, 120), 25)], 1e-5)
    problem.measured = W.synthesize_measurements(model.with_gamma(truth), problem, refine=1)
    res = W.gradient_superposed(problem, model, W.SuperpositionConfig(k=1e13, precision=prec))
    omat = O.Material("rho_scaled", np.ones(shape), dx, rho0=2700.0, c0=6000.0)
    shots = [(O.Source(src.node, 1e12, 1e6, 2),
              O.FwiShot(sens.flat_indices(grid), problem.measured[0], dt))]
    cost, grad, _ = O.gradient_superposed(omat, dt, n_steps, shots, 1e13, prec)
    assert bits_equal(res.gradient, grad)
    assert abs(res.cost - cost) <= 1e-13 * abs(cost)


def test_c3_tato_192_large_region_matches_oracle(W):
    """C3 3D TATO at 192^3, acoustic flavor (tato.py:175-178),
    an objective region of 40 x 40 x 40 = 64,000 support nodes
    (tato.py:143-163, 214-218), projected random design on a box: fp32
    superposed gradient bit-exact against the oracle."""
    n, n_steps = 192, 60
    shape = (n, n, n)
    dx = 0.01
    rho1, kappa1, rho2, kappa2 = 1.204, 1.419e5, 2643.0, 6.87e8
    dt = 0.5 * dx / np.sqrt(kappa2 / rho2)
    design = np.zeros(shape, dtype=bool)
    design[60:132, 40:152, 40:152] = True
    objective = np.zeros(shape, dtype=bool)
    objective[140:180, 76:116, 76:116] = True
    rng = np.random.default_rng(192)
    g_bar = np.where(design, rng.uniform(0.0, 1.0, size=shape), 0.0)
    grid = W.build_grid(shape, dx)
    src = W.SourceSpec(node=(20, 96, 96), amplitude=1.0, frequency=650.0 * 40, cycles=2)
    problem = W.TatoProblem(grid=grid, time=W.TimeConfig(n_steps, dt), source=src,
                            design_mask=design, objective_mask=objective, rho1=rho1,
                            kappa1=kappa1, rho2=rho2, kappa2=kappa2, r_f=1.5, eta=0.5,
                            mode="suppress")
    mat = problem.material(g_bar)
    res = W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=1e16, precision="single"))
    omat = O.Material("acoustic", g_bar, dx, rho1=rho1, kappa1=kappa1, rho2=rho2, kappa2=kappa2)
    support = np.flatnonzero(objective.reshape(-1)).astype(np.int64)
    area = float(objective.sum()) * dx ** 3
    shots = [(O.Source(src.node, 1.0, 650.0 * 40, 2),
              O.TatoShot(support, area, dt, dx, 3, "suppress"))]
    cost, grad, _ = O.gradient_superposed(omat, dt, n_steps, shots, 1e16, "single")
    assert len(support) == 64000
    assert bits_equal(res.gradient, grad)
    assert abs(res.cost - cost) <= 1e-13 * abs(cost)


def _crop_case(W, shape, src_node, n_steps, prec, two_step, seed):
    """Superposed gradient on a big grid vs the oracle on a crop around the
    source: after N steps the field (and every kernel increment) is exactly
    +0 farther than N cells from the source, in both computations, so the
    crop (margin N + 2 cells, or the real boundary) is an exact restatement.
    Exercises the plane offsets far from the origin (64-bit addressing)."""
    from paper_2509_15744_b200 import engine

    dx = 1e-4
    dt = 0.45 * dx / 6000.0 / np.sqrt(3)
    rng = np.random.default_rng(seed)
    m = n_steps + 2
    lo = [max(c - m, 0) for c in src_node]
    hi = [min(c + m + 1, n) for c, n in zip(src_node, shape)]
    crop = tuple(slice(a, b) for a, b in zip(lo, hi))
    gamma = np.empty(shape)
    for i in range(shape[0]):             # plane by plane: bounded temporaries
        gamma[i] = 0.5 + 0.5 * rng.random(shape[1:])
    grid = W.build_grid(shape, dx)
    mat = W.MaterialModel.rho_scaled(gamma, grid, rho0=2700.0, c0=6000.0)
    src = W.SourceSpec(node=src_node, amplitude=1e12, frequency=0.05 / dt, cycles=2)
    sens = [(src_node[0] + di, src_node[1] + dj, src_node[2] + dk)
            for di, dj, dk in ((-2, 1, 0), (1, -3, 2), (0, 4, -4))]
    sens = [s for s in sens if all(0 <= c < n for c, n in zip(s, shape))]
    meas = rng.normal(scale=1e-10, size=(1, len(sens), n_steps))
    problem = W.FwiProblem(grid=grid, time=W.TimeConfig(n_steps, dt), material=mat,
                           sources=[src], sensors=W.SensorArray(nodes=sens), measured=meas)
    ctx = engine.get_context(grid, W.precision_dtype(prec))
    try:
        ctx.set_two_step(two_step)
        ctx.reset_stats()
        res = W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=1e13, precision=prec))
        pairs = ctx.stats()["pair_launches"]
    finally:
        engine.release_contexts()
    g = res.gradient
    del gamma, mat, problem, res
    cshape = tuple(b - a for a, b in zip(lo, hi))
    cgrid_node = lambda s: tuple(c - a for c, a in zip(s, lo))  # noqa: E731
    rng2 = np.random.default_rng(seed)
    cg = np.empty(cshape)
    for i in range(hi[0]):                # replay the same random planes, keep the crop
        plane = 0.5 + 0.5 * rng2.random(shape[1:])
        if i >= lo[0]:
            cg[i - lo[0]] = plane[crop[1], crop[2]]
    omat = O.Material("rho_scaled", cg, dx, rho0=2700.0, c0=6000.0)
    support = np.array([np.ravel_multi_index(cgrid_node(s), cshape) for s in sens], dtype=np.int64)
    shots = [(O.Source(cgrid_node(src_node), 1e12, 0.05 / dt, 2),
              O.FwiShot(support, meas[0], dt))]
    _, ogr, _ = O.gradient_superposed(omat, dt, n_steps, shots, 1e13, prec)
    assert bits_equal(g[crop], ogr)
    g[crop] = 0
    assert not np.any(g)
    return pairs


@pytest.mark.parametrize("shape,src,two_step", [
    ((1024, 1024, 1024), (1019, 1000, 1010), 1),   # C4 grid, production 64-plane chunks
    ((520, 2048, 2048), (514, 1500, 2040), 1),     # > 2^31 cells, C5 planes
    ((1030, 2048, 2048), (1026, 30, 2000), 0),     # > 2^32 cells (single steps: 4 fields)
])
def test_big_grids_match_oracle_crop(W, shape, src, two_step):
    cells = int(np.prod(shape))
    if _host_ram_gb() < cells * 8 * 2.6 / 1e9:
        pytest.skip("not enough host memory for the fp64 gamma + gradient download")
    pairs = _crop_case(W, shape, src, 8, "single", two_step, seed=sum(shape))
    assert (pairs > 0) == bool(two_step)
