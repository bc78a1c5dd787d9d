"""GPU parity: the CUDA path (through the public API / C ABI) against the
reference golden fixtures and the CPU oracle.  Bit-exact for fields, traces
and gradients in fp32 and fp64; costs within 1e-13 relative (the reference
sums np.dot partials through BLAS)."""

import numpy as np
import pytest

import cases
from helpers import bits_equal, product_fwi_problem, product_tato_problem, rel_l2
from oracle import oracle as O

pytestmark = pytest.mark.gpu

COST_RTOL = 1e-13


@pytest.fixture(scope="module")
def W():
    import paper_2509_15744_b200 as W

    from paper_2509_15744_b200 import _native

    _native.load(require_device=True)
    return W


def _dt(dn):
    return np.float32 if dn == "f32" else np.float64


# ------------------------------------------------------------ single steps
@pytest.mark.parametrize("si", range(len(cases.STENCIL_SHAPES)))
@pytest.mark.parametrize("flavor", ["rho_scaled", "acoustic"])
@pytest.mark.parametrize("dn", ["f32", "f64"])
def test_fused_step_matches_reference(W, golden, si, flavor, dn):
    """propagate_step (fused kernel, coefficients recomputed from gamma)
    == reference apply_step on the reference's prepared coefficients."""
    g = golden("stencil")
    key = f"{flavor}_{dn}_{si}"
    shape = cases.STENCIL_SHAPES[si]
    gamma, u_prev, u_cur, dt, dx, consts = cases.stencil_inputs(shape, flavor, _dt(dn),
                                                                int(g[f"seed_{key}"]))
    grid = W.build_grid(shape, dx)
    if flavor == "rho_scaled":
        mat = W.MaterialModel.rho_scaled(gamma, grid, eps=1e-3, **consts)
    else:
        mat = W.MaterialModel.acoustic(gamma, grid, **consts)
    win = W.SolverWindow(u_prev=u_prev.copy(), u_cur=u_cur.copy(), u_next=np.zeros_like(u_cur))
    W.propagate_step(win, None, mat, dt)
    assert bits_equal(win.u_cur, g[f"step_{key}"])


@pytest.mark.parametrize("si", range(len(cases.STENCIL_SHAPES)))
@pytest.mark.parametrize("dn", ["f32", "f64"])
def test_dropin_apply_step(W, golden, si, dn):
    """wo_apply_step (literal kernels.apply_step drop-in) on the reference's
    own prepared arrays."""
    from paper_2509_15744_b200 import _native as N

    g = golden("stencil")
    key = f"rho_scaled_{dn}_{si}"
    shape = cases.STENCIL_SHAPES[si]
    _, u_prev, u_cur, _, _, _ = cases.stencil_inputs(shape, "rho_scaled", _dt(dn),
                                                     int(g[f"seed_{key}"]))
    wf = [np.ascontiguousarray(g[f"wf{a}_{key}"]) for a in range(len(shape))] + [None] * 3
    coef = np.ascontiguousarray(g[f"coef_{key}"])
    out = np.empty_like(u_cur)
    L = N.load(require_device=True)
    rc = L.wo_apply_step(len(shape), N.shape3(shape), out.itemsize, N.ptr(u_prev), N.ptr(u_cur),
                         N.ptr(wf[0]), N.ptr(wf[1]), N.ptr(wf[2]), N.ptr(coef), N.ptr(out), 0)
    assert rc == 0
    assert bits_equal(out, g[f"step_{key}"])


@pytest.mark.parametrize("si", range(len(cases.STENCIL_SHAPES)))
@pytest.mark.parametrize("dn", ["f32", "f64"])
def test_kernel_increment(W, golden, si, dn):
    gk = golden("kernel_increment")
    shape = cases.STENCIL_SHAPES[si]
    acc, wins, scal = cases.ki_inputs(shape, _dt(dn), 2000 + 10 * si + (dn == "f64"))
    grid = W.build_grid(shape, 1.0)
    # kernel_increment derives (cv, cg, 1/2dt, 1/2dx, sign*dt) from a material;
    # use the literal drop-in entry to feed the golden scalars directly
    from paper_2509_15744_b200 import _native as N

    L = N.load(require_device=True)
    for mode, wb in (("mixed", wins[3:]), ("self", wins[:3])):
        a = acc.copy()
        rc = L.wo_apply_kernel_increment(len(shape), N.shape3(shape), a.itemsize, N.ptr(a),
                                         *[N.ptr(w) for w in list(wins[:3]) + list(wb)],
                                         *[float(s) for s in scal], 0)
        assert rc == 0
        assert bits_equal(a, gk[f"{mode}_{dn}_{si}"]), mode
    del grid


# -------------------------------------------------------------- full sweeps
@pytest.mark.parametrize("name", ["fwi3d", "desk_fwi"])
@pytest.mark.parametrize("prec", ["double", "single"])
def test_gradient_superposed_bitexact(W, golden, name, prec):
    g = golden(name)
    c = cases.fwi3d_case() if name == "fwi3d" else cases.DESK
    problem, mat = product_fwi_problem(W, c, g["gamma_model"], g["measured"])
    res = W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=c["k"], precision=prec))
    assert res.gradient.dtype == g[f"sup_grad_{prec}"].dtype
    assert bits_equal(res.gradient, g[f"sup_grad_{prec}"])
    ref_cost = float(g[f"sup_cost_{prec}"])
    assert abs(res.cost - ref_cost) <= COST_RTOL * abs(ref_cost)
    # these grids do not tile into two-step CTAs: gamma, 2 levels, acc
    assert res.counter.peak_fields == 4


def test_buffer_counter_reports_device_fields(W):
    """BufferCounter reads the buffers the context really holds: 10 on the
    fast fp32 path (4 levels, acc, gamma, coef + 3 faces), 4 in the
    four-field mode (SPEC acceptance 5), with identical gradients."""
    rng = np.random.default_rng(4)
    shape, n_steps, dx = (10, 16, 64), 30, 1e-4
    dt = 0.45 * dx / 6000.0 / np.sqrt(3)
    grid = W.build_grid(shape, dx)
    mat = W.MaterialModel.rho_scaled(rng.uniform(0.4, 1.0, size=shape), grid, rho0=2700.0,
                                     c0=6000.0)
    src = W.SourceSpec(node=(4, 8, 30), amplitude=1e12, frequency=4e6, cycles=2)
    sens = [(8, j, 10) for j in (1, 7, 14)]
    problem = W.FwiProblem(grid=grid, time=W.TimeConfig(n_steps, dt), material=mat,
                           sources=[src], sensors=W.SensorArray(nodes=sens),
                           measured=rng.normal(scale=1e-10, size=(1, 3, n_steps)))
    fast = W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=1e13, precision="single"))
    four = W.gradient_superposed(problem, mat, W.SuperpositionConfig(
        k=1e13, precision="single", memory="four_fields"))
    assert fast.counter.peak_fields == 10
    assert four.counter.peak_fields == 4
    assert bits_equal(fast.gradient, four.gradient)


@pytest.mark.parametrize("prec", ["single", "double"])
def test_gradient_download_pinned_and_pageable(W, golden, prec):
    """The accumulator downloads identically into a page-locked array (one
    DMA), a fresh pageable array (staged copy) and the plan's pre-faulted
    output; a wrong output array is refused."""
    import torch

    from paper_2509_15744_b200 import engine
    from paper_2509_15744_b200 import gradients as G

    g = golden("fwi3d")
    c = cases.fwi3d_case()
    problem, mat = product_fwi_problem(W, c, g["gamma_model"], g["measured"])
    plan = G.SuperposedPlan(problem, mat, W.SuperpositionConfig(k=c["k"], precision=prec))
    plan.upload()
    plan.run()
    dt = np.float32 if prec == "single" else np.float64
    tdt = torch.float32 if prec == "single" else torch.float64
    pinned = torch.empty(problem.grid.shape, dtype=tdt, pin_memory=True).numpy()
    plan.ctx.get_accumulator(pinned)
    pageable = plan.ctx.get_accumulator()
    via_plan = plan.download()
    assert bits_equal(pinned, g[f"sup_grad_{prec}"])
    assert bits_equal(pageable, pinned) and bits_equal(via_plan, pinned)
    with pytest.raises(W.ConfigError):
        plan.ctx.get_accumulator(np.empty(problem.grid.shape, np.float16 if dt == np.float32
                                          else np.float32))


def test_closed_pooled_context_is_replaced(W, golden):
    """A user closing the cached context of a grid does not poison later
    evaluations on that grid; a closed handle raises DeviceError."""
    from paper_2509_15744_b200 import engine

    g = golden("fwi3d")
    c = cases.fwi3d_case()
    problem, mat = product_fwi_problem(W, c, g["gamma_model"], g["measured"])
    ctx = engine.get_context(problem.grid, np.float64)
    ctx.close()
    with pytest.raises(engine.DeviceError, match="closed"):
        ctx.set_material(mat, problem.time.dt)
    res = W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=c["k"], precision="double"))
    assert bits_equal(res.gradient, g["sup_grad_double"])


@pytest.mark.parametrize("prec", ["double", "single"])
def test_division_paths_agree(W, golden, prec):
    """The verified branch-free division path is active on the desk material
    and gives the same bits as the IEEE-intrinsic path."""
    from paper_2509_15744_b200 import engine

    g = golden("fwi3d")
    c = cases.fwi3d_case()
    problem, mat = product_fwi_problem(W, c, g["gamma_model"], g["measured"])
    ctx = engine.get_context(problem.grid, W.precision_dtype(prec))
    ctx.set_material(mat, problem.time.dt)
    assert ctx.fast_div_active()
    fast = W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=c["k"], precision=prec))
    try:
        ctx.set_fast_div(False)
        assert not ctx.fast_div_active()
        plan = W.gradients.SuperposedPlan(problem, mat, W.SuperpositionConfig(k=c["k"],
                                                                            precision=prec))
        plan.upload()
        ctx.set_fast_div(False)          # upload re-verified; force the precise path
        plan.run()
        slow = plan.download()
    finally:
        ctx.set_fast_div(True)
    assert bits_equal(fast.gradient, slow)
    assert bits_equal(slow, g[f"sup_grad_{prec}"])


@pytest.mark.parametrize("name", ["fwi3d", "desk_fwi"])
@pytest.mark.parametrize("prec", ["double", "single"])
def test_gradient_reference_bitexact(W, golden, name, prec):
    g = golden(name)
    c = cases.fwi3d_case() if name == "fwi3d" else cases.DESK
    problem, mat = product_fwi_problem(W, c, g["gamma_model"], g["measured"])
    res = W.gradient_reference(problem, mat, precision=prec)
    assert bits_equal(res.gradient, g[f"ref_grad_{prec}"])
    if prec == "double":
        ref_cost = float(g["ref_cost_double"])
        assert abs(res.cost - ref_cost) <= COST_RTOL * abs(ref_cost)


@pytest.mark.parametrize("name", ["fwi3d", "desk_fwi"])
def test_forward_cost(W, golden, name):
    g = golden(name)
    c = cases.fwi3d_case() if name == "fwi3d" else cases.DESK
    problem, mat = product_fwi_problem(W, c, g["gamma_model"], g["measured"])
    for prec in ("double", "single"):
        cost = W.forward_cost(problem, mat, precision=prec)
        ref = float(g[f"fcost_{prec}"])
        assert abs(cost - ref) <= COST_RTOL * abs(ref), prec


@pytest.mark.parametrize("name", ["fwi3d", "desk_fwi"])
@pytest.mark.parametrize("dn", ["f32", "f64"])
def test_run_forward_traces(W, golden, name, dn):
    g = golden(name)
    c = cases.fwi3d_case() if name == "fwi3d" else cases.DESK
    problem, mat = product_fwi_problem(W, c, g["gamma_model"], g["measured"])
    truth = mat.with_gamma(g["truth"])
    res = W.run_forward(truth, problem.time, problem.sources,
                        W.SensorArray(nodes=problem.sensors.nodes), dtype=_dt(dn))
    assert bits_equal(res.traces, g[f"fwd_traces_{dn}"])
    assert bits_equal(res.window.u_prev, g[f"fwd_uprev_{dn}"])
    assert bits_equal(res.window.u_cur, g[f"fwd_ucur_{dn}"])
    assert res.peak_abs == float(g[f"fwd_peak_{dn}"])


@pytest.mark.parametrize("name", ["fwi3d", "desk_fwi"])
def test_synthesize_measurements(W, golden, name):
    g = golden(name)
    c = cases.fwi3d_case() if name == "fwi3d" else cases.DESK
    problem, mat = product_fwi_problem(W, c, g["gamma_model"], None)
    measured = W.synthesize_measurements(mat.with_gamma(g["truth"]), problem, refine=c["refine"])
    assert bits_equal(measured, g["measured"])


def test_tato_design_chain(W, golden):
    g = golden("tato2d")
    c = cases.tato2d_case()
    problem = product_tato_problem(W, c)
    beta, g_tilde, g_bar = W.design_fields(problem, c["gamma_raw"], c["beta_iter"])
    assert beta == float(g["beta"])
    assert bits_equal(g_tilde, g["g_tilde"])            # sums are bit-exact
    assert np.max(np.abs(g_bar - g["g_bar"])) <= 1e-14    # tanh: a few ulp
    chain = W.chain_rule(g["ref_grad_double"], g["g_tilde"], beta, c["eta"], c["r_f"],
                         c["design_mask"])
    assert rel_l2(chain, g["chain"]) <= 1e-14


@pytest.mark.parametrize("prec", ["double", "single"])
def test_tato_gradients_bitexact(W, golden, prec):
    g = golden("tato2d")
    c = cases.tato2d_case()
    problem = product_tato_problem(W, c)
    mat = problem.material(g["g_bar"])
    res = W.gradient_superposed(problem, mat,
                                W.SuperpositionConfig(k=float(g["cal_k"]), precision=prec))
    assert bits_equal(res.gradient, g[f"sup_grad_{prec}"])
    ref_cost = float(g[f"sup_cost_{prec}"])
    assert abs(res.cost - ref_cost) <= COST_RTOL * abs(ref_cost)
    if prec == "double":
        r = W.gradient_reference(problem, mat)
        assert bits_equal(r.gradient, g["ref_grad_double"])


def test_calibrate_k_tato(W, golden):
    g = golden("tato2d")
    c = cases.tato2d_case()
    problem = product_tato_problem(W, c)
    cal = W.calibrate_k(problem, problem.material(g["g_bar"]), k_start=1e18)
    assert cal.k == float(g["cal_k"])
    rows = np.array(cal.rows)
    np.testing.assert_allclose(rows, g["cal_rows"], rtol=1e-6, atol=0)


# ------------------------------------------------------ oracle comparisons
@pytest.mark.parametrize("shape", [(40, 9, 70), (5, 64, 33), (130, 3, 3), (200,), (3, 257),
                                   (17, 13, 66), (6, 9, 130), (3, 64), (33, 4),
                                   (12, 16, 64), (9, 24, 128), (64, 128), (3, 8, 64)])
@pytest.mark.parametrize("prec", ["single", "double"])
def test_odd_shapes_vs_oracle(W, shape, prec):
    """Ragged tiles, tiny axes and chunk boundaries: bit-exact vs the oracle."""
    rng = np.random.default_rng(sum(shape))
    dx = 1e-4
    dt = 0.45 * dx / 6000.0 / np.sqrt(len(shape))
    gamma = rng.uniform(0.3, 1.0, size=shape)
    n_steps = 60
    src_node = tuple(s // 3 for s in shape)
    sens = [tuple((s * (q + 1)) // 4 for s in shape) for q in range(3)]
    sens = list(dict.fromkeys(sens))
    measured = rng.normal(scale=1e-10, size=(1, len(sens), n_steps))
    grid = W.build_grid(shape, dx)
    mat = W.MaterialModel.rho_scaled(gamma, grid, rho0=2700.0, c0=6000.0)
    src = W.SourceSpec(node=src_node, amplitude=1e12, frequency=4e6, cycles=2)
    problem = W.FwiProblem(grid=grid, time=W.TimeConfig(n_steps, dt), material=mat,
                           sources=[src], sensors=W.SensorArray(nodes=sens), measured=measured)
    res = W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=1e13, precision=prec))
    omat = O.Material("rho_scaled", gamma, dx, rho0=2700.0, c0=6000.0)
    support = np.array([grid.flat_index(n) for n in sens], dtype=np.int64)
    shots = [(O.Source(src_node, 1e12, 4e6, 2), O.FwiShot(support, measured[0], dt))]
    cost, grad, _ = O.gradient_superposed(omat, dt, n_steps, shots, 1e13, prec)
    assert bits_equal(res.gradient, grad)
    assert abs(res.cost - cost) <= COST_RTOL * abs(cost)


@pytest.mark.parametrize("prec", ["single", "double"])
def test_pair_and_scalar_kernels_agree(W, golden, prec):
    """Even last axis: the pair-vectorised kernel and the scalar kernel give
    identical bits (fwi3d has n2 = 26)."""
    from paper_2509_15744_b200 import engine

    g = golden("fwi3d")
    c = cases.fwi3d_case()
    problem, mat = product_fwi_problem(W, c, g["gamma_model"], g["measured"])
    cfg = W.SuperpositionConfig(k=c["k"], precision=prec)
    ctx = engine.get_context(problem.grid, W.precision_dtype(prec))
    try:
        ctx.set_pair_kernel(False)
        scalar = W.gradient_superposed(problem, mat, cfg).gradient
    finally:
        ctx.set_pair_kernel(True)
    pair = W.gradient_superposed(problem, mat, cfg).gradient
    assert bits_equal(pair, scalar)
    assert bits_equal(pair, g[f"sup_grad_{prec}"])


@pytest.mark.parametrize("prec", ["single", "double"])
def test_tma_pair_scalar_kernels_agree(W, prec):
    """A grid of whole 64x8 tiles runs the TMA pipeline; it must match the
    pair and scalar kernels and the oracle bit for bit (sensor plane and a
    source on tile edges, random heterogeneous gamma)."""
    from paper_2509_15744_b200 import engine

    shape, dx, n_steps = (20, 16, 128), 1e-4, 90
    dt = 0.45 * dx / 6000.0 / np.sqrt(3)
    rng = np.random.default_rng(5)
    gamma = rng.uniform(0.2, 1.0, size=shape)
    grid = W.build_grid(shape, dx)
    mat = W.MaterialModel.rho_scaled(gamma, grid, rho0=2700.0, c0=6000.0)
    src = W.SourceSpec(node=(4, 8, 63), amplitude=1e12, frequency=5e6, cycles=2)
    sens = [(15, j, k) for j in (0, 7, 8, 15) for k in (0, 1, 63, 64, 127)]
    measured = rng.normal(scale=1e-10, size=(1, len(sens), n_steps))
    problem = W.FwiProblem(grid=grid, time=W.TimeConfig(n_steps, dt), material=mat,
                           sources=[src], sensors=W.SensorArray(nodes=sens), measured=measured)
    cfg = W.SuperpositionConfig(k=1e13, precision=prec)
    ctx = engine.get_context(grid, W.precision_dtype(prec))
    out = {}
    for name, tma, pair in (("tma4", 1, True), ("pair", 0, True),
                            ("scalar", 0, False)):
        ctx.set_tma_kernel(tma)
        ctx.set_pair_kernel(pair)
        out[name] = W.gradient_superposed(problem, mat, cfg)
    ctx.set_tma_kernel(True)
    ctx.set_pair_kernel(True)
    omat = O.Material("rho_scaled", gamma, dx, rho0=2700.0, c0=6000.0)
    support = np.array([grid.flat_index(n) for n in sens], dtype=np.int64)
    shots = [(O.Source(src.node, 1e12, 5e6, 2), O.FwiShot(support, measured[0], dt))]
    cost, grad, _ = O.gradient_superposed(omat, dt, n_steps, shots, 1e13, prec)
    for name, res in out.items():
        assert bits_equal(res.gradient, grad), name
        assert abs(res.cost - cost) <= COST_RTOL * abs(cost), name


def test_instability_reported_like_reference(W):
    """A Courant number above the limit blows up; the device raises the same
    SolverInstabilityError (step, max) as the oracle."""
    shape, dx = (40, 40), 1e-4
    dt = 1.2 * dx / 6000.0
    grid = W.build_grid(shape, dx)
    gamma = np.ones(shape)
    mat = W.MaterialModel.rho_scaled(gamma, grid, rho0=2700.0, c0=6000.0)
    src = W.SourceSpec(node=(20, 20), amplitude=1e12, frequency=3e6, cycles=2)
    n_steps = 400
    with pytest.raises(W.SolverInstabilityError) as ei:
        W.run_forward(mat, W.TimeConfig(n_steps, dt), [src], None)
    omat = O.Material("rho_scaled", gamma, dx, rho0=2700.0, c0=6000.0)
    with pytest.raises(O.OracleInstability) as eo:
        O.run_forward(omat, dt, n_steps, [O.Source((20, 20), 1e12, 3e6, 2)])
    assert ei.value.step == eo.value.step
    assert ei.value.max_abs == eo.value.max_abs or (
        np.isnan(ei.value.max_abs) and np.isnan(eo.value.max_abs))


def test_time_reversal_roundtrip(W):
    """SPEC acceptance 2: forward 500 steps then backward replay recovers the
    zero initial state (fp64, 101x101, burst source)."""
    shape, dx, n_steps = (101, 101), 2e-4, 500
    dt = 0.5 * dx / 6000.0
    grid = W.build_grid(shape, dx)
    mat = W.MaterialModel.rho_scaled(np.ones(shape), grid, rho0=2700.0, c0=6000.0)
    src = W.SourceSpec(node=(50, 50), amplitude=1e12, frequency=1.5e6, cycles=2)
    time = W.TimeConfig(n_steps, dt)
    fwd = W.run_forward(mat, time, [src])
    peak = fwd.peak_abs
    idx = np.array([grid.flat_index(src.node)])
    back = W.run_backward(mat, time, fwd.window,
                          lambda n: (idx, np.array([W.burst_amplitude(n * dt, src)])))
    assert np.max(np.abs(back.u_cur)) <= 1e-10 * peak


def test_superposed_matches_reference_engine(W, golden):
    """SPEC agreement contract: superposed vs full-storage < 5% rel. MSE."""
    g = golden("desk_fwi")
    c = cases.DESK
    problem, mat = product_fwi_problem(W, c, g["gamma_model"], g["measured"])
    sup = W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=c["k"]))
    ref = W.gradient_reference(problem, mat)
    assert W.rel_mse(sup.gradient, ref.gradient) < 0.05


# ------------------------------------------ run_forward history / on_step
@pytest.mark.parametrize("shape", [(37, 29), (12, 16, 64)])
@pytest.mark.parametrize("dn", ["f32", "f64"])
@pytest.mark.parametrize("fused", [True, False])
def test_run_forward_full_history_and_on_step(W, shape, dn, fused, monkeypatch):
    """recorder_mode='full_history' and on_step (solver.py:306-336): every
    level u^0..u^N and every callback (n, u^{n+1}) bit-exact vs the oracle's
    run_forward history, through the fused recording sweep (levels read back
    in chunks) and through the per-step fallback."""
    from paper_2509_15744_b200 import solver

    if not fused:   # more nodes than a recording sweep injects in-kernel: per step
        monkeypatch.setattr(solver, "MAX_KERNEL_SOURCES", 0)
    monkeypatch.setattr(solver, "HISTORY_CHUNK_BYTES", 7 * int(np.prod(shape)) * 8)
    dx, n_steps = 2e-4, 57
    dt = 0.45 * dx / 6000.0 / np.sqrt(len(shape))
    grid = W.build_grid(shape, dx)
    rng = np.random.default_rng(len(shape) + n_steps)
    gamma = rng.uniform(0.3, 1.0, size=shape)
    mat = W.MaterialModel.rho_scaled(gamma, grid, rho0=2700.0, c0=6000.0)
    node = tuple(n // 2 for n in shape)
    src = W.SourceSpec(node=node, amplitude=1e12, frequency=3e6, cycles=2)
    sens = [tuple(max(0, c - 3) for c in node), tuple(n - 1 for n in shape)]
    time = W.TimeConfig(n_steps, dt)
    seen = []
    res = W.run_forward(mat, time, [src], W.SensorArray(nodes=sens),
                        recorder_mode="full_history", dtype=_dt(dn),
                        on_step=lambda n, u: seen.append((n, u.copy())))
    omat = O.Material("rho_scaled", gamma, dx, rho0=2700.0, c0=6000.0)
    sidx = np.array([grid.flat_index(s) for s in sens], dtype=np.int64)
    up, uc, tr, hist, _ = O.run_forward(omat, dt, n_steps, [O.Source(node, 1e12, 3e6, 2)], sidx,
                                        dtype=_dt(dn), full_history=True)
    assert bits_equal(res.history, hist)
    assert bits_equal(res.traces, tr)
    assert bits_equal(res.window.u_cur, uc) and bits_equal(res.window.u_prev, up)
    assert [n for n, _ in seen] == list(range(1, n_steps))
    for n, u in seen:
        assert bits_equal(u, hist[n + 1])
    # on_step alone (no host history): levels straight from the device history
    seen2 = []
    W.run_forward(mat, time, [src], None, dtype=_dt(dn),
                  on_step=lambda n, u: seen2.append((n, u.copy())))
    assert len(seen2) == n_steps - 1
    for n, u in seen2:
        assert bits_equal(u, hist[n + 1])
