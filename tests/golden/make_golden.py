"""Generate the golden fixtures by running the REFERENCE itself.

Run in the dev container only (it needs /root/reference):

    python tests/golden/make_golden.py

It imports waveopt from /root/reference/pkg/src under the alias
``waveopt_ref`` (Numba cache redirected to /tmp so nothing is written into
the read-only reference tree), evaluates the cases of tests/golden/cases.py
and writes tests/golden/*.npz.  The fixtures are committed; the GPU box never
reads /root/reference.
"""

from __future__ import annotations

import importlib.util
import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_waveopt_ref")
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import cases  # noqa: E402

REF_SRC = "/root/reference/pkg/src/waveopt"


def load_reference():
    spec = importlib.util.spec_from_file_location(
        "waveopt_ref", os.path.join(REF_SRC, "__init__.py"),
        submodule_search_locations=[REF_SRC])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["waveopt_ref"] = mod
    spec.loader.exec_module(mod)
    import importlib as _il

    mod.config = _il.import_module("waveopt_ref.config")
    return mod


def dtname(dt):
    return "f32" if np.dtype(dt) == np.float32 else "f64"


def gen_stencil(W):
    out = {}
    for si, shape in enumerate(cases.STENCIL_SHAPES):
        grid = W.build_grid(shape, 1e-3)
        for flavor in ("rho_scaled", "acoustic"):
            for dtype in (np.float32, np.float64):
                seed = 1000 + 10 * si + (flavor == "acoustic") * 3 + (dtype == np.float64)
                gamma, u_prev, u_cur, dt, dx, consts = cases.stencil_inputs(
                    shape, flavor, dtype, seed)
                if flavor == "rho_scaled":
                    mat = W.MaterialModel.rho_scaled(gamma, grid, eps=1e-3, **consts)
                else:
                    mat = W.MaterialModel.acoustic(gamma, grid, **consts)
                prep = W.solver.prepare_material(mat, dt, dtype=dtype)
                res = np.empty_like(u_cur)
                W.kernels.apply_step(u_prev, u_cur, prep.face_weights, prep.coef, res)
                key = f"{flavor}_{dtname(dtype)}_{si}"
                out[f"step_{key}"] = res
                out[f"coef_{key}"] = prep.coef
                out[f"fc_{key}"] = prep.force_coef
                for a, w in enumerate(prep.face_weights):
                    out[f"wf{a}_{key}"] = w
                out[f"seed_{key}"] = np.int64(seed)
    return out


def gen_ki(W):
    out = {}
    for si, shape in enumerate(cases.STENCIL_SHAPES):
        for dtype in (np.float32, np.float64):
            seed = 2000 + 10 * si + (dtype == np.float64)
            acc, wins, scal = cases.ki_inputs(shape, dtype, seed)
            a_mixed = acc.copy()
            W.kernels.apply_kernel_increment(a_mixed, tuple(wins[:3]), tuple(wins[3:]), *scal)
            a_self = acc.copy()
            W.kernels.apply_kernel_increment(a_self, tuple(wins[:3]), tuple(wins[:3]), *scal)
            out[f"mixed_{dtname(dtype)}_{si}"] = a_mixed
            out[f"self_{dtname(dtype)}_{si}"] = a_self
    return out


def make_fwi_problem(W, c, gamma_model, measured=None):
    grid = W.build_grid(c["shape"], c["dx"])
    time_cfg = W.TimeConfig(n_steps=c["n_steps"], dt=c["dt"])
    mat = W.MaterialModel.rho_scaled(gamma_model, grid, rho0=c["rho0"], c0=c["c0"],
                                     eps=c["eps"])
    sources = [W.SourceSpec(node=n, amplitude=a, frequency=f, cycles=cy)
               for n, a, f, cy in c["sources"]]
    if "ring" in c:
        nodes = cases.ring_nodes(c["shape"], *c["ring"])
    else:
        nodes = c["sensors"]
    sensors = W.SensorArray(nodes=nodes)
    problem = W.FwiProblem(grid=grid, time=time_cfg, material=mat, sources=sources,
                           sensors=sensors, measured=measured)
    return problem, mat


def gen_fwi(W, c):
    out = {}
    shape = c["shape"]
    if "truth_disks" in c:
        gamma_model = np.ones(shape)
        truth = cases.disk_gamma(shape, c["truth_disks"], c["eps"])
    else:
        gamma_model = c["gamma"]
        truth = gamma_model.copy()
        idx = np.indices(shape)
        for center, radius in c["truth_spheres"]:
            d2 = sum((idx[a] - center[a]) ** 2 for a in range(len(shape)))
            truth[d2 <= radius**2] = c["eps"]
    problem, mat = make_fwi_problem(W, c, gamma_model)
    t0 = time.time()
    measured = W.synthesize_measurements(mat.with_gamma(truth), problem, refine=c["refine"])
    print(f"  {c['name']}: synthesize {time.time() - t0:.1f}s")
    problem.measured = measured
    out["measured"] = measured
    out["gamma_model"] = np.asarray(gamma_model, dtype=np.float64)
    out["truth"] = truth
    out["sensor_idx"] = problem.sensors.flat_indices(problem.grid)
    for prec in ("double", "single"):
        t0 = time.time()
        res = W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=c["k"], precision=prec))
        print(f"  {c['name']}: superposed {prec} {time.time() - t0:.1f}s")
        out[f"sup_grad_{prec}"] = res.gradient
        out[f"sup_cost_{prec}"] = np.float64(res.cost)
        out[f"sup_peak_fields_{prec}"] = np.int64(res.counter.peak_fields)
    res = W.gradient_reference(problem, mat, precision="double")
    out["ref_grad_double"] = res.gradient
    out["ref_cost_double"] = np.float64(res.cost)
    res = W.gradient_reference(problem, mat, precision="single")
    out["ref_grad_single"] = res.gradient
    out["fcost_double"] = np.float64(W.forward_cost(problem, mat, precision="double"))
    out["fcost_single"] = np.float64(W.forward_cost(problem, mat, precision="single"))
    # multi-source forward run with trace recording (solver.py:282-340)
    for dtype in (np.float32, np.float64):
        fr = W.run_forward(mat.with_gamma(truth), problem.time, problem.sources,
                           W.SensorArray(nodes=problem.sensors.nodes), dtype=dtype)
        out[f"fwd_traces_{dtname(dtype)}"] = fr.traces
        out[f"fwd_uprev_{dtname(dtype)}"] = fr.window.u_prev
        out[f"fwd_ucur_{dtname(dtype)}"] = fr.window.u_cur
        out[f"fwd_peak_{dtname(dtype)}"] = np.float64(fr.peak_abs)
    return out


def make_tato_problem(W, c):
    grid = W.build_grid(c["shape"], c["dx"])
    time_cfg = W.TimeConfig(n_steps=c["n_steps"], dt=c["dt"])
    node, amp, freq, cyc = c["source"]
    src = W.SourceSpec(node=node, amplitude=amp, frequency=freq, cycles=cyc)
    return W.TatoProblem(grid=grid, time=time_cfg, source=src,
                         design_mask=c["design_mask"], objective_mask=c["objective_mask"],
                         rho1=c["rho1"], kappa1=c["kappa1"], rho2=c["rho2"],
                         kappa2=c["kappa2"], r_f=c["r_f"], eta=c["eta"], mode=c["mode"])


def gen_tato(W, c):
    out = {}
    problem = make_tato_problem(W, c)
    beta, g_tilde, g_bar = W.tato.design_fields(problem, c["gamma_raw"], c["beta_iter"])
    out["beta"] = np.float64(beta)
    out["g_tilde"] = g_tilde
    out["g_bar"] = g_bar
    mat = problem.material(g_bar)
    cal = W.calibrate_k(problem, mat, k_start=1e18)
    out["cal_k"] = np.float64(cal.k)
    out["cal_rows"] = np.array(cal.rows, dtype=np.float64)
    k = cal.k
    for prec in ("double", "single"):
        res = W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=k, precision=prec))
        out[f"sup_grad_{prec}"] = res.gradient
        out[f"sup_cost_{prec}"] = np.float64(res.cost)
    res = W.gradient_reference(problem, mat, precision="double")
    out["ref_grad_double"] = res.gradient
    out["ref_cost_double"] = np.float64(res.cost)
    out["chain"] = W.chain_rule(np.asarray(res.gradient, dtype=np.float64), g_tilde, beta,
                                problem.eta, problem.r_f, problem.design_mask)
    out["fcost_double"] = np.float64(W.forward_cost(problem, mat, precision="double"))
    return out


def _log_arrays(out, key, log):
    out[f"{key}_cost"] = np.array([r["cost"] for r in log], dtype=np.float64)
    out[f"{key}_gnorm"] = np.array([r["grad_norm"] for r in log], dtype=np.float64)
    if "beta" in log[0]:
        out[f"{key}_beta"] = np.array([r["beta"] for r in log], dtype=np.float64)


def gen_loops(W):
    """Optimisation loops of the reference: 3 iterations of
    invert on configs/fwi_desk.toml (fwi.py:178-238), with and without a
    frozen mask, and of optimize_design on the tato2d case (tato.py:238-304):
    parameters after every iteration and the cost / gradient-norm logs."""
    out = {}
    g = np.load(os.path.join(HERE, "desk_fwi.npz"))
    c = cases.DESK
    problem, _ = make_fwi_problem(W, c, g["gamma_model"], g["measured"])
    for prec in ("double", "single"):
        t0 = time.time()
        res = W.invert(problem, method="superposed", k=c["k"], iterations=3, precision=prec,
                       snapshot_every=1)
        print(f"  invert {prec} {time.time() - t0:.1f}s")
        out[f"inv_hist_{prec}"] = np.array(res.gamma_history)
        _log_arrays(out, f"inv_{prec}", res.log)
    mask = cases.desk_mask(c["shape"])
    problem.mask = mask
    res = W.invert(problem, method="superposed", k=c["k"], iterations=2, precision="double",
                   snapshot_every=1)
    out["inv_mask"] = mask
    out["invm_hist_double"] = np.array(res.gamma_history)
    _log_arrays(out, "invm_double", res.log)
    res = W.invert(problem, method="reference", iterations=2, precision="double",
                   snapshot_every=1)
    out["invr_hist_double"] = np.array(res.gamma_history)
    _log_arrays(out, "invr_double", res.log)

    t = np.load(os.path.join(HERE, "tato2d.npz"))
    ct = cases.tato2d_case()
    tp = make_tato_problem(W, ct)
    for prec in ("double", "single"):
        t0 = time.time()
        res = W.optimize_design(tp, method="superposed", k=float(t["cal_k"]), iterations=3,
                                precision=prec, snapshot_every=1)
        print(f"  optimize_design {prec} {time.time() - t0:.1f}s")
        out[f"des_raw_{prec}"] = res.gamma_raw
        out[f"des_hist_{prec}"] = np.array(res.design_history)
        _log_arrays(out, f"des_{prec}", res.log)
    return out


def gen_config_desk(W):
    """configs/fwi_desk.toml through the reference's own config path
    (config.py:74-215: parse, assemble, synthesize on the refine = 2 grid)
    and 3 iterations of its invert with the config's optimizer (alpha 0.02,
    Adam eps 1e-40: real updates, unlike the FwiProblem defaults) at k = 1e13.
    The TOML bytes are stored with the outputs (the GPU box has no
    /root/reference)."""
    import tomllib

    import waveopt_ref.config as RC

    path = "/root/reference/pkg/configs/fwi_desk.toml"
    raw_bytes = open(path, "rb").read()
    cfg = tomllib.loads(raw_bytes.decode())
    rc = RC.parse_config(cfg)
    problem, truth = RC.build_fwi(cfg, rc)
    out = {"toml": np.frombuffer(raw_bytes, dtype=np.uint8), "measured": problem.measured,
           "truth_gamma": np.asarray(truth.gamma, dtype=np.float64),
           "sensor_idx": problem.sensors.flat_indices(problem.grid)}
    for prec in ("double", "single"):
        t0 = time.time()
        res = W.invert(problem, method="superposed", k=1e13, iterations=3, precision=prec,
                       snapshot_every=1)
        print(f"  config invert {prec} {time.time() - t0:.1f}s")
        out[f"hist_{prec}"] = np.array(res.gamma_history)
        _log_arrays(out, f"inv_{prec}", res.log)
    return out


def gen_solver(W):
    """run_forward with co-located sources (solver.py:154-170: numpy fancy
    `+=` keeps the LAST duplicate) and run_backward (solver.py:343-372), from
    the forward's end window and from a random end window, 3D and 2D."""
    out = {}
    for tag, c in (("3d", cases.fwi3d_case()), ("2d", cases.solver2d_case())):
        grid = W.build_grid(c["shape"], c["dx"])
        tcfg = W.TimeConfig(n_steps=c["n_steps"], dt=c["dt"])
        mat = W.MaterialModel.rho_scaled(c["gamma"], grid, rho0=c["rho0"], c0=c["c0"],
                                         eps=c["eps"])
        srcs = [W.SourceSpec(node=n, amplitude=a, frequency=f, cycles=cy)
                for n, a, f, cy in cases.colocated_sources(c)]
        sens = W.SensorArray(nodes=cases.solver_sensors(c))
        for dtype in (np.float32, np.float64):
            key = f"{tag}_{dtname(dtype)}"
            fr = W.run_forward(mat, tcfg, srcs, sens, dtype=dtype)
            out[f"fwd_traces_{key}"] = fr.traces
            out[f"fwd_uprev_{key}"] = fr.window.u_prev
            out[f"fwd_ucur_{key}"] = fr.window.u_cur
            forces = lambda n: W.solver.source_injections(srcs, grid, n * c["dt"])  # noqa: E731
            wb = W.run_backward(mat, tcfg, fr.window, forces)
            out[f"bwd_uprev_{key}"] = wb.u_prev
            out[f"bwd_ucur_{key}"] = wb.u_cur
            rng = np.random.default_rng(77 + dtype().itemsize)
            end = W.SolverWindow(u_prev=rng.normal(size=c["shape"]).astype(dtype),
                                 u_cur=rng.normal(size=c["shape"]).astype(dtype),
                                 u_next=np.zeros(c["shape"], dtype))
            out[f"rnd_uprev_in_{key}"] = end.u_prev.copy()
            out[f"rnd_ucur_in_{key}"] = end.u_cur.copy()
            wr = W.run_backward(mat, tcfg, end, forces)
            out[f"rnd_uprev_{key}"] = wr.u_prev
            out[f"rnd_ucur_{key}"] = wr.u_cur
    return out


def gen_kats(W):
    """SPEC KATs, evaluated on the reference."""
    out = {}
    src = W.SourceSpec(node=(1, 1), amplitude=1.0, frequency=1.0, cycles=2)
    t = (np.pi / 2) / src.omega
    out["burst_quarter"] = np.float64(W.burst_amplitude(t, src))
    grid = W.build_grid((5, 5), 1e-3)
    mat = W.MaterialModel.rho_scaled(np.full((5, 5), 0.5), grid, rho0=2700.0, c0=6000.0)
    win = W.SolverWindow.zeros(grid)
    W.propagate_step(win, (np.array([12]), np.array([1.0])), mat, 1e-8)
    out["unit_force"] = win.u_cur.copy()
    out["filter_spike"] = np.float64(
        W.density_filter(np.pad(np.ones((1, 1)), 4), 1.5, np.ones((9, 9), bool))[4, 4])
    out["heaviside_075"] = np.float64(W.heaviside_project(0.75, 1.0, 0.5))
    out["beta_0_5_10"] = np.array([W.beta_schedule(i) for i in (0, 5, 10)])
    return out


def gen_io(W):
    """Field dumps and raw traces written by the reference's io.py (byte
    fixtures for the first-axis-fastest layout and the sidecars)."""
    import tempfile

    import waveopt_ref.io as RIO

    rng = np.random.default_rng(21)
    out = {}
    cases_io = [
        ("f32_3d", rng.normal(size=(5, 4, 3)).astype(np.float32), (5, 4, 3), 2e-4,
         dict(dt=3e-9, step_index=17, extra={"what": "acc"})),
        ("f64_2d", rng.normal(size=(6, 7)), (6, 7), 0.5, {}),
        ("f32_1d", rng.normal(size=(9,)).astype(np.float32), (9,), 1.0, dict(step_index=0)),
    ]
    with tempfile.TemporaryDirectory() as tmp:
        for name, vals, shape, dx, kw in cases_io:
            grid = W.build_grid(shape, dx)
            path = RIO.dump_field(os.path.join(tmp, name), vals, grid, **kw)
            out[f"{name}_values"] = vals
            out[f"{name}_bin"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
            out[f"{name}_json"] = np.array(open(str(path)[:-4] + ".json").read())
        traces = rng.normal(size=(3, 11))
        path = RIO.save_traces_raw(os.path.join(tmp, "traces"), traces, 2.5e-9)
        out["traces_values"] = traces
        out["traces_bin"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
        out["traces_json"] = np.array(open(str(path)[:-4] + ".json").read())
    return out


def main():
    W = load_reference()
    import waveopt_ref.kernels  # noqa: F401
    import waveopt_ref.solver  # noqa: F401
    import waveopt_ref.tato  # noqa: F401

    W.kernels = sys.modules["waveopt_ref.kernels"]
    W.solver = sys.modules["waveopt_ref.solver"]
    W.tato = sys.modules["waveopt_ref.tato"]
    jobs = [
        ("stencil", lambda: gen_stencil(W)),
        ("kernel_increment", lambda: gen_ki(W)),
        ("kats", lambda: gen_kats(W)),
        ("fwi3d", lambda: gen_fwi(W, cases.fwi3d_case())),
        ("tato2d", lambda: gen_tato(W, cases.tato2d_case())),
        ("desk_fwi", lambda: gen_fwi(W, cases.DESK)),
        ("io_dumps", lambda: gen_io(W)),
        ("loops", lambda: gen_loops(W)),
        ("solver", lambda: gen_solver(W)),
        ("config_desk", lambda: gen_config_desk(W)),
    ]
    only = set(sys.argv[1:])
    for name, fn in jobs:
        if only and name not in only:
            continue
        t0 = time.time()
        data = fn()
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **data)
        print(f"{name}: {len(data)} arrays, {os.path.getsize(path) / 1e3:.0f} kB, "
              f"{time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
