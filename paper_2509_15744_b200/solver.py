"""Forward/backward propagation API (waveopt.solver) on the device.

Reference: /root/reference/pkg/src/waveopt/solver.py.  The time loops run
inside the native sweeps (engine.DeviceGrid); this module keeps the
reference's call signatures, result types and error behaviour.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import engine
from .engine import ResourceBudgetError, SolverInstabilityError, source_amplitude_table
from .grids import ConfigError, Grid, MaterialModel, SensorArray, SourceSpec, TimeConfig

STABILITY_CHECK_INTERVAL = 50            # solver.py:29
STABILITY_GROWTH_FACTOR = 1e6            # solver.py:30
DEFAULT_HISTORY_BUDGET = 4 * 1024**3     # solver.py:31
MAX_KERNEL_SOURCES = 8                   # source nodes a recording sweep injects in-kernel
DEVICE_HISTORY_CAP = 16 * 1024**3        # on_step without full_history: device levels recorded
HISTORY_CHUNK_BYTES = 256 * 1024**2      # on_step levels read back per host copy

__all__ = [
    "ResourceBudgetError", "SolverInstabilityError", "SolverWindow", "ForwardResult",
    "burst_amplitude", "apply_ghost_material", "propagate_step", "run_forward",
    "run_backward", "injection_scale", "STABILITY_CHECK_INTERVAL", "DEFAULT_HISTORY_BUDGET",
]


def burst_amplitude(t, src: SourceSpec):
    """psi0 sin(wt) sin^2(wt/(2 n_c)) on [0, 2 pi n_c/w], else 0 (solver.py:48-54)."""
    if t < 0 or t > src.duration:
        return 0.0
    w = src.omega
    return src.amplitude * math.sin(w * t) * math.sin(w * t / (2 * src.cycles)) ** 2


def apply_ghost_material(material: MaterialModel):
    """Edge-padded indicator (inspection only; solver.py:57-63)."""
    return np.pad(material.gamma, 1, mode="edge")


@dataclass
class SolverWindow:
    """Three host-visible levels (solver.py:128-151).  Device sweeps keep
    their own window; this type backs propagate_step / run_backward."""

    u_prev: np.ndarray
    u_cur: np.ndarray
    u_next: np.ndarray
    step: int = 1

    @classmethod
    def zeros(cls, grid: Grid, dtype=np.float64, allocate=np.zeros):
        return cls(u_prev=allocate(grid.shape, dtype=dtype), u_cur=allocate(grid.shape, dtype=dtype),
                   u_next=allocate(grid.shape, dtype=dtype))

    def rotate(self):
        self.u_prev, self.u_cur, self.u_next = self.u_cur, self.u_next, self.u_prev
        self.step += 1

    def swap_direction(self):
        self.u_prev, self.u_cur = self.u_cur, self.u_prev


@dataclass
class ForwardResult:
    window: SolverWindow
    traces: np.ndarray | None
    history: np.ndarray | None
    peak_abs: float


def source_injections(sources, grid: Grid, t):
    """(flat indices, fp64 values) of the nodal sources at time t, the force
    form propagate_step / run_backward take (solver.py:267-270)."""
    idx = np.array([grid.flat_index(s.node) for s in sources], dtype=np.int64)
    values = np.array([burst_amplitude(t, s) for s in sources])
    return idx, values


def injection_scale(sources, material: MaterialModel, dt, dtype):
    """max |psi0| * force_coef[node] over the sources (solver.py:273-279)."""
    scale = 0.0
    for s in sources:
        fc = engine.force_coef_at(material, dt, dtype, s.node)
        scale = max(scale, abs(s.amplitude) * float(fc))
    return scale


def _check(m, step, scale=0.0, detail=""):
    if not math.isfinite(m):
        raise SolverInstabilityError(step, m, detail=detail)
    if scale > 0.0 and m > STABILITY_GROWTH_FACTOR * scale:
        raise SolverInstabilityError(step, m, detail=f"exceeds 1e6 x scale {scale:g}")
    return m


def _dx_matches(dx, material):
    if dx is not None and not math.isclose(dx, material.grid.dx):
        raise ConfigError(f"dx {dx} does not match grid spacing {material.grid.dx}")


def propagate_step(window: SolverWindow, force, material: MaterialModel, dt,
                   dx=None) -> SolverWindow:
    """One update u^{n+1} from (u^{n-1}, u^n) on the device; advances the
    window (solver.py:189-202).  force: dense field, (flat_idx, values) or None."""
    _dx_matches(dx, material)
    ctx = engine.get_context(material.grid, window.u_cur.dtype)
    ctx.set_material(material, dt)
    ctx.set_window(window.u_prev, window.u_cur)
    m = ctx.step(force, want_max=True)
    up, uc = ctx.get_window()
    window.u_next[...] = uc
    _check(m, window.step)
    window.rotate()
    return window


def run_forward(material: MaterialModel, time: TimeConfig, sources,
                sensors: SensorArray | None = None, recorder_mode="traces_only",
                history_budget=DEFAULT_HISTORY_BUDGET, dtype=np.float64,
                on_step=None) -> ForwardResult:
    """N steps from u^0 = u^1 = 0 with trace recording (solver.py:282-340).

    Trace entry j records level u^j (entry 0 stays 0).  One native sweep;
    with recorder_mode='full_history' or an on_step callback the sweep also
    records every level on the device and the levels come back in bulk
    afterwards (the callback runs after the sweep, in step order; a sweep that
    fails its stability check raises before any callback).  More than 8
    source nodes, or an on_step history beyond DEVICE_HISTORY_CAP, step
    level by level with one read-back per step."""
    grid = material.grid
    n_steps = time.n_steps
    for s in sources:
        s.validate_on(grid)
    if sensors is not None:
        sensors.validate_on(grid)
    dtype = np.dtype(dtype)
    if recorder_mode not in ("traces_only", "full_history"):
        raise ConfigError(f"unknown recorder_mode {recorder_mode!r}")
    history = None
    if recorder_mode == "full_history":
        need = (n_steps + 1) * grid.n_nodes * dtype.itemsize
        if need > history_budget:
            raise ResourceBudgetError(
                f"full history needs {need} bytes ({n_steps + 1} levels of "
                f"{grid.n_nodes} nodes) > budget {history_budget}")
        history = np.zeros((n_steps + 1,) + grid.shape, dtype=dtype)

    ctx = engine.get_context(grid, dtype)
    ctx.set_material(material, time.dt)
    ctx.reset_window()
    scale = injection_scale(sources, material, time.dt, dtype) * n_steps
    src_flat = np.array([grid.flat_index(s.node) for s in sources], dtype=np.int64)
    amp = source_amplitude_table(sources, time.dt, n_steps)
    traces = None
    sensor_idx = sensors.flat_indices(grid) if sensors is not None else None

    level_bytes = grid.n_nodes * dtype.itemsize
    fused_levels = (len(set(src_flat.tolist())) <= MAX_KERNEL_SOURCES and
                    (history is not None or (n_steps + 1) * level_bytes <= DEVICE_HISTORY_CAP))
    if (history is None and on_step is None) or fused_levels:
        # one native sweep; with a history / callback the levels are recorded
        # on the device during the sweep (WO_FWD_HISTORY) and read back in
        # bulk afterwards instead of one step launch + one D2H per step
        if sensor_idx is not None:
            order = ctx.set_support(sensor_idx)
        else:
            ctx.clear_support()
        record = history is not None or on_step is not None
        try:
            peak = ctx.sweep_forward(n_steps, src_flat, amp, accumulate=False, dt=time.dt,
                                     scale=scale, history=record)
            if sensor_idx is not None:
                store = ctx.get_store(n_steps)            # [N][n_sup], device order
                traces = np.empty((len(sensor_idx), n_steps), dtype=dtype)
                traces[order] = store.T
            if history is not None:
                ctx.get_history(0, history)
            if on_step is not None:
                chunk = max(1, min(n_steps - 1, HISTORY_CHUNK_BYTES // level_bytes))
                for n0 in range(1, n_steps, chunk):
                    k = min(chunk, n_steps - n0)
                    levels = (history[n0 + 1:n0 + 1 + k] if history is not None else
                              ctx.get_history(n0 + 1, np.empty((k,) + grid.shape, dtype)))
                    for i in range(k):
                        on_step(n0 + i, levels[i])
        finally:
            if record:
                ctx.free_history()
        up, uc = ctx.get_window()
    else:
        traces = (np.zeros((len(sensor_idx), n_steps), dtype=dtype)
                  if sensor_idx is not None else None)
        uc = np.zeros(grid.shape, dtype)        # u^1 = 0 after the reset
        peak = 0.0
        for n in range(1, n_steps):
            if traces is not None:
                traces[:, n] = uc.reshape(-1)[sensor_idx]
            force = (src_flat, amp[:, n]) if len(sources) else None
            check = n % STABILITY_CHECK_INTERVAL == 0 or n == n_steps - 1
            m = ctx.step(force, want_max=check)
            uc = ctx.get_field("u_cur").reshape(grid.shape)   # one D2H per step
            if check:
                peak = max(peak, _check(m, n + 1, scale))
            if history is not None:
                history[n + 1] = uc
            if on_step is not None:
                on_step(n, uc)
        up, uc = ctx.get_window()
    window = SolverWindow(u_prev=up, u_cur=uc, u_next=np.zeros_like(uc), step=n_steps)
    if sensors is not None:
        sensors.traces = traces
    return ForwardResult(window=window, traces=traces, history=history, peak_abs=peak)


def run_backward(material: MaterialModel, time: TimeConfig, end_window: SolverWindow,
                 forces_by_step, on_step=None, copy=True) -> SolverWindow:
    """Reversed stepping from (u^{N-1}, u^N) to u^0 (solver.py:343-372)."""
    grid = material.grid
    dtype = end_window.u_cur.dtype
    ctx = engine.get_context(grid, dtype)
    ctx.set_material(material, time.dt)
    # the 'two steps back' slot takes u^N, the centre u^{N-1}
    ctx.set_window(end_window.u_cur, end_window.u_prev)
    for n in range(time.n_steps - 1, 0, -1):
        check = n % STABILITY_CHECK_INTERVAL == 0 or n == 1
        m = ctx.step(forces_by_step(n), want_max=check)
        if check:
            _check(m, n - 1)
        if on_step is not None:
            on_step(n, ctx.get_field("u_cur").reshape(grid.shape))
    up, uc = ctx.get_window()
    if copy:
        window = SolverWindow(u_prev=up, u_cur=uc, u_next=np.empty_like(uc))
    else:
        window = end_window
        window.u_prev[...] = up
        window.u_cur[...] = uc
    window.step = 0
    return window
