"""TEST INFRASTRUCTURE ONLY — CPU oracle for the superposed-adjoint hot path.

A restatement of the reference algorithm (waveopt, /root/reference/pkg/src/
waveopt) with the same operation order, used by tests/, by
``__graft_entry__.smoke()`` and by bench.py's cpu_baseline / ``--impl
reference`` leg as the checker and the CPU comparator.  The product package
``paper_2509_15744_b200`` never imports this module.

* Per-cell arithmetic (the reference's Numba kernels, kernels.py:18-128) is in
  ``wave_oracle.c``, compiled by ``oracle/Makefile`` into
  ``oracle/_build/libwave_oracle.so`` (OpenMP over axis 0; bitwise independent
  of the thread count).
* Host-side numpy work (material preparation, sparse injection, sensor
  gathers, shot costs) is restated here with the same numpy expressions, so
  dtype promotion and rounding follow the reference exactly.

Pinned: tests/test_oracle_golden.py checks every function here bit for bit
against tests/golden/*.npz, which tests/golden/make_golden.py produced by
running the reference itself.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libwave_oracle.so")
_lib = None

RHO_SCALED = "rho_scaled"
ACOUSTIC = "acoustic"
STABILITY_CHECK_INTERVAL = 50          # solver.py:29
STABILITY_GROWTH_FACTOR = 1e6          # solver.py:30


class OracleInstability(RuntimeError):
    """Mirror of SolverInstabilityError (solver.py:34-41)."""

    def __init__(self, step, max_abs, detail=""):
        self.step = step
        self.max_abs = max_abs
        super().__init__(f"unstable field at step {step}: max|u| = {max_abs:g}"
                         + (f" ({detail})" if detail else ""))


def build():
    """Compile wave_oracle.c (gcc, -ffp-contract=off, OpenMP)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        vp, i64p = ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)
        L.or_apply_step.argtypes = [ctypes.c_int, ctypes.c_int, i64p] + [vp] * 7
        L.or_apply_step.restype = ctypes.c_int
        L.or_apply_kernel_increment.argtypes = (
            [ctypes.c_int, ctypes.c_int, i64p] + [vp] * 7 + [ctypes.c_double] * 5)
        L.or_apply_kernel_increment.restype = ctypes.c_int
        L.or_max_abs.argtypes = [ctypes.c_int, ctypes.c_int64, vp]
        L.or_max_abs.restype = ctypes.c_double
        L.or_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def num_threads():
    return int(lib().or_num_threads())


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _shape(a):
    return (ctypes.c_int64 * 3)(*(list(a.shape) + [1] * (3 - a.ndim)))


# ---------------------------------------------------------------- kernels.py
def apply_step(u_prev, u_cur, face_weights, coef, out):
    """kernels.py:136-139."""
    for a in (u_prev, u_cur, coef, out, *face_weights):
        assert a.flags.c_contiguous and a.dtype == u_cur.dtype
    wf = list(face_weights) + [None] * (3 - len(face_weights))
    rc = lib().or_apply_step(u_cur.dtype.itemsize, u_cur.ndim, _shape(u_cur),
                             _ptr(u_prev), _ptr(u_cur), _ptr(wf[0]), _ptr(wf[1]),
                             _ptr(wf[2]), _ptr(coef), _ptr(out))
    assert rc == 0


def apply_kernel_increment(acc, win_a, win_b, cv, cg, inv2dt, inv2dx, sdt):
    """kernels.py:142-152 (scalars cast to the accumulator dtype in C)."""
    a_old, a_mid, a_new = win_a
    b_old, b_mid, b_new = win_b
    rc = lib().or_apply_kernel_increment(
        acc.dtype.itemsize, acc.ndim, _shape(acc), _ptr(acc),
        _ptr(a_old), _ptr(a_mid), _ptr(a_new), _ptr(b_old), _ptr(b_mid), _ptr(b_new),
        float(cv), float(cg), float(inv2dt), float(inv2dx), float(sdt))
    assert rc == 0


def max_abs(u):
    return float(lib().or_max_abs(u.dtype.itemsize, u.size, _ptr(u)))


# ------------------------------------------------------------------ solver.py
@dataclass
class Material:
    """Flavor, indicator and constants (grids.py:103-169)."""

    flavor: str
    gamma: np.ndarray
    dx: float
    rho0: float = 0.0
    c0: float = 0.0
    rho1: float = 0.0
    kappa1: float = 0.0
    rho2: float = 0.0
    kappa2: float = 0.0


@dataclass
class Source:
    """Sine burst at one node (grids.py:172-199)."""

    node: tuple
    amplitude: float
    frequency: float
    cycles: int = 2

    @property
    def omega(self):
        return 2.0 * math.pi * self.frequency

    @property
    def duration(self):
        return 2.0 * math.pi * self.cycles / self.omega


def burst_amplitude(t, src):
    """solver.py:48-54."""
    if t < 0 or t > src.duration:
        return 0.0
    w = src.omega
    return src.amplitude * math.sin(w * t) * math.sin(w * t / (2 * src.cycles)) ** 2


@dataclass
class Prepared:
    dtype: np.dtype
    coef: np.ndarray
    face_weights: tuple
    force_coef: np.ndarray


def interpolate_material_fields(mat, g):
    """grids.py:247-254."""
    inv_rho = 1.0 / mat.rho1 + g * (1.0 / mat.rho2 - 1.0 / mat.rho1)
    inv_kappa = 1.0 / mat.kappa1 + g * (1.0 / mat.kappa2 - 1.0 / mat.kappa1)
    return inv_rho, inv_kappa


def prepare_material(mat: Material, dt, dtype):
    """solver.py:89-125."""
    dtype = np.dtype(dtype)
    dt = float(dt)
    gamma = np.ascontiguousarray(mat.gamma, dtype=dtype)
    if mat.flavor == RHO_SCALED:
        m = dtype.type(1.0) / gamma
        r2 = dtype.type((mat.c0 * dt / mat.dx) ** 2)
        coef = dtype.type(2.0) * r2 / gamma
        force_coef = dtype.type(dt * dt) / (dtype.type(mat.rho0) * gamma)
    else:
        inv_rho, inv_kappa = interpolate_material_fields(mat, gamma)
        inv_rho = inv_rho.astype(dtype, copy=False)
        inv_kappa = inv_kappa.astype(dtype, copy=False)
        m = dtype.type(1.0) / inv_rho
        kappa = dtype.type(1.0) / inv_kappa
        s2 = dtype.type((dt / mat.dx) ** 2)
        coef = dtype.type(2.0) * kappa * s2
        force_coef = kappa * dtype.type(dt * dt)
    weights = []
    for axis in range(gamma.ndim):
        lo = [slice(None)] * gamma.ndim
        hi = [slice(None)] * gamma.ndim
        lo[axis] = slice(None, -1)
        hi[axis] = slice(1, None)
        weights.append(np.ascontiguousarray(dtype.type(1.0) / (m[tuple(lo)] + m[tuple(hi)])))
    return Prepared(dtype, np.ascontiguousarray(coef), tuple(weights),
                    np.ascontiguousarray(force_coef))


class Window:
    """solver.py:128-151 (three levels, pointer rotation)."""

    def __init__(self, shape, dtype):
        self.u_prev = np.zeros(shape, dtype)
        self.u_cur = np.zeros(shape, dtype)
        self.u_next = np.zeros(shape, dtype)

    def rotate(self):
        self.u_prev, self.u_cur, self.u_next = self.u_cur, self.u_next, self.u_prev

    def swap_direction(self):
        self.u_prev, self.u_cur = self.u_cur, self.u_prev


def add_force(out, prep, force):
    """solver.py:154-170."""
    if force is None:
        return
    if isinstance(force, np.ndarray):
        out += prep.force_coef * force.astype(out.dtype, copy=False)
        return
    idx, values = force
    if len(idx) == 0:
        return
    flat = out.reshape(-1)
    flat[idx] += prep.force_coef.reshape(-1)[idx] * np.asarray(values, dtype=out.dtype)


def step_window(w, prep, force=None):
    """solver.py:173-177."""
    apply_step(w.u_prev, w.u_cur, prep.face_weights, prep.coef, w.u_next)
    add_force(w.u_next, prep, force)


def check_finite(values, step, scale=0.0):
    """solver.py:180-186."""
    m = max_abs(values)
    if not math.isfinite(m):
        raise OracleInstability(step, m)
    if scale > 0.0 and m > STABILITY_GROWTH_FACTOR * scale:
        raise OracleInstability(step, m, detail=f"exceeds 1e6 x scale {scale:g}")
    return m


def flat_index(shape, node):
    return int(np.ravel_multi_index(tuple(int(i) for i in node), shape))


# --------------------------------------------------------------------- shots
class FwiShot:
    """fwi.py:48-63."""

    def __init__(self, support_idx, measured, dt):
        self.support_idx = np.asarray(support_idx, dtype=np.int64)
        self.measured = np.asarray(measured, dtype=np.float64)
        self.dt = dt

    def adjoint_values(self, u_support, n):
        return -(np.asarray(u_support, dtype=np.float64) - self.measured[:, n])

    def cost_increment(self, u_support, n):
        r = np.asarray(u_support, dtype=np.float64) - self.measured[:, n]
        return 0.5 * float(np.dot(r, r)) * self.dt


class TatoShot:
    """tato.py:143-163."""

    def __init__(self, support_idx, area, dt, dx, ndim, mode):
        self.support_idx = np.asarray(support_idx, dtype=np.int64)
        self.area = area
        self.dt = dt
        self.cell = dx**ndim
        self.sign = 1.0 if mode == "suppress" else -1.0

    def adjoint_values(self, u_support, n):
        return (-self.sign * 2.0 * self.cell / self.area) * np.asarray(
            u_support, dtype=np.float64)

    def cost_increment(self, u_support, n):
        u = np.asarray(u_support, dtype=np.float64)
        return self.sign * float(np.dot(u, u)) * self.cell * self.dt / self.area


# ------------------------------------------------------------------ gradients
def kernel_coefficients(mat):
    """gradients.py:117-129."""
    if mat.flavor == RHO_SCALED:
        return -mat.rho0, mat.rho0 * mat.c0**2
    dk = 1.0 / mat.kappa2 - 1.0 / mat.kappa1
    dr = 1.0 / mat.rho2 - 1.0 / mat.rho1
    return -dk, dr


def injection_scale(sources, prep, shape):
    """solver.py:273-279."""
    fc = prep.force_coef.reshape(-1)
    scale = 0.0
    for s in sources:
        scale = max(scale, abs(s.amplitude) * float(fc[flat_index(shape, s.node)]))
    return scale


def forward_pass(prep, dt, n_steps, source, shot, window, accum, coeffs, adj_store,
                 history=None, trace_out=None):
    """gradients.py:214-250 (trace_out optionally records u^n on the support)."""
    shape = window.u_cur.shape
    dx_inv2 = coeffs[2]
    support = shot.support_idx
    src_idx = np.array([flat_index(shape, source.node)], dtype=np.int64)
    cv, cg = coeffs[0], coeffs[1]
    inv2dt, inv2dx = 1.0 / (2.0 * dt), dx_inv2
    scale = injection_scale([source], prep, shape) * n_steps
    cost = shot.cost_increment(np.zeros(len(support)), 0)
    peak = 0.0
    if history is not None:
        history[0] = window.u_prev
        history[1] = window.u_cur
    for n in range(1, n_steps):
        u_sup = window.u_cur.reshape(-1)[support]
        if trace_out is not None:
            trace_out[n] = u_sup
        cost += shot.cost_increment(u_sup, n)
        adj_store[n] = shot.adjoint_values(u_sup, n)
        force = (src_idx, np.array([burst_amplitude(n * dt, source)]))
        step_window(window, prep, force)
        if accum is not None:
            win = (window.u_prev, window.u_cur, window.u_next)
            apply_kernel_increment(accum, win, win, cv, cg, inv2dt, inv2dx, -dt)
        if history is not None:
            history[n + 1] = window.u_next
        if n % STABILITY_CHECK_INTERVAL == 0 or n == n_steps - 1:
            peak = max(peak, check_finite(window.u_next, n + 1, scale))
        window.rotate()
    return cost


def superposed_backward(prep, dt, n_steps, source, shot, window, accum, coeffs,
                        adj_store, k):
    """gradients.py:253-281."""
    shape = window.u_cur.shape
    support = shot.support_idx
    src_idx = np.array([flat_index(shape, source.node)], dtype=np.int64)
    cv, cg = coeffs[0], coeffs[1]
    inv2dt, inv2dx = 1.0 / (2.0 * dt), coeffs[2]
    adj_store *= adj_store.dtype.type(k)
    window.swap_direction()
    flat_fc = prep.force_coef.reshape(-1)
    for n in range(n_steps - 1, 0, -1):
        step_window(window, prep, (src_idx, np.array([burst_amplitude(n * dt, source)])))
        out = window.u_next.reshape(-1)
        out[support] += flat_fc[support] * adj_store[n]
        win = (window.u_next, window.u_cur, window.u_prev)
        apply_kernel_increment(accum, win, win, cv, cg, inv2dt, inv2dx, dt)
        if n % STABILITY_CHECK_INTERVAL == 0 or n == 1:
            try:
                check_finite(window.u_next, n - 1)
            except OracleInstability as exc:
                raise OracleInstability(
                    exc.step, exc.max_abs,
                    detail="superposed pass diverged; raise k if underflowing, "
                           "lower k if the approximation blows up") from None
        window.rotate()


def _coeffs(mat, dx):
    cv, cg = kernel_coefficients(mat)
    return (cv, cg, 1.0 / (2.0 * dx))


def gradient_superposed(mat: Material, dt, n_steps, shots, k, precision="double"):
    """gradients.py:284-326.  shots: list of (Source, FwiShot|TatoShot).

    Returns (cost, gradient, adj_stores) — adj_stores are the per-shot
    compact adjoint stores after the backward pass (i.e. scaled by k)."""
    dtype = np.dtype(np.float32 if precision == "single" else np.float64)
    shape = mat.gamma.shape
    coeffs = _coeffs(mat, mat.dx)
    prep = prepare_material(mat, dt, dtype)
    accum = np.zeros(shape, dtype)
    window = Window(shape, dtype)
    total = 0.0
    stores = []
    for source, shot in shots:
        adj = np.zeros((n_steps, len(shot.support_idx)), dtype=dtype)
        for level in (window.u_prev, window.u_cur):
            level[...] = 0
        total += forward_pass(prep, dt, n_steps, source, shot, window, accum, coeffs, adj)
        superposed_backward(prep, dt, n_steps, source, shot, window, accum, coeffs, adj, k)
        stores.append(adj)
    accum /= dtype.type(2.0 * k)
    return total, accum, stores


def gradient_reference(mat: Material, dt, n_steps, shots, precision="double"):
    """gradients.py:329-391 (full-history adjoint)."""
    dtype = np.dtype(np.float32 if precision == "single" else np.float64)
    shape = mat.gamma.shape
    coeffs = _coeffs(mat, mat.dx)
    cv, cg, inv2dx = coeffs
    inv2dt = 1.0 / (2.0 * dt)
    prep = prepare_material(mat, dt, dtype)
    history = np.zeros((n_steps + 1,) + shape, dtype=dtype)
    accum = np.zeros(shape, dtype)
    window = Window(shape, dtype)
    adjoint = Window(shape, dtype)
    total = 0.0
    for source, shot in shots:
        adj = np.zeros((n_steps, len(shot.support_idx)), dtype=dtype)
        for level in (window.u_prev, window.u_cur):
            level[...] = 0
        total += forward_pass(prep, dt, n_steps, source, shot, window, None, coeffs, adj,
                              history=history)
        for level in (adjoint.u_prev, adjoint.u_cur, adjoint.u_next):
            level[...] = 0
        flat_fc = prep.force_coef.reshape(-1)
        support = shot.support_idx
        for n in range(n_steps - 1, 0, -1):
            step_window(adjoint, prep)
            out = adjoint.u_next.reshape(-1)
            out[support] += flat_fc[support] * adj[n]
            fwd_win = (history[n - 1], history[n], history[n + 1])
            adj_win = (adjoint.u_next, adjoint.u_cur, adjoint.u_prev)
            apply_kernel_increment(accum, fwd_win, adj_win, cv, cg, inv2dt, inv2dx, dt)
            if n % STABILITY_CHECK_INTERVAL == 0 or n == 1:
                check_finite(adjoint.u_next, n - 1)
            adjoint.rotate()
    return total, accum


def forward_cost(mat: Material, dt, n_steps, shots, precision="double"):
    """gradients.py:394-414."""
    dtype = np.dtype(np.float32 if precision == "single" else np.float64)
    shape = mat.gamma.shape
    prep = prepare_material(mat, dt, dtype)
    total = 0.0
    for source, shot in shots:
        window = Window(shape, dtype)
        support = shot.support_idx
        src_idx = np.array([flat_index(shape, source.node)], dtype=np.int64)
        scale = injection_scale([source], prep, shape) * n_steps
        cost = shot.cost_increment(np.zeros(len(support)), 0)
        for n in range(1, n_steps):
            cost += shot.cost_increment(window.u_cur.reshape(-1)[support], n)
            force = (src_idx, np.array([burst_amplitude(n * dt, source)]))
            step_window(window, prep, force)
            if n % STABILITY_CHECK_INTERVAL == 0 or n == n_steps - 1:
                check_finite(window.u_next, n + 1, scale)
            window.rotate()
        total += cost
    return total


def run_forward(mat: Material, dt, n_steps, sources, sensor_idx=None, dtype=np.float64,
                full_history=False):
    """solver.py:282-340.  Returns (u_prev, u_cur, traces, history, peak)."""
    dtype = np.dtype(dtype)
    shape = mat.gamma.shape
    prep = prepare_material(mat, dt, dtype)
    history = np.zeros((n_steps + 1,) + shape, dtype=dtype) if full_history else None
    traces = (np.zeros((len(sensor_idx), n_steps), dtype=dtype)
              if sensor_idx is not None else None)
    window = Window(shape, dtype)
    scale = injection_scale(sources, prep, shape) * n_steps
    peak = 0.0
    for n in range(1, n_steps):
        if sensor_idx is not None:
            traces[:, n] = window.u_cur.reshape(-1)[sensor_idx]
        if sources:
            idx = np.array([flat_index(shape, s.node) for s in sources], dtype=np.int64)
            vals = np.array([burst_amplitude(n * dt, s) for s in sources])
            force = (idx, vals)
        else:
            force = None
        step_window(window, prep, force)
        if n % STABILITY_CHECK_INTERVAL == 0 or n == n_steps - 1:
            peak = max(peak, check_finite(window.u_next, n + 1, scale))
        if history is not None:
            history[n + 1] = window.u_next
        window.rotate()
    return window.u_prev, window.u_cur, traces, history, peak


def run_backward(mat: Material, dt, n_steps, u_prev_end, u_cur_end, forces_by_step):
    """solver.py:343-372 (copy=True form).  Returns (u_prev, u_cur) at the end
    — u_cur = u^0."""
    dtype = u_cur_end.dtype
    prep = prepare_material(mat, dt, dtype)
    window = Window(u_cur_end.shape, dtype)
    window.u_prev = u_cur_end.copy()
    window.u_cur = u_prev_end.copy()
    for n in range(n_steps - 1, 0, -1):
        step_window(window, prep, forces_by_step(n))
        if n % STABILITY_CHECK_INTERVAL == 0 or n == 1:
            check_finite(window.u_next, n - 1)
        window.rotate()
    return window.u_prev, window.u_cur


# ------------------------------------------------------- TATO design chain
def filter_kernel(r_f, ndim):
    """tato.py:59-68 — linear-decay weights r_f - |x| on |x| < r_f."""
    reach = int(math.ceil(r_f))
    axes = [np.arange(-reach, reach + 1)] * ndim
    grids = np.meshgrid(*axes, indexing="ij")
    dist = np.sqrt(sum(g.astype(float) ** 2 for g in grids))
    return np.where(dist < r_f, r_f - dist, 0.0)


def _masked_correlate(values, mask, r_f):
    """tato.py:71-75."""
    from scipy import ndimage

    kernel = filter_kernel(float(r_f), values.ndim)
    num = ndimage.correlate(np.where(mask, values, 0.0), kernel, mode="constant")
    den = ndimage.correlate(mask.astype(float), kernel, mode="constant")
    return num, den


def density_filter(gamma, r_f, design_mask=None):
    """tato.py:78-94."""
    gamma = np.asarray(gamma, dtype=float)
    mask = (np.ones_like(gamma, dtype=bool) if design_mask is None
            else np.asarray(design_mask, dtype=bool))
    num, den = _masked_correlate(gamma, mask, r_f)
    out = gamma.copy()
    out[mask] = num[mask] / den[mask]
    return out


def heaviside_project(gamma_tilde, beta, eta=0.5):
    """tato.py:97-108."""
    g = np.asarray(gamma_tilde, dtype=float)
    denom = math.tanh(beta * eta) + math.tanh(beta * (1.0 - eta))
    out = (math.tanh(beta * eta) + np.tanh(beta * (g - eta))) / denom
    return np.clip(out, 0.0, 1.0)


def project_derivative(gamma_tilde, beta, eta=0.5):
    """tato.py:111-115."""
    g = np.asarray(gamma_tilde, dtype=float)
    denom = math.tanh(beta * eta) + math.tanh(beta * (1.0 - eta))
    return beta / (denom * np.cosh(beta * (g - eta)) ** 2)


def beta_schedule(iteration):
    """tato.py:118-122."""
    return 1.1 ** (int(iteration) // 5)


def chain_rule(dcost_dbar, gamma_tilde, beta, eta, r_f, design_mask=None):
    """tato.py:124-140."""
    from scipy import ndimage

    g = np.asarray(dcost_dbar, dtype=float)
    mask = (np.ones_like(g, dtype=bool) if design_mask is None
            else np.asarray(design_mask, dtype=bool))
    inner = np.where(mask, g * project_derivative(gamma_tilde, beta, eta), 0.0)
    _, den = _masked_correlate(inner, mask, r_f)
    ratio = np.zeros_like(inner)
    ratio[mask] = inner[mask] / den[mask]
    out = ndimage.correlate(ratio, filter_kernel(float(r_f), g.ndim), mode="constant")
    out[~mask] = 0.0
    return out


def design_fields(gamma_raw, iteration, r_f, eta, design_mask):
    """tato.py:221-227."""
    beta = beta_schedule(iteration)
    g_tilde = density_filter(gamma_raw, r_f, design_mask)
    g_bar = heaviside_project(g_tilde, beta, eta)
    g_bar = np.where(design_mask, g_bar, 0.0)
    return beta, g_tilde, g_bar
