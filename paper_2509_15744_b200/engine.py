"""Device context: one grid at one dtype on one GPU (wraps ``wo_ctx``).

This is the only module that talks to the native library; the API modules
(solver, gradients, fwi, tato) describe WHAT to run in the reference's terms
and call the sweep-level entry points here.
"""

from __future__ import annotations

import ctypes
import math
from collections import OrderedDict

import numpy as np

from . import _native as N
from .grids import RHO_SCALED, ConfigError, Grid, MaterialModel


class SolverInstabilityError(RuntimeError):
    """Blow-up or NaN/Inf during time integration (CLI exit code 2; solver.py:34-41)."""

    def __init__(self, step, max_abs, detail=""):
        self.step = step
        self.max_abs = max_abs
        msg = f"unstable field at step {step}: max|u| = {max_abs:g}"
        super().__init__(msg + (f" ({detail})" if detail else ""))


class ResourceBudgetError(RuntimeError):
    """Allocation exceeds the configured budget (CLI exit code 3; solver.py:44-45)."""


class DeviceError(RuntimeError):
    """CUDA / driver failure inside the native library."""


def _raise(ctx_handle, rc, what):
    L = N.load()
    msg = L.wo_last_error(ctx_handle)
    msg = msg.decode() if msg else ""
    text = f"{what}: {msg}"
    if rc == N.WO_ERR_CONFIG:
        raise ConfigError(text)
    if rc == N.WO_ERR_BUDGET:
        raise ResourceBudgetError(text)
    raise DeviceError(text)


def source_amplitude_table(sources, dt, n_steps):
    """[n_src][N] fp64 table of burst_amplitude(n*dt) (solver.py:48-54),
    evaluated with math.sin exactly like the reference."""
    out = np.zeros((len(sources), n_steps), dtype=np.float64)
    for s, src in enumerate(sources):
        w = src.omega
        dur = src.duration
        amp = src.amplitude
        half = 2 * src.cycles
        for n in range(n_steps):
            t = n * dt
            if t < 0 or t > dur:
                continue
            out[s, n] = amp * math.sin(w * t) * math.sin(w * t / half) ** 2
    return out


def force_coef_at(material: MaterialModel, dt, dtype, node):
    """force_coef[node] of prepare_material (solver.py:98,110), as a T scalar."""
    T = np.dtype(dtype).type
    g = T(material.gamma[tuple(node)])
    if material.flavor == RHO_SCALED:
        return T(dt * dt) / (T(material.rho0) * g)
    ik = 1.0 / material.kappa1 + g * (1.0 / material.kappa2 - 1.0 / material.kappa1)
    return (T(1.0) / T(ik)) * T(dt * dt)


def material_ratio2(material: MaterialModel, dt, dx):
    """The squared ratio the reference evaluates with ** (solver.py:96,108)."""
    if material.flavor == RHO_SCALED:
        return (material.c0 * dt / dx) ** 2
    return (dt / dx) ** 2


def kernel_coefficients(material: MaterialModel):
    """(velocity, gradient) kernel coefficients (gradients.py:117-129)."""
    if material.flavor == RHO_SCALED:
        return -material.rho0, material.rho0 * material.c0**2
    dk = 1.0 / material.kappa2 - 1.0 / material.kappa1
    dr = 1.0 / material.rho2 - 1.0 / material.rho1
    return -dk, dr


class _SlabShape:
    """Minimal grid-like record for a slab's local planes."""

    def __init__(self, shape, dx):
        self.shape = tuple(int(n) for n in shape)
        self.dx = float(dx)
        self.ndim = len(self.shape)
        self.n_nodes = int(np.prod(self.shape))


class DeviceGrid:
    """Device buffers + sweeps for one grid at one dtype (include/waveb200.h)."""

    def __init__(self, grid: Grid, dtype, device=0, slab=None):
        """slab=(i_begin, i_end): a slab of a 3D grid along axis 0 (global
        planes [i_begin, i_end) plus ghost planes at interior faces)."""
        self.L = N.load(require_device=True)
        self.dtype = np.dtype(dtype)
        self.device = device
        h = ctypes.c_void_p()
        if slab is None:
            self.global_grid = grid
            self.i_begin, self.i_end = 0, grid.shape[0]
            self.grid = grid
            rc = self.L.wo_create(ctypes.byref(h), grid.ndim, N.shape3(grid.shape),
                                  float(grid.dx), self.dtype.itemsize, device)
        else:
            if grid.ndim != 3:
                raise ConfigError("slab decomposition needs a 3D grid")
            self.global_grid = grid
            self.i_begin, self.i_end = int(slab[0]), int(slab[1])
            # local view: the slab's own planes (Grid needs >= 3 nodes per axis,
            # so keep the dataclass-free shape separately)
            self.grid = _SlabShape((self.i_end - self.i_begin,) + grid.shape[1:], grid.dx)
            rc = self.L.wo_create_slab(ctypes.byref(h), N.shape3(grid.shape), self.i_begin,
                                       self.i_end, float(grid.dx), self.dtype.itemsize, device)
        if rc:
            _raise(None, rc, "wo_create")
        self.h = h
        self._support_key = None
        self.n_sup = 0
        self.claim = None      # the plan / batch whose material and support are loaded

    @property
    def is_slab(self):
        return self.grid is not self.global_grid

    @property
    def alloc_range(self):
        """Global planes [lo, hi) held on the device: own planes plus up to two
        ghost planes per neighbour (wo_create_slab)."""
        n0 = self.global_grid.shape[0]
        if not self.is_slab:
            return 0, n0
        return self.i_begin - min(2, self.i_begin), self.i_end + min(2, n0 - self.i_end)

    # --------------------------------------------------------------- basics
    def close(self):
        if getattr(self, "h", None):
            self.L.wo_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ck(self, rc, what):
        if rc:
            if not self.h:
                raise DeviceError(f"{what}: context is closed")
            _raise(self.h, rc, what)

    def _field(self, a):
        a = np.ascontiguousarray(a, dtype=self.dtype)
        if a.shape != self.grid.shape:
            raise ConfigError(f"field shape {a.shape} != grid {self.grid.shape}")
        return a

    def set_material(self, material: MaterialModel, dt, gamma_local=None):
        """Material constants of `material` and its gamma (fp64, cast on the
        device).  gamma_local: this context's planes of gamma (own + ghost
        planes, alloc_range) as a C-contiguous fp64 array, used instead of
        slicing material.gamma (e.g. a pinned host copy of a slab)."""
        if material.grid.shape != self.global_grid.shape:
            raise ConfigError("material lives on a different grid")
        self.claim = None      # loaded state changed: a plan that cached it re-uploads
        flavor = N.WO_RHO_SCALED if material.flavor == RHO_SCALED else N.WO_ACOUSTIC
        lo, hi = self.alloc_range
        if gamma_local is not None:
            gamma = gamma_local
            if (gamma.dtype != np.float64 or not gamma.flags.c_contiguous or
                    gamma.shape != (hi - lo,) + tuple(self.global_grid.shape[1:])):
                raise ConfigError("gamma_local must be this context's planes, C-order fp64")
        elif self.is_slab:   # own planes plus the ghost planes (solver.py:94 per slab)
            gamma = np.ascontiguousarray(material.gamma[lo:hi], dtype=np.float64)
        else:
            gamma = np.ascontiguousarray(material.gamma, dtype=np.float64)
        ratio2 = material_ratio2(material, float(dt), self.grid.dx)
        self._ck(self.L.wo_set_material(self.h, flavor, N.ptr(gamma), float(material.rho0),
                                        float(material.rho1), float(material.kappa1),
                                        float(material.rho2), float(material.kappa2),
                                        float(dt), float(ratio2)), "wo_set_material")
        cv, cg = kernel_coefficients(material)
        self._ck(self.L.wo_set_kernel_coefficients(
            self.h, float(cv), float(cg), 1.0 / (2.0 * float(dt)), 1.0 / (2.0 * self.grid.dx)),
            "wo_set_kernel_coefficients")

    def set_support(self, flat_idx):
        """Set the support; returns the permutation sorting flat_idx (device
        order = increasing flat index)."""
        flat_idx = np.asarray(flat_idx, dtype=np.int64)
        order = np.argsort(flat_idx, kind="stable")
        srt = np.ascontiguousarray(flat_idx[order])
        key = srt.tobytes()
        if key != self._support_key:
            self._ck(self.L.wo_set_support(self.h, len(srt), N.ptr(srt)), "wo_set_support")
            self._support_key = key
        self.n_sup = len(srt)
        return order

    def clear_support(self):
        self.set_support(np.zeros(0, dtype=np.int64))

    def reset_window(self):
        self._ck(self.L.wo_reset_window(self.h), "wo_reset_window")

    def set_window(self, u_prev, u_cur):
        self._ck(self.L.wo_set_window(self.h, N.ptr(self._field(u_prev)),
                                      N.ptr(self._field(u_cur))), "wo_set_window")

    def get_window(self):
        up = np.empty(self.grid.shape, self.dtype)
        uc = np.empty(self.grid.shape, self.dtype)
        self._ck(self.L.wo_get_window(self.h, N.ptr(up), N.ptr(uc)), "wo_get_window")
        return up, uc

    def get_field(self, which, first_axis_fastest=False):
        """A device field ("gamma", "u_prev", "u_cur", "acc") on the host; with
        first_axis_fastest the flat bytes of the reference's dumps
        (io.py:29-52), reordered on the device."""
        code = {"gamma": N.WO_FIELD_GAMMA, "u_prev": N.WO_FIELD_UPREV,
                "u_cur": N.WO_FIELD_UCUR, "acc": N.WO_FIELD_ACC}[which]
        out = np.empty(int(np.prod(self.grid.shape)), self.dtype)
        self._ck(self.L.wo_get_field(self.h, code, int(bool(first_axis_fastest)), N.ptr(out)),
                 "wo_get_field")
        return out if first_axis_fastest else out.reshape(self.grid.shape)

    # ------------------------------------------- device optimiser (8f-3)
    def opt_init(self, params, frozen=None, zero_frozen_grad=False, lo=0.0, hi=1.0,
                 frozen_value=0.0, alpha=1e-3, beta1=0.9, beta2=0.999, eps=1e-8):
        p = np.ascontiguousarray(params, dtype=np.float64)
        fz = None if frozen is None else np.ascontiguousarray(frozen, dtype=np.uint8)
        self._ck(self.L.wo_opt_init(self.h, N.ptr(p), N.ptr(fz), int(bool(zero_frozen_grad)),
                                    float(lo), float(hi), float(frozen_value), float(alpha),
                                    float(beta1), float(beta2), float(eps)), "wo_opt_init")

    def opt_step(self, t):
        """Adam step t from the accumulator's gradient; returns its L2 norm."""
        norm = ctypes.c_double(0.0)
        self._ck(self.L.wo_opt_step(self.h, int(t), ctypes.byref(norm)), "wo_opt_step")
        return norm.value

    def opt_get(self):
        out = np.empty(self.grid.shape, np.float64)
        self._ck(self.L.wo_opt_get(self.h, N.ptr(out)), "wo_opt_get")
        return out

    def design_setup(self, mask, offsets, weights):
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
        offs = np.ascontiguousarray(offsets, dtype=np.int32)
        ws = np.ascontiguousarray(weights, dtype=np.float64)
        self._ck(self.L.wo_design_setup(self.h, N.ptr(m), len(ws), N.ptr(offs), N.ptr(ws)),
                 "wo_design_setup")

    def design_material(self, beta, eta, t_be, denom):
        self._ck(self.L.wo_design_material(self.h, float(beta), float(eta), float(t_be),
                                           float(denom)), "wo_design_material")

    def design_gradient(self, beta, eta, denom):
        self._ck(self.L.wo_design_gradient(self.h, float(beta), float(eta), float(denom)),
                 "wo_design_gradient")

    def design_get(self, which):
        out = np.empty(self.grid.shape, np.float64)
        code = {"g_tilde": 0, "g_bar": 1, "grad": 2}[which]
        self._ck(self.L.wo_design_get(self.h, code, N.ptr(out)), "wo_design_get")
        return out

    def snapshot(self, op, n_steps=0):
        """Save / restore / free the post-forward device state (wo_snapshot)."""
        code = {"save": N.WO_SNAP_SAVE, "restore": N.WO_SNAP_RESTORE, "free": N.WO_SNAP_FREE}[op]
        self._ck(self.L.wo_snapshot(self.h, code, int(n_steps)), "wo_snapshot")

    def swap_direction(self):
        self._ck(self.L.wo_swap_direction(self.h), "wo_swap_direction")

    def zero_accumulator(self):
        self._ck(self.L.wo_zero_accumulator(self.h), "wo_zero_accumulator")

    def get_accumulator(self, out=None):
        """The accumulator as a host array (into ``out``, a C-contiguous array
        of the grid's shape and dtype, when given)."""
        if out is None:
            out = np.empty(self.grid.shape, self.dtype)
        elif (out.shape != self.grid.shape or out.dtype != self.dtype
              or not out.flags.c_contiguous):
            raise ConfigError("accumulator output must be a C-contiguous "
                              f"{self.grid.shape} {np.dtype(self.dtype).name} array")
        self._ck(self.L.wo_get_accumulator(self.h, N.ptr(out)), "wo_get_accumulator")
        return out

    def set_accumulator(self, values):
        self._ck(self.L.wo_set_accumulator(self.h, N.ptr(self._field(values))),
                 "wo_set_accumulator")

    # --------------------------------------------------------------- sweeps
    def sweep_forward(self, n_steps, src_flat, amp_table, accumulate, dt, scale,
                      detail_on_fail="", history=False):
        src = np.ascontiguousarray(np.asarray(src_flat, dtype=np.int64).reshape(-1))
        amp = np.ascontiguousarray(np.asarray(amp_table, dtype=np.float64))
        peak = ctypes.c_double(0.0)
        fstep = ctypes.c_int64(0)
        fmax = ctypes.c_double(0.0)
        flags = (N.WO_FWD_ACCUMULATE if accumulate else 0) | (N.WO_FWD_HISTORY if history else 0)
        rc = self.L.wo_sweep_forward(self.h, int(n_steps), len(src), N.ptr(src), N.ptr(amp),
                                     flags, float(dt), float(scale),
                                     ctypes.byref(peak), ctypes.byref(fstep), ctypes.byref(fmax))
        if rc == N.WO_ERR_UNSTABLE:
            m = fmax.value
            detail = detail_on_fail
            if math.isfinite(m) and scale > 0:
                detail = f"exceeds 1e6 x scale {scale:g}"
            raise SolverInstabilityError(int(fstep.value), m, detail=detail)
        self._ck(rc, "wo_sweep_forward")
        return peak.value

    def shot_misfit(self, n_steps, kind, measured, c, adj_coef, write_adj, k):
        meas = (np.ascontiguousarray(measured, dtype=np.float64) if measured is not None
                else None)
        if meas is not None:
            self.claim = None  # new measured traces resident: the owner re-claims
        cost = ctypes.c_double(0.0)
        self._ck(self.L.wo_shot_misfit(self.h, int(n_steps), int(kind), N.ptr(meas),
                                       float(c[0]), float(c[1]), float(c[2]), float(c[3]),
                                       float(adj_coef), int(bool(write_adj)), float(k),
                                       ctypes.byref(cost)), "wo_shot_misfit")
        return cost.value

    def get_store(self, n_steps):
        out = np.empty((int(n_steps), self.n_sup), self.dtype)
        self._ck(self.L.wo_get_store(self.h, int(n_steps), N.ptr(out)), "wo_get_store")
        return out

    def sweep_backward(self, n_steps, src_flat, amp_row, inject, accumulate, dt,
                       detail_on_fail=""):
        amp = np.ascontiguousarray(np.asarray(amp_row, dtype=np.float64))
        fstep = ctypes.c_int64(0)
        fmax = ctypes.c_double(0.0)
        rc = self.L.wo_sweep_backward(self.h, int(n_steps), int(src_flat), N.ptr(amp),
                                      int(bool(inject)), int(bool(accumulate)), float(dt),
                                      ctypes.byref(fstep), ctypes.byref(fmax))
        if rc == N.WO_ERR_UNSTABLE:
            raise SolverInstabilityError(int(fstep.value), fmax.value, detail=detail_on_fail)
        self._ck(rc, "wo_sweep_backward")

    def sweep_forward_range(self, n_steps, n_begin, n_end, src_flat, amp_table, accumulate, dt):
        src = np.ascontiguousarray(np.asarray(src_flat, dtype=np.int64).reshape(-1))
        amp = np.ascontiguousarray(np.asarray(amp_table, dtype=np.float64))
        flags = N.WO_FWD_ACCUMULATE if accumulate else 0
        self._ck(self.L.wo_sweep_forward_range(self.h, int(n_steps), int(n_begin), int(n_end),
                                               len(src), N.ptr(src), N.ptr(amp), flags,
                                               float(dt)), "wo_sweep_forward_range")

    def sweep_backward_range(self, n_steps, n_hi, n_lo, src_flat, amp_row, inject, accumulate,
                             dt):
        amp = np.ascontiguousarray(np.asarray(amp_row, dtype=np.float64))
        self._ck(self.L.wo_sweep_backward_range(self.h, int(n_steps), int(n_hi), int(n_lo),
                                                int(src_flat), N.ptr(amp), int(bool(inject)),
                                                int(bool(accumulate)), float(dt)),
                 "wo_sweep_backward_range")

    def check_maxima(self, n_steps):
        out = np.empty(int(n_steps) + 2, dtype=np.float64)
        self._ck(self.L.wo_check_maxima(self.h, int(n_steps), N.ptr(out)), "wo_check_maxima")
        return out

    def halo_planes(self, out=False):
        """(first, last, ghost_lo, ghost_hi) device addresses of the current
        level (out=True: the level a split step is writing) and the plane
        size in bytes."""
        p = [ctypes.c_void_p() for _ in range(4)]
        pb = ctypes.c_int64()
        fn = self.L.wo_halo_planes_out if out else self.L.wo_halo_planes
        self._ck(fn(self.h, *[ctypes.byref(x) for x in p], ctypes.byref(pb)), "wo_halo_planes")
        return tuple(x.value for x in p), pb.value

    def slab_ghosts(self):
        """(ghost_lo[4], ghost_hi[4], flags[2]) device addresses of this
        slab's ghost planes per level buffer and of its incoming flags."""
        lo = (ctypes.c_void_p * 4)()
        hi = (ctypes.c_void_p * 4)()
        fl = (ctypes.c_void_p * 2)()
        self._ck(self.L.wo_slab_ghosts(self.h, lo, hi, fl), "wo_slab_ghosts")
        return [x or 0 for x in lo], [x or 0 for x in hi], [x or 0 for x in fl]

    def set_slab_peers(self, lo_ghost=None, hi_ghost=None, lo_flag=0, hi_flag=0):
        """Peer ghost stores (wo_slab_peers); no arguments: off."""
        arr = lambda v: None if v is None else (ctypes.c_void_p * 4)(*[x or None for x in v])
        self._ck(self.L.wo_slab_peers(self.h, arr(lo_ghost), arr(hi_ghost), lo_flag or None,
                                      hi_flag or None), "wo_slab_peers")

    def ipc_export(self, ptr):
        """(64-byte CUDA IPC handle, byte offset) of the device address ptr
        (wo_ipc_export), for a neighbour process's ipc_open."""
        h = ctypes.create_string_buffer(64)
        off = ctypes.c_int64()
        self._ck(self.L.wo_ipc_export(self.h, ptr, h, ctypes.byref(off)), "wo_ipc_export")
        return h.raw, off.value

    def ipc_open(self, handle, offset):
        """Device address in this process of a neighbour's exported pointer
        (wo_ipc_open; the mapping lives as long as this context)."""
        p = ctypes.c_void_p()
        self._ck(self.L.wo_ipc_open(self.h, bytes(handle), int(offset), ctypes.byref(p)),
                 "wo_ipc_open")
        return p.value

    def set_graphs(self, on):
        """Replay repeated sweeps from captured CUDA graphs (default on)."""
        self._ck(self.L.wo_set_option(self.h, N.WO_OPT_GRAPHS, int(bool(on))), "wo_set_option")

    def set_cluster(self, on):
        """Cluster-resident whole sweeps of small 2D grids (WO_OPT_CLUSTER):
        True / False, or None for the default (on)."""
        v = 2 if on is None else int(bool(on))
        self._ck(self.L.wo_set_option(self.h, N.WO_OPT_CLUSTER, v), "wo_set_option")

    def slab_abort(self):
        """Release streams waiting on this slab's peer flags (wo_slab_abort)."""
        self._ck(self.L.wo_slab_abort(self.h), "wo_slab_abort")

    def slab_state(self):
        """(flag words [4], signals sent, epoch, stream idle) — wo_slab_state."""
        out = np.zeros(7, dtype=np.int64)
        self._ck(self.L.wo_slab_state(self.h, N.ptr(out)), "wo_slab_state")
        return out.tolist()

    def set_two_step(self, on):
        """Two time steps per HBM pass where the grid allows it (fp32 and
        fp64; WO_OPT_TWO_STEP, default on; slabs: off until the decomposition
        enables it on every slab)."""
        self._ck(self.L.wo_set_option(self.h, N.WO_OPT_TWO_STEP, int(on)), "wo_set_option")

    def prepare_two_step(self):
        """Allocate and build the two-step buffers now (wo_prepare_two_step):
        True when this context will take two-step passes."""
        ready = ctypes.c_int(0)
        self._ck(self.L.wo_prepare_two_step(self.h, ctypes.byref(ready)), "wo_prepare_two_step")
        return bool(ready.value)

    def set_plane_part(self, part):
        """Split slab steps: 1 boundary planes, 2 interior (+rotation), 0 whole."""
        self._ck(self.L.wo_set_option(self.h, N.WO_OPT_PLANE_PART, int(part)), "wo_set_option")

    @property
    def stream_ptr(self):
        return int(self.L.wo_stream(self.h) or 0)

    def sweep_adjoint_reference(self, n_steps, dt):
        fstep = ctypes.c_int64(0)
        fmax = ctypes.c_double(0.0)
        rc = self.L.wo_sweep_adjoint_reference(self.h, int(n_steps), float(dt),
                                               ctypes.byref(fstep), ctypes.byref(fmax))
        if rc == N.WO_ERR_UNSTABLE:
            raise SolverInstabilityError(int(fstep.value), fmax.value)
        self._ck(rc, "wo_sweep_adjoint_reference")

    def get_history(self, n_first, out):
        """Recorded levels u^{n_first} .. into out ([k] + grid shape, C order)."""
        assert out.dtype == self.dtype and out.flags.c_contiguous
        k = out.shape[0]
        self._ck(self.L.wo_get_history(self.h, int(n_first), int(k), N.ptr(out)),
                 "wo_get_history")
        return out

    def free_history(self):
        self._ck(self.L.wo_free_history(self.h), "wo_free_history")

    def gradient(self, two_k, copy=True):
        """acc /= T(2k); returns the host copy (copy=False: stays on the device)."""
        out = np.empty(self.grid.shape, self.dtype) if copy else None
        self._ck(self.L.wo_get_gradient(self.h, float(two_k), N.ptr(out)), "wo_get_gradient")
        return out

    def timer_mark(self, idx):
        self._ck(self.L.wo_timer_mark(self.h, int(idx)), "wo_timer_mark")

    def timer_elapsed_ms(self, a, b):
        ms = ctypes.c_double(0.0)
        self._ck(self.L.wo_timer_elapsed(self.h, int(a), int(b), ctypes.byref(ms)),
                 "wo_timer_elapsed")
        return ms.value

    def set_fast_div(self, allow):
        self._ck(self.L.wo_set_option(self.h, N.WO_OPT_FAST_DIV, int(bool(allow))),
                 "wo_set_option")

    def set_pair_kernel(self, on):
        self._ck(self.L.wo_set_option(self.h, N.WO_OPT_PAIR_KERNEL, int(bool(on))),
                 "wo_set_option")

    def set_tma_kernel(self, mode):
        """0/False: never; 1/True: the TMA kernels on whole-tile grids (default)."""
        self._ck(self.L.wo_set_option(self.h, N.WO_OPT_TMA_KERNEL, int(mode)), "wo_set_option")

    def fast_div_active(self):
        return bool(self.L.wo_fast_div_active(self.h))

    def synchronize(self):
        self._ck(self.L.wo_synchronize(self.h), "wo_synchronize")

    def step(self, force=None, want_max=False):
        """One step with a sparse/dense/None force; returns max|u_new| or None."""
        idx = vals = dense = None
        n = 0
        if isinstance(force, np.ndarray):
            dense = np.ascontiguousarray(force, dtype=np.float64)
            if dense.shape != self.grid.shape:
                raise ConfigError("dense force shape does not match the grid")
        elif force is not None:
            idx = np.ascontiguousarray(np.asarray(force[0], dtype=np.int64).reshape(-1))
            vals = np.ascontiguousarray(np.asarray(force[1], dtype=np.float64).reshape(-1))
            n = len(idx)
        m = ctypes.c_double(0.0)
        self._ck(self.L.wo_step(self.h, n, N.ptr(idx), N.ptr(vals), N.ptr(dense),
                                int(bool(want_max)), ctypes.byref(m)), "wo_step")
        return m.value if want_max else None

    # ---------------------------------------------------------- profiling
    def set_profiling(self, on):
        """on: False/0 off, True/1 every step launch, k: every k-th launch."""
        self._ck(self.L.wo_set_profiling(self.h, int(on)), "wo_set_profiling")

    def stats(self):
        a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
        self._ck(self.L.wo_stats(self.h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)),
                 "wo_stats")
        sm, sn, pm, pn = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double(), ctypes.c_int64()
        self._ck(self.L.wo_profile_stats(self.h, ctypes.byref(sm), ctypes.byref(sn),
                                         ctypes.byref(pm), ctypes.byref(pn)), "wo_profile_stats")
        return {"launches": a.value, "step_launches": b.value, "step_kernel_ms": c.value,
                "pair_launches": int(self.L.wo_pair_launches(self.h)),
                "profiled_single_ms": sm.value, "profiled_single_n": sn.value,
                "profiled_pair_ms": pm.value, "profiled_pair_n": pn.value}

    def reset_stats(self):
        self._ck(self.L.wo_reset_stats(self.h), "wo_reset_stats")

    def device_bytes(self):
        return int(self.L.wo_device_bytes(self.h))

    def field_buffers(self):
        """Solution-sized device buffers held now (wo_field_buffers)."""
        return int(self.L.wo_field_buffers(self.h))


_CACHE: OrderedDict = OrderedDict()
_CACHE_MAX = 3


def get_context(grid: Grid, dtype, device=0, four_fields=False) -> DeviceGrid:
    """Cached DeviceGrid per (shape, dx, dtype, device, memory mode).

    four_fields: a context that never takes two-step passes, so it holds the
    reference's memory contract of four solution-sized buffers (SPEC
    acceptance 5: gamma, two window levels — u^{n+1} in place over u^{n-1} —
    and the accumulator) instead of the fast path's ten (four levels, the
    accumulator, gamma and four precomputed material fields)."""
    key = (grid.shape, float(grid.dx), np.dtype(dtype).str, device, bool(four_fields))
    ctx = _CACHE.get(key)
    if ctx is not None and not ctx.h:      # closed by its user: replace it
        del _CACHE[key]
        ctx = None
    if ctx is None:
        while len(_CACHE) >= _CACHE_MAX:
            _, old = _CACHE.popitem(last=False)
            old.close()
        ctx = DeviceGrid(grid, dtype, device)
        if four_fields:
            ctx.set_two_step(0)
        _CACHE[key] = ctx
    else:
        _CACHE.move_to_end(key)
    return ctx


def release_contexts():
    while _CACHE:
        _, c = _CACHE.popitem()
        c.close()
