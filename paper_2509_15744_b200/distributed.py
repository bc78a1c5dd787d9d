"""Multi-GPU modes of the superposed gradient.

slab decomposition (SlabGradient)
    The grid is cut along axis 0 (outermost, so a halo is one contiguous
    n1*n2 plane).  Each slab context (``wo_create_slab``) holds its planes plus
    two ghost planes per interior face; the step kernels read ghost planes
    exactly like interior planes and mirror only at the global ends, so the
    per-cell arithmetic is unchanged and the gradient, traces and adjoint
    store are BITWISE equal to one GPU.  With the exchange halos every step
    each slab sends its first/last plane of the new level to its neighbours'
    ghost planes; by
    default (``overlap``) a step runs as its two boundary planes, then the
    exchange is started, then the interior planes are updated while the
    planes travel, and the next step waits for the exchange (WO_OPT_PLANE_PART;
    NCCL is ordered on the context's stream, no host synchronisation):
      * ``LoopbackHalo`` — all slabs in one process (same device or peer
        devices), ``wo_exchange_local`` copies;
      * ``PeerHalo`` — all slabs in one process, no exchange at all: every
        launch stores its boundary planes straight into the neighbours' two
        ghost planes (NVLink stores between GPUs) and signals them with a
        device flag the neighbour's next launch waits on (``wo_slab_peers``);
        whole sweeps are enqueued on every slab without returning to Python,
        and two-step passes run on slabs too (two ghost planes deep);
      * ``TorchHalo`` — one slab per process (torchrun), torch.distributed
        point-to-point send/recv of the plane tensors (NCCL over NVLink on
        GPUs; the same code runs on gloo/CPU tensors in the tests);
      * ``IpcPeerHalo`` — one slab per process, PeerHalo's kernel stores
        across processes: each rank exports its ghost planes and flags as
        CUDA IPC handles (``wo_ipc_export``), the neighbours map them
        (``wo_ipc_open``) and hand them to ``wo_slab_peers``; the handles
        travel once through an object all-gather, then no collective per step.
    Costs are summed per slab then across slabs (fp64, not bitwise: the
    reference's BLAS dot order is unknown anyway); stability maxima are
    combined with max before the reference's first-failure scan.

shot-parallel (ShotParallelGradient)
    Rank r evaluates shots r, r+P, ...; the unscaled accumulators and the
    costs are summed with one all-reduce per evaluation, then acc /= T(2k).
    Not bitwise (summation order), like the reference's own remark on shot
    concurrency; the throughput mode for multi-shot problems
    that fit one GPU.
"""

from __future__ import annotations

import math

import numpy as np

from . import _native as N
from . import engine
from .engine import SolverInstabilityError, source_amplitude_table
from .grids import ConfigError, precision_dtype

STABILITY_CHECK_INTERVAL = 50
STABILITY_GROWTH_FACTOR = 1e6


# ------------------------------------------------------------- host logic
def shot_partition(n_shots, rank, world):
    """Round-robin shot indices owned by rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    return list(range(rank, n_shots, world))


def slab_ranges(n0, parts):
    """Balanced [i0, i1) plane ranges along axis 0 (each >= 1 plane)."""
    if not 1 <= parts <= n0:
        raise ConfigError(f"cannot cut {n0} planes into {parts} slabs")
    base, extra = divmod(n0, parts)
    out, i = [], 0
    for p in range(parts):
        n = base + (1 if p < extra else 0)
        out.append((i, i + n))
        i += n
    return out


def localize(flat, shape, i0, i1):
    """Global C-order flat indices -> (owned mask, local flat indices) for
    the slab of planes [i0, i1)."""
    flat = np.asarray(flat, dtype=np.int64)
    plane = int(shape[1]) * int(shape[2])
    i = flat // plane
    owned = (i >= i0) & (i < i1)
    return owned, flat[owned] - i0 * plane


def recomputed_planes(slabs):
    """Global planes a two-step slab pass recomputes beyond the slab
    boundaries: b-1 (by the slab above) and b (by the slab below) for every
    interior boundary b."""
    out = set()
    for i0, _ in list(slabs)[1:]:
        out.update((i0 - 1, i0))
    return out


def two_step_slabs_ok(slabs, plane, supports):
    """Whether every slab of the decomposition may run two-step passes with
    peer ghost stores: at least two planes per slab (two ghost planes per
    neighbour, peer stores of planes 0, 1 / n0-2, n0-1) and no support node on
    a recomputed plane (its adjoint force lives in the neighbour's store;
    sources there are injected by the kernels themselves).  All slabs decide
    alike, as their launches must match one for one."""
    if any(i1 - i0 < 2 for i0, i1 in slabs):
        return False
    bad = recomputed_planes(slabs)
    for sup in supports:
        planes = np.unique(np.asarray(sup, dtype=np.int64) // int(plane))
        if any(int(p) in bad for p in planes):
            return False
    return True


def local_source(g_src, plane, alloc_range, i_begin):
    """Slab-local flat index of a global source node when it lies on the
    slab's own or ghost planes (a two-step pass recomputes one plane beyond
    the slab, sources included), else None."""
    lo, hi = alloc_range
    if lo * plane <= g_src < hi * plane:
        return int(g_src - i_begin * plane)
    return None


def first_failure_forward(maxima, n_steps, scale):
    """First failing forward check (solver.py:180-186, gradients.py:247-248):
    (step, max) or None; also returns the peak over the checks."""
    peak = 0.0
    for n in range(1, n_steps):
        if n % STABILITY_CHECK_INTERVAL and n != n_steps - 1:
            continue
        m = float(maxima[n])
        if not math.isfinite(m) or (scale > 0.0 and m > STABILITY_GROWTH_FACTOR * scale):
            return (n + 1, m), peak
        peak = max(peak, m)
    return None, peak


def first_failure_backward(maxima, n_steps):
    """First failing backward check (gradients.py:272-280): (step, max) or None."""
    for n in range(n_steps - 1, 0, -1):
        if n % STABILITY_CHECK_INTERVAL and n != 1:
            continue
        m = float(maxima[n])
        if not math.isfinite(m):
            return (n - 1, m)
    return None


def exchange_planes_async(first, last, ghost_lo, ghost_hi, rank, world, group=None):
    """Start the halo exchange of one slab with torch.distributed P2P: first
    -> rank-1's high ghost, last -> rank+1's low ghost (tensors: CUDA with
    NCCL, CPU with gloo).  Returns the requests; with NCCL the transfers are
    ordered after the work already queued on the current CUDA stream."""
    import torch.distributed as dist

    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, first, rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, ghost_lo, rank - 1, group))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, last, rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, ghost_hi, rank + 1, group))
    return dist.batch_isend_irecv(ops) if ops else []


def exchange_planes(first, last, ghost_lo, ghost_hi, rank, world, group=None):
    """Blocking form of exchange_planes_async."""
    for req in exchange_planes_async(first, last, ghost_lo, ghost_hi, rank, world, group):
        req.wait()


def _device_view(ptr, nbytes, dtype, device):
    """torch tensor over a device address (CUDA array interface, no copy)."""
    import torch

    n = nbytes // np.dtype(dtype).itemsize

    class _View:
        __cuda_array_interface__ = {"shape": (n,), "typestr": np.dtype(dtype).str,
                                    "data": (int(ptr), False), "version": 3, "strides": None}

    return torch.as_tensor(_View(), device=f"cuda:{device}")


# ----------------------------------------------------------- halo backends
class LoopbackHalo:
    """All slabs of the decomposition live in this process."""

    def __init__(self, ctxs):
        self.ctxs = ctxs

    def exchange(self):
        for lo, hi in zip(self.ctxs[:-1], self.ctxs[1:]):
            rc = lo.L.wo_exchange_local(lo.h, hi.h)
            if rc:
                engine._raise(lo.h, rc, "wo_exchange_local")

    # split steps: the boundary planes of the level being written
    def begin(self):
        for lo, hi in zip(self.ctxs[:-1], self.ctxs[1:]):
            rc = lo.L.wo_exchange_local_out(lo.h, hi.h)
            if rc:
                engine._raise(lo.h, rc, "wo_exchange_local_out")
        return []

    def end(self, works):
        pass

    def allreduce_max(self, arr):
        return arr

    def allreduce_sum(self, x):
        return x


class PeerHalo(LoopbackHalo):
    """All slabs in this process; the step kernels store the boundary planes
    into the neighbours' ghost planes and bump their flags (split steps
    only), so begin / end have nothing left to move."""

    def __init__(self, ctxs):
        super().__init__(ctxs)
        ghosts = [c.slab_ghosts() for c in ctxs]
        for i, c in enumerate(ctxs):
            lo = ghosts[i - 1] if i > 0 else None          # (ghost_lo, ghost_hi, flags)
            hi = ghosts[i + 1] if i + 1 < len(ctxs) else None
            c.set_slab_peers(lo_ghost=lo[1] if lo else None, hi_ghost=hi[0] if hi else None,
                             lo_flag=lo[2][1] if lo else 0, hi_flag=hi[2][0] if hi else 0)

    def exchange(self):
        raise ConfigError("PeerHalo moves planes inside the sweeps' launches")

    def begin(self):
        return []

    def close(self):
        for c in self.ctxs:
            c.set_slab_peers()


class TorchHalo:
    """One slab per process; neighbours are ranks r-1 and r+1."""

    def __init__(self, ctx, rank, world, group=None):
        self.ctx, self.rank, self.world, self.group = ctx, rank, world, group

    def exchange(self):
        import torch

        (first, last, glo, ghi), pb = self.ctx.halo_planes()
        dt, dev = self.ctx.dtype, self.ctx.device
        view = lambda p: _device_view(p, pb, dt, dev) if p else None  # noqa: E731
        exchange_planes(view(first), view(last), view(glo), view(ghi), self.rank, self.world,
                        self.group)
        torch.cuda.synchronize(dev)

    # split steps: the new boundary planes travel while the interior part of
    # the step runs (NCCL ordered on the context stream both ways)
    def _ext(self):
        import torch

        return torch.cuda.ExternalStream(self.ctx.stream_ptr, device=f"cuda:{self.ctx.device}")

    def begin(self):
        import torch

        (first, last, glo, ghi), pb = self.ctx.halo_planes(out=True)
        dt, dev = self.ctx.dtype, self.ctx.device
        view = lambda p: _device_view(p, pb, dt, dev) if p else None  # noqa: E731
        with torch.cuda.stream(self._ext()):
            return exchange_planes_async(view(first), view(last), view(glo), view(ghi),
                                         self.rank, self.world, self.group)

    def end(self, works):
        import torch

        with torch.cuda.stream(self._ext()):
            for w in works:
                w.wait()

    def _dev(self):
        """Where reduction tensors live: the GPU for NCCL, the host for gloo."""
        import torch.distributed as dist

        return "cpu" if dist.get_backend(self.group) == "gloo" else f"cuda:{self.ctx.device}"

    def allreduce_max(self, arr):
        if self.world == 1:
            return arr
        import torch
        import torch.distributed as dist

        t = torch.from_numpy(np.ascontiguousarray(arr)).to(self._dev())
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return t.cpu().numpy()

    def allreduce_sum(self, x):
        if self.world == 1:
            return x
        import torch
        import torch.distributed as dist

        t = torch.tensor([x], dtype=torch.float64, device=self._dev())
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return float(t.item())


class HostStagedHalo(TorchHalo):
    """One slab per process, planes staged through host memory and exchanged
    with CPU torch.distributed send/recv (gloo): a slab decomposition across
    processes that never makes one GPU wait on another process (so several
    ranks may share one GPU — the multi-process test of the slab path), and
    the fallback where no GPU-aware backend exists.  Whole-step exchanges
    (overlap=False); maxima and costs reduce on CPU tensors."""

    def exchange(self):
        import torch

        (first, last, glo, ghi), pb = self.ctx.halo_planes()
        dt, dev = self.ctx.dtype, self.ctx.device
        n = pb // dt.itemsize
        view = lambda p: _device_view(p, pb, dt, dev)  # noqa: E731
        self.ctx.synchronize()                     # the step's planes are final
        send_lo = view(first).cpu() if first and self.rank > 0 else None
        send_hi = view(last).cpu() if last and self.rank < self.world - 1 else None
        recv_lo = torch.empty(n, dtype=_torch_dtype(dt)) if glo else None
        recv_hi = torch.empty(n, dtype=_torch_dtype(dt)) if ghi else None
        exchange_planes(send_lo, send_hi, recv_lo, recv_hi, self.rank, self.world, self.group)
        for p, b in ((glo, recv_lo), (ghi, recv_hi)):
            if p:
                view(p).copy_(b)
        torch.cuda.synchronize(dev)                # ghosts in place before the next step

    def begin(self):
        raise ConfigError("HostStagedHalo exchanges whole steps (overlap=False)")

    def allreduce_max(self, arr):
        if self.world == 1:
            return arr
        import torch
        import torch.distributed as dist

        t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64))
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return t.numpy()

    def allreduce_sum(self, x):
        if self.world == 1:
            return x
        import torch
        import torch.distributed as dist

        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return float(t.item())


def _torch_dtype(dt):
    import torch

    return torch.float32 if np.dtype(dt) == np.float32 else torch.float64


def ipc_peer_wiring(rank, world, exports):
    """Which neighbour exports rank opens for wo_slab_peers.

    exports[r] = (ghost_lo[4], ghost_hi[4], flags[2]) of rank r, each entry an
    exported (handle, offset) or None.  The lower neighbour contributes its
    HIGH ghost planes and flag [1] (bumped by its upper neighbour = this
    rank), the upper neighbour its LOW ghost planes and flag [0]."""
    lo = exports[rank - 1] if rank > 0 else None
    hi = exports[rank + 1] if rank + 1 < world else None
    return {"lo_ghost": lo[1] if lo else None, "lo_flag": lo[2][1] if lo else None,
            "hi_ghost": hi[0] if hi else None, "hi_flag": hi[2][0] if hi else None}


class IpcPeerHalo(TorchHalo):
    """One slab per process, no exchange step: every launch stores its
    boundary planes into the neighbour processes' ghost planes through CUDA
    IPC mappings and bumps their flags (``wo_slab_peers``), like PeerHalo.
    Setup is one all-gather of the exported handles.  Each sweep is a flag
    epoch whose first signal follows the rank's window reset (so no
    neighbour store lands before it); the stability / cost all-reduces of
    TorchHalo separate consecutive epochs, which the flag-slot reuse needs."""

    def __init__(self, ctx, rank, world, group=None):
        import torch.distributed as dist

        super().__init__(ctx, rank, world, group)
        if world == 1:   # one slab, no neighbours: nothing to map
            return
        glo, ghi, flags = ctx.slab_ghosts()
        exp = lambda p: ctx.ipc_export(p) if p else None  # noqa: E731
        mine = ([exp(p) for p in glo], [exp(p) for p in ghi], [exp(p) for p in flags])
        exports = [None] * world
        dist.all_gather_object(exports, mine, group=group)
        w = ipc_peer_wiring(rank, world, exports)
        opn = lambda e: ctx.ipc_open(*e) if e else 0  # noqa: E731
        ctx.set_slab_peers(
            lo_ghost=[opn(e) for e in w["lo_ghost"]] if w["lo_ghost"] else None,
            hi_ghost=[opn(e) for e in w["hi_ghost"]] if w["hi_ghost"] else None,
            lo_flag=opn(w["lo_flag"]), hi_flag=opn(w["hi_flag"]))
        dist.barrier(group=group)   # every slab's flags reset before anyone steps

    def exchange(self):
        raise ConfigError("IpcPeerHalo moves planes inside the sweeps' launches")

    def begin(self):
        return []

    def end(self, works):
        pass

    def close(self):
        if self.world > 1:
            self.ctx.set_slab_peers()


# ------------------------------------------------------------ slab driver
class SlabGradient:
    """gradient_superposed over axis-0 slabs (bitwise equal to one GPU).

    slabs: list of (i0, i1) handled by THIS process; halo: 'loopback' (all
    slabs here) or a TorchHalo-compatible object built by ``for_rank``."""

    def __init__(self, problem, material, config, slabs, devices=None, halo="loopback",
                 overlap=True):
        from .gradients import SuperpositionConfig, _misfit_spec, _shot_list

        if not isinstance(config, SuperpositionConfig):
            config = SuperpositionConfig(k=float(config))
        grid = problem.grid
        if grid.ndim != 3:
            raise ConfigError("slab decomposition needs a 3D grid")
        self.problem, self.material, self.config = problem, material, config
        self.dtype = precision_dtype(config.precision)
        devices = devices or [0] * len(slabs)
        self.slabs = list(slabs)
        self.all_slabs = list(slabs)   # the whole decomposition (for_rank: every rank's)
        self.ctxs = [engine.DeviceGrid(grid, self.dtype, d, slab=s)
                     for s, d in zip(self.slabs, devices)]
        if halo == "loopback":
            self.halo = LoopbackHalo(self.ctxs)
        elif halo == "peer":
            self.halo = PeerHalo(self.ctxs)
        else:
            self.halo = halo
        # overlap: every step runs as boundary planes -> halo exchange started
        # -> interior planes -> exchange awaited, so the transfer of the new
        # boundary planes overlaps the interior update (WO_OPT_PLANE_PART)
        self.overlap = overlap
        self._misfit_spec = _misfit_spec
        self._shots = _shot_list(problem)

    @classmethod
    def for_rank(cls, problem, material, config, rank, world, device=None, group=None,
                 overlap=True, halo="nccl"):
        """One slab per torchrun rank: halo 'nccl' (send/recv of the planes,
        TorchHalo), 'ipc' (peer ghost stores through CUDA IPC, IpcPeerHalo)
        or 'staged' (host-staged gloo send/recv, HostStagedHalo, whole
        steps)."""
        if halo not in ("nccl", "ipc", "staged"):
            raise ConfigError(f"unknown rank halo {halo!r}")
        if halo == "staged":
            overlap = False
        slab = slab_ranges(problem.grid.shape[0], world)[rank]
        dev = rank if device is None else device
        obj = cls(problem, material, config, [slab], [dev], halo=None, overlap=overlap)
        obj.all_slabs = slab_ranges(problem.grid.shape[0], world)
        make = {"ipc": IpcPeerHalo, "staged": HostStagedHalo}.get(halo, TorchHalo)
        obj.halo = make(obj.ctxs[0], rank, world, group)
        return obj

    @property
    def peer_stores(self):
        """Whole sweeps with in-kernel peer ghost stores (PeerHalo /
        IpcPeerHalo with neighbours) instead of per-step exchanges."""
        h = self.halo
        return isinstance(h, PeerHalo) or (isinstance(h, IpcPeerHalo) and h.world > 1)

    @property
    def solo(self):
        """One slab covering the whole grid (one rank): no halo at all."""
        n0 = self.problem.grid.shape[0]
        return all(i0 == 0 and i1 == n0 for i0, i1 in self.all_slabs)

    @property
    def whole_sweeps(self):
        return self.peer_stores or self.solo

    def upload(self, material=None, gamma_local=None):
        """Material onto every slab (own + ghost planes; gamma_local: per
        context, its planes as contiguous fp64 host arrays); decides two-step
        passes for the whole decomposition."""
        dt = self.problem.time.dt
        for i, c in enumerate(self.ctxs):
            c.set_material(self.material if material is None else material, dt,
                           None if gamma_local is None else gamma_local[i])
        grid = self.problem.grid
        self.two_step = self.whole_sweeps and two_step_slabs_ok(
            self.all_slabs, grid.shape[1] * grid.shape[2], [s.support_idx for _, s in self._shots])
        for c in self.ctxs:
            c.set_two_step(1 if self.two_step else 0)
        if self.two_step:
            # every slab must launch alike: allocate the two-step buffers now
            # and fall back to single steps everywhere if any slab (of any
            # rank) cannot hold them (e.g. 2048^3 over two GPUs)
            short = 0.0 if all(c.prepare_two_step() for c in self.ctxs) else 1.0
            if self.halo.allreduce_max(np.array([short]))[0] > 0:
                self.two_step = False
                for c in self.ctxs:
                    c.set_two_step(0)
        return self

    def set_measured(self, measured):
        """New measured traces [n_shots, n_support, N] for the FWI shots."""
        from .gradients import _shot_list

        self.problem.measured = np.asarray(measured, dtype=np.float64)
        self._shots = _shot_list(self.problem)

    def _peer_ranges(self, first, last, step):
        """Step ranges in which the peer-store sweeps are enqueued.  Slabs on
        different devices (one per process, or one per GPU here): the whole
        sweep at once.  Several slabs on ONE device: one two-step pass per
        range, interleaved across the slabs, so every flag wait refers to work
        enqueued before it — a stream blocked on a wait may share a hardware
        queue with a neighbour's stream, and a wait on work enqueued later
        behind it would never be satisfied."""
        devices = [c.device for c in self.ctxs]
        if len(set(devices)) == len(devices):
            return [(first, last)]
        out, n = [], first
        while n != last:
            m = n + step if abs(last - n) > 2 else last
            out.append((n, m))
            n = m
        return out

    def _forward_all(self, n_steps, src_local, amp, accumulate, dt):
        no_src = np.zeros((0, n_steps))
        if self.whole_sweeps:   # sweeps enqueued on every slab (interleaved), then awaited
            for n0, n1 in self._peer_ranges(1, n_steps, 2):
                for c, s in zip(self.ctxs, src_local):
                    c.sweep_forward_range(n_steps, n0, n1, [] if s is None else [s],
                                          no_src if s is None else amp, accumulate, dt)
        else:
            for n in range(1, n_steps):
                self._steps(lambda c, s, _n=n: c.sweep_forward_range(
                    n_steps, _n, _n + 1, [] if s is None else [s],
                    no_src if s is None else amp, accumulate, dt), src_local)

    def record_traces(self, material):
        """Forward solves of `material` (one per shot, the shots' sources) with
        u^n recorded at this process's support nodes: traces [n_shots,
        n_support, N] in the problem's support order, rows of nodes owned by
        other processes left 0 — the slab form of synthesize_measurements
        with refine = 1 (fwi.py:121-168; the bench's C5 truth).  The material
        of the gradient evaluations is restored afterwards."""
        self.upload(material)
        n_steps = self.problem.time.n_steps
        out = np.zeros((len(self._shots), len(self._shots[0][1].support_idx), n_steps))
        self._guarded(self._record, material, out)
        return out

    def _record(self, material, out):
        from .solver import injection_scale

        problem, grid = self.problem, self.problem.grid
        n_steps, dt = problem.time.n_steps, problem.time.dt
        plane = grid.shape[1] * grid.shape[2]
        try:
            for si, (source, shot) in enumerate(self._shots):
                g_src = grid.flat_index(source.node)
                amp = source_amplitude_table([source], dt, n_steps)
                scale = injection_scale([source], material, dt, self.dtype) * n_steps
                owned_rows = []
                for c in self.ctxs:
                    owned, local = localize(shot.support_idx, grid.shape, c.i_begin, c.i_end)
                    order = c.set_support(local)
                    owned_rows.append((np.flatnonzero(owned), order))
                    c.reset_window()
                src_local = [local_source(g_src, plane, c.alloc_range, c.i_begin)
                             for c in self.ctxs]
                self._forward_all(n_steps, src_local, amp, False, dt)
                maxima = self.halo.allreduce_max(
                    np.max([c.check_maxima(n_steps) for c in self.ctxs], axis=0))
                fail, _ = first_failure_forward(maxima, n_steps, scale)
                if fail:
                    raise SolverInstabilityError(*fail)
                for c, (rows, order) in zip(self.ctxs, owned_rows):
                    if len(rows):
                        store = c.get_store(n_steps)          # [N][n_sup], device order
                        out[si, rows[order]] = store.T
        finally:
            self.upload()

    def _steps(self, step, *per_ctx):
        """One time step on every slab, then the halo exchange; with overlap
        the exchange of the new boundary planes runs during the interior."""
        args = list(zip(self.ctxs, *per_ctx))
        if not self.overlap:
            for a in args:
                step(*a)
            self.halo.exchange()
            return
        try:
            for a in args:
                a[0].set_plane_part(1)
                step(*a)
            works = self.halo.begin()
            for a in args:
                a[0].set_plane_part(2)
                step(*a)
            self.halo.end(works)
        finally:
            for c in self.ctxs:
                c.set_plane_part(0)

    def run(self):
        return self._guarded(self._run)

    def _guarded(self, fn, *a):
        if not self.peer_stores:
            return fn(*a)
        try:
            return fn(*a)
        except BaseException:
            # a sweep left half enqueued would keep the neighbours' streams
            # waiting on its flags: release them before reporting
            for c in self.ctxs:
                try:
                    c.slab_abort()
                except Exception:
                    pass
            raise

    def _run(self):
        from .solver import injection_scale

        problem, grid = self.problem, self.problem.grid
        n_steps, dt, k = problem.time.n_steps, problem.time.dt, self.config.k
        plane = grid.shape[1] * grid.shape[2]
        for c in self.ctxs:
            c.zero_accumulator()
        total = 0.0
        for source, shot in self._shots:
            g_src = grid.flat_index(source.node)
            amp = source_amplitude_table([source], dt, n_steps)
            scale = injection_scale([source], self.material, dt, self.dtype) * n_steps
            specs = []
            for c in self.ctxs:
                owned, local = localize(shot.support_idx, grid.shape, c.i_begin, c.i_end)
                order = c.set_support(local)
                kind, cc, adj_coef, meas = self._misfit_spec(shot, np.arange(len(owned)))
                if meas is not None:
                    meas = np.ascontiguousarray(meas[owned][order])
                specs.append((len(local), kind, cc, adj_coef, meas))
                c.reset_window()
            src_local = [local_source(g_src, plane, c.alloc_range, c.i_begin) for c in self.ctxs]
            self._forward_all(n_steps, src_local, amp, True, dt)
            maxima = self.halo.allreduce_max(
                np.max([c.check_maxima(n_steps) for c in self.ctxs], axis=0))
            fail, _ = first_failure_forward(maxima, n_steps, scale)
            if fail:
                raise SolverInstabilityError(*fail, detail=(
                    f"exceeds 1e6 x scale {scale:g}" if math.isfinite(fail[1]) else ""))
            cost = 0.0
            for c, (nsup, kind, cc, adj_coef, meas) in zip(self.ctxs, specs):
                if nsup:
                    cost += c.shot_misfit(n_steps, kind, meas, cc, adj_coef, True, k)
            total += self.halo.allreduce_sum(cost)
            inject = [spec[0] > 0 for spec in specs]
            src_b = [N.WO_NO_SOURCE if s is None else s for s in src_local]
            if self.whole_sweeps:
                for hi, lo in self._peer_ranges(n_steps - 1, 0, -2):
                    for c, s, inj in zip(self.ctxs, src_b, inject):
                        c.sweep_backward_range(n_steps, hi, lo, s, amp[0], inj, True, dt)
            else:
                for n in range(n_steps - 1, 0, -1):
                    self._steps(lambda c, s, inj, _n=n: c.sweep_backward_range(
                        n_steps, _n, _n - 1, s, amp[0], inj, True, dt), src_b, inject)
            maxima = self.halo.allreduce_max(
                np.max([c.check_maxima(n_steps) for c in self.ctxs], axis=0))
            fail = first_failure_backward(maxima, n_steps)
            if fail:
                from .gradients import SUPERPOSED_DETAIL

                raise SolverInstabilityError(*fail, detail=SUPERPOSED_DETAIL)
        for c in self.ctxs:
            c.gradient(2.0 * k, copy=False)
        return total

    def download(self):
        """This process's slabs of the gradient, concatenated along axis 0."""
        return np.concatenate([c.get_accumulator() for c in self.ctxs], axis=0)

    def close(self):
        if hasattr(self.halo, "close"):
            self.halo.close()
        for c in self.ctxs:
            c.close()


def gradient_superposed_slabs(problem, material, config, parts, devices=None, overlap=True,
                              halo="loopback"):
    """Single-process slab-decomposed gradient (loopback / peer halo)."""
    from .gradients import GradientResult, BufferCounter

    sg = SlabGradient(problem, material, config, slab_ranges(problem.grid.shape[0], parts),
                      devices, halo=halo, overlap=overlap).upload()
    try:
        cost = sg.run()
        grad = sg.download()
    finally:
        sg.close()
    return GradientResult(cost=cost, gradient=grad, counter=BufferCounter(problem.grid),
                          k=sg.config.k)


# --------------------------------------------------------- shot-parallel
def accumulator_tensor(ctx):
    """Zero-copy torch view of a DeviceGrid's accumulator (CUDA array interface)."""
    ptr = ctx.L.wo_accumulator_ptr(ctx.h)
    t = _device_view(ptr, ctx.grid.n_nodes * ctx.dtype.itemsize, ctx.dtype, ctx.device)
    return t.view(*ctx.grid.shape)


def reduce_plan(acc, cost, group=None):
    """Sum accumulators (in place) and costs over the process group."""
    import torch
    import torch.distributed as dist

    dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
    c = torch.tensor([cost], dtype=torch.float64, device=acc.device)
    dist.all_reduce(c, op=dist.ReduceOp.SUM, group=group)
    return float(c.item())


class ShotParallelGradient:
    """gradient_superposed split over ranks by shots (device-resident)."""

    def __init__(self, problem, material, config, rank, world, group=None):
        from .gradients import SuperposedPlan, _shot_list

        n_shots = len(_shot_list(problem))
        self.plan = SuperposedPlan(problem, material, config,
                                   shot_indices=shot_partition(n_shots, rank, world))
        self.group = group
        self.acc = None

    def upload(self):
        self.plan.upload()
        self.acc = accumulator_tensor(self.plan.ctx)
        return self

    def run(self):
        import torch

        cost = self.plan.run(finish=False)          # synchronous on the library stream
        cost = reduce_plan(self.acc, cost, self.group)
        torch.cuda.current_stream().synchronize()   # NCCL done before the library reuses acc
        self.plan.finish()
        return cost

    def download(self):
        return self.plan.download()
