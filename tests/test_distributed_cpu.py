"""Multi-process host logic of the multi-GPU modes, on CPU with gloo
(world_size 2): slab halo exchange protocol, shot partition, check
combination.  The same exchange code drives NCCL on GPUs."""

import os
import socket

import numpy as np
import pytest

from paper_2509_15744_b200 import distributed as D


def test_slab_ranges_and_localize():
    assert D.slab_ranges(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert D.slab_ranges(8, 8) == [(i, i + 1) for i in range(8)]
    with pytest.raises(Exception):
        D.slab_ranges(3, 4)
    shape = (6, 4, 5)
    flat = np.array([0, 19, 20, 59, 60, 119])
    owned, local = D.localize(flat, shape, 1, 3)
    assert owned.tolist() == [False, False, True, True, False, False]
    assert local.tolist() == [0, 39]


def test_two_step_slab_decision():
    """Two-step slab passes recompute planes b-1 and b at every interior
    boundary b: a support node there keeps all slabs on single steps; so do
    slabs thinner than two planes.  Sources anywhere are fine."""
    slabs = D.slab_ranges(32, 2)                 # boundary at 16
    assert D.recomputed_planes(slabs) == {15, 16}
    plane = 16 * 64
    assert D.two_step_slabs_ok(slabs, plane, [np.array([3 * plane + 5, 28 * plane])])
    assert not D.two_step_slabs_ok(slabs, plane, [np.array([3 * plane, 15 * plane + 7])])
    assert not D.two_step_slabs_ok(slabs, plane, [np.array([16 * plane])])
    assert D.recomputed_planes(D.slab_ranges(12, 4)) == {2, 3, 5, 6, 8, 9}
    assert not D.two_step_slabs_ok([(0, 1), (1, 4)], plane, [np.array([3 * plane])])
    assert D.two_step_slabs_ok([(0, 10)], plane, [np.array([9 * plane])])   # one slab


def test_local_source_covers_ghost_planes():
    plane = 100
    # slab [10, 20) of a 40-plane grid holds planes 8..21 (two ghosts a side)
    assert D.local_source(9 * plane + 3, plane, (8, 22), 10) == -plane + 3
    assert D.local_source(21 * plane, plane, (8, 22), 10) == 11 * plane
    assert D.local_source(7 * plane, plane, (8, 22), 10) is None
    assert D.local_source(22 * plane, plane, (8, 22), 10) is None
    assert D.local_source(12 * plane + 1, plane, (8, 22), 10) == 2 * plane + 1


def test_shot_partition_covers_all():
    for world in (1, 2, 3, 8):
        got = sorted(s for r in range(world) for s in D.shot_partition(5, r, world))
        assert got == list(range(5))


def test_check_scans_follow_reference_order():
    n = 120
    m = np.zeros(n + 2)
    m[50] = 1.0
    m[100] = 5.0
    assert D.first_failure_forward(m, n, scale=1e-6)[0] == (101, 5.0)
    assert D.first_failure_forward(m, n, scale=1.0)[0] is None
    m[100] = np.nan
    assert D.first_failure_forward(m, n, 0.0)[0][0] == 101
    b = np.zeros(n + 2)
    b[50] = np.inf
    b[100] = np.inf
    assert D.first_failure_backward(b, n) == (99, np.inf)   # descending n: 100 first


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plane = 12
        # slab r holds planes [2r, 2r+2) of a 2*world-plane field: value = 100*plane + j
        field = torch.arange(2 * world * plane, dtype=torch.float64).view(2 * world, plane)
        mine = field[2 * rank:2 * rank + 2].clone()
        ghost_lo = torch.full((plane,), -1.0, dtype=torch.float64)
        ghost_hi = torch.full((plane,), -1.0, dtype=torch.float64)
        D.exchange_planes(mine[0].contiguous(), mine[1].contiguous(), ghost_lo, ghost_hi,
                          rank, world)
        ok = True
        if rank > 0:
            ok &= bool(torch.equal(ghost_lo, field[2 * rank - 1]))
        if rank < world - 1:
            ok &= bool(torch.equal(ghost_hi, field[2 * rank + 2]))
        # split-step form: start the exchange, do "interior" work, then wait
        field2 = field * 2.0
        mine2 = field2[2 * rank:2 * rank + 2].clone()
        glo2 = torch.full((plane,), -1.0, dtype=torch.float64)
        ghi2 = torch.full((plane,), -1.0, dtype=torch.float64)
        works = D.exchange_planes_async(mine2[0].contiguous(), mine2[1].contiguous(), glo2, ghi2,
                                        rank, world)
        interior = (mine2 * 0.5).sum()   # stands for the interior update
        for w in works:
            w.wait()
        ok &= float(interior) == float(mine2.sum()) * 0.5
        if rank > 0:
            ok &= bool(torch.equal(glo2, field2[2 * rank - 1]))
        if rank < world - 1:
            ok &= bool(torch.equal(ghi2, field2[2 * rank + 2]))
        # cost / maxima reductions as the slab driver does them
        c = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(c)
        mx = torch.tensor([float(rank), 3.0 - rank], dtype=torch.float64)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        ok &= float(c.item()) == world * (world + 1) / 2
        ok &= mx.tolist() == [world - 1.0, 3.0]
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_gloo(world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res


class _FakeSlab:
    """Stands in for a slab DeviceGrid: distinct fake addresses per slab."""

    def __init__(self, idx, has_lo, has_hi):
        base = 0x10000 * (idx + 1)
        self.ghost_lo = [base + b if has_lo else 0 for b in range(4)]
        self.ghost_hi = [base + 0x100 + b if has_hi else 0 for b in range(4)]
        self.flags = [base + 0x200, base + 0x204]
        self.peers = None

    def slab_ghosts(self):
        return self.ghost_lo, self.ghost_hi, self.flags

    def set_slab_peers(self, lo_ghost=None, hi_ghost=None, lo_flag=0, hi_flag=0):
        self.peers = (lo_ghost, hi_ghost, lo_flag, hi_flag)


@pytest.mark.parametrize("parts", [1, 2, 3, 5])
def test_peer_halo_wiring(parts):
    """PeerHalo hands slab i the lower neighbour's HIGH ghost planes and its
    flag [1], the upper neighbour's LOW ghost planes and its flag [0]; the
    end slabs get nothing on their open side; close() switches all off."""
    slabs = [_FakeSlab(i, i > 0, i + 1 < parts) for i in range(parts)]
    halo = D.PeerHalo(slabs)
    for i, s in enumerate(slabs):
        lo_ghost, hi_ghost, lo_flag, hi_flag = s.peers
        if i > 0:
            assert lo_ghost == slabs[i - 1].ghost_hi and lo_flag == slabs[i - 1].flags[1]
        else:
            assert lo_ghost is None and lo_flag == 0
        if i + 1 < parts:
            assert hi_ghost == slabs[i + 1].ghost_lo and hi_flag == slabs[i + 1].flags[0]
        else:
            assert hi_ghost is None and hi_flag == 0
    assert halo.begin() == []
    with pytest.raises(D.ConfigError):
        halo.exchange()
    halo.close()
    assert all(s.peers == (None, None, 0, 0) for s in slabs)


class _FakeIpcSlab(_FakeSlab):
    """A slab context whose IPC export / open round-trip is a byte encoding:
    the handle names the exporting address, the opened address is that
    address tagged as mapped (bit 40)."""

    MAPPED = 1 << 40

    def ipc_export(self, ptr):
        return ptr.to_bytes(8, "little") + b"\0" * 56, 0

    def ipc_open(self, handle, offset):
        assert len(handle) == 64
        return int.from_bytes(handle[:8], "little") + offset + self.MAPPED


def _ipc_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        slabs = [_FakeIpcSlab(i, i > 0, i + 1 < world) for i in range(world)]
        me = slabs[rank]
        halo = D.IpcPeerHalo(me, rank, world)
        lo_ghost, hi_ghost, lo_flag, hi_flag = me.peers
        m = _FakeIpcSlab.MAPPED
        ok = True
        if rank > 0:
            ok &= lo_ghost == [p + m for p in slabs[rank - 1].ghost_hi]
            ok &= lo_flag == slabs[rank - 1].flags[1] + m
        else:
            ok &= lo_ghost is None and lo_flag == 0
        if rank + 1 < world:
            ok &= hi_ghost == [p + m for p in slabs[rank + 1].ghost_lo]
            ok &= hi_flag == slabs[rank + 1].flags[0] + m
        else:
            ok &= hi_ghost is None and hi_flag == 0
        ok &= halo.begin() == []
        halo.close()
        ok &= me.peers == (None, None, 0, 0)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ipc_peer_halo_wiring_gloo(world):
    """IpcPeerHalo: one slab per rank, handles all-gathered over the group;
    rank r maps its lower neighbour's HIGH ghost planes and flag [1] and its
    upper neighbour's LOW ghost planes and flag [0]."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res


def test_for_rank_rejects_unknown_halo():
    with pytest.raises(D.ConfigError):
        D.SlabGradient.for_rank(None, None, 1e13, 0, 2, halo="shm")


def test_ipc_peer_halo_single_rank_is_inert():
    """world 1: one slab without neighbours; nothing exported, mapped or set."""
    s = _FakeIpcSlab(0, False, False)
    halo = D.IpcPeerHalo(s, 0, 1)
    assert s.peers is None and halo.begin() == []
    halo.close()
    assert s.peers is None


class _FakeSlabCtx:
    """Stands in for a slab DeviceGrid in SlabGradient.upload (no GPU)."""

    def __init__(self, fits):
        self.fits = fits
        self.two_step = None
        self.prepared = False

    def set_material(self, material, dt, gamma_local=None):
        pass

    def set_two_step(self, on):
        self.two_step = int(on)

    def prepare_two_step(self):
        self.prepared = True
        return self.fits


@pytest.mark.parametrize("fits,expect", [((True, True, True), 1), ((True, False, True), 0)])
def test_slabs_agree_on_two_step_passes(fits, expect):
    """SlabGradient.upload: every slab prepares its two-step buffers and, if
    any slab cannot hold them, two-step passes go off on every slab (their
    peer-store launches must match one for one; capi REQUIREs it)."""
    from types import SimpleNamespace

    sg = D.SlabGradient.__new__(D.SlabGradient)
    sg.ctxs = [_FakeSlabCtx(f) for f in fits]
    sg.halo = D.PeerHalo.__new__(D.PeerHalo)          # peer stores, no wiring needed
    sg.halo.ctxs = sg.ctxs
    n0 = 8 * len(fits)
    sg.all_slabs = sg.slabs = [(8 * i, 8 * i + 8) for i in range(len(fits))]
    sg.problem = SimpleNamespace(time=SimpleNamespace(dt=1e-9),
                                 grid=SimpleNamespace(shape=(n0, 16, 64)))
    sg.material = None
    sg._shots = []
    sg.upload()
    assert sg.two_step == bool(expect)
    assert all(c.two_step == expect for c in sg.ctxs)
