"""The slab decomposition across PROCESSES (SlabGradient.for_rank, one slab
per rank as under torchrun) with real kernels: two and three ranks on the one
GPU of the box, halos staged through host memory and exchanged with gloo
send/recv (HostStagedHalo: no GPU ever waits on another process, so ranks can
share a GPU).  The gathered gradient is bitwise the one-context gradient and
the all-reduced cost matches; this runs the per-rank localisation of the
sensors and the source, the misfit on the owning rank, the cross-rank
stability / cost reductions and the plane exchange of the multi-GPU path."""

import os
import socket

import numpy as np
import pytest

from helpers import bits_equal

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(W, shape, prec, seed, mid_sensor=True):
    rng = np.random.default_rng(seed)
    dx, n_steps = 1e-4, 47
    dt = 0.45 * dx / 6000.0 / np.sqrt(3)
    grid = W.build_grid(shape, dx)
    gamma = rng.uniform(0.3, 1.0, size=shape)
    mat = W.MaterialModel.rho_scaled(gamma, grid, rho0=2700.0, c0=6000.0)
    srcs = [W.SourceSpec(node=(shape[0] // 2, 5, 9), amplitude=1e12, frequency=5e6, cycles=2)]
    planes = (1, shape[0] // 2 - 1, shape[0] - 2) if mid_sensor else (1, shape[0] - 2)
    sens = sorted({(i, j, k) for i in planes
                   for j in (0, shape[1] - 1) for k in (3, shape[2] - 4)})
    meas = rng.normal(scale=1e-10, size=(1, len(sens), n_steps))
    problem = W.FwiProblem(grid=grid, time=W.TimeConfig(n_steps, dt), material=mat,
                           sources=srcs, sensors=W.SensorArray(nodes=sens), measured=meas)
    return problem, mat, W.SuperpositionConfig(k=1e13, precision=prec)


def _rank(rank, world, port, shape, prec, seed, q, halo="staged", mid_sensor=True):
    try:
        import torch.distributed as dist

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2509_15744_b200 as W
        from paper_2509_15744_b200.distributed import SlabGradient

        problem, mat, cfg = _problem(W, shape, prec, seed, mid_sensor)
        sg = SlabGradient.for_rank(problem, mat, cfg, rank, world, device=0, halo=halo)
        sg.upload()
        q.put((rank, "two_step", bool(sg.two_step), None))
        costs = [sg.run() for _ in range(2)]
        grad = sg.download()
        sg.close()
        dist.destroy_process_group()
        q.put((rank, costs, grad, sg.slabs[0]))
    except Exception as e:  # noqa: BLE001 - reported to the parent
        import traceback

        q.put((rank, "error", traceback.format_exc(), repr(e)))


@pytest.mark.parametrize("world,shape,prec", [(2, (20, 8, 32), "single"),
                                              (3, (21, 16, 24), "double")])
def test_slab_ranks_across_processes_bitwise(world, shape, prec):
    import multiprocessing as mp

    import paper_2509_15744_b200 as W
    from paper_2509_15744_b200 import _native

    _native.load(require_device=True)
    seed = sum(shape) + world
    problem, mat, cfg = _problem(W, shape, prec, seed)
    ref = W.gradient_superposed(problem, mat, cfg)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank, args=(r, world, port, shape, prec, seed, q))
          for r in range(world)]
    for p in ps:
        p.start()
    out = {}
    try:
        while len(out) < world:
            r, costs, grad, slab = q.get(timeout=300)
            assert costs != "error", grad
            if costs == "two_step":
                continue
            out[r] = (costs, grad, slab)
    finally:
        for p in ps:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    got = np.concatenate([out[r][1] for r in range(world)], axis=0)
    assert [out[r][2] for r in range(world)][0][0] == 0
    assert bits_equal(got, ref.gradient)
    for r in range(world):
        for c in out[r][0]:
            assert abs(c - ref.cost) <= 1e-13 * abs(ref.cost)


@pytest.mark.parametrize("world,shape,prec", [(2, (24, 16, 64), "single"),
                                              (3, (36, 16, 64), "double")])
def test_ipc_peer_store_ranks_across_processes_bitwise(world, shape, prec):
    """Ranks (processes) on the one GPU with CUDA-IPC peer ghost stores
    (IpcPeerHalo, the production multi-GPU path): whole sweeps with two-step
    passes whose launches store into the other processes' mapped ghost
    planes and wait on their flags (on the stream; nothing spins on an SM);
    a middle rank with two neighbours at world 3.  Bitwise the one-context
    gradient."""
    import multiprocessing as mp

    import paper_2509_15744_b200 as W
    from paper_2509_15744_b200 import _native

    _native.load(require_device=True)
    seed = 99 + world
    problem, mat, cfg = _problem(W, shape, prec, seed, mid_sensor=False)
    ref = W.gradient_superposed(problem, mat, cfg)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank, args=(r, world, port, shape, prec, seed, q, "ipc", False))
          for r in range(world)]
    for p in ps:
        p.start()
    out, two = {}, {}
    try:
        while len(out) < world:
            r, costs, grad, slab = q.get(timeout=120)
            assert costs != "error", grad
            if costs == "two_step":
                two[r] = grad
                continue
            out[r] = (costs, grad, slab)
    finally:
        for p in ps:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    assert all(two.values())
    got = np.concatenate([out[r][1] for r in range(world)], axis=0)
    assert bits_equal(got, ref.gradient)
    for r in range(world):
        for c in out[r][0]:
            assert abs(c - ref.cost) <= 1e-13 * abs(ref.cost)
