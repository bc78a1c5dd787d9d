"""CUDA IPC plumbing of the cross-process peer ghost stores (wo_ipc_export /
wo_ipc_open, distributed.IpcPeerHalo): a second process maps a slab's ghost
plane and flag and writes them with plain stores; the owner sees the bytes.
No kernel waits on another process here (the flag-waiting path itself is
covered in one process by test_slabs_gpu.py::test_slabs_peer_stores_*)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPE, SLAB = (12, 8, 64), (4, 8)


def _mapper(handles, q):
    try:
        import torch

        from paper_2509_15744_b200 import engine
        from paper_2509_15744_b200.distributed import _device_view

        ctx = engine.DeviceGrid(engine.Grid((4, 4, 32), 1e-4), np.float32, 0)
        (hg, og), (hf, of) = handles
        ghost = ctx.ipc_open(hg, og)
        again = ctx.ipc_open(hg, og)             # one mapping per allocation
        flag = ctx.ipc_open(hf, of)
        plane = SHAPE[1] * SHAPE[2]
        _device_view(ghost, plane * 4, np.float32, 0).fill_(7.0)
        _device_view(flag, 4, np.int32, 0).fill_(3)
        torch.cuda.synchronize()
        # the mapped addresses are what wo_slab_peers gets across processes:
        # a lower slab of its own accepts them as its upper neighbour's
        lower = engine.DeviceGrid(engine.Grid(SHAPE, 1e-4), np.float32, 0, slab=(0, SLAB[0]))
        lower.set_slab_peers(hi_ghost=[ghost] * 4, hi_flag=flag)
        lower.set_slab_peers()
        lower.close()
        ctx.close()
        q.put(("ok", ghost == again))
    except Exception as e:  # noqa: BLE001 - reported to the parent
        q.put(("error", repr(e)))


def test_ipc_export_open_cross_process():
    import torch
    import torch.multiprocessing as mp

    from paper_2509_15744_b200 import _native, engine
    from paper_2509_15744_b200.distributed import _device_view

    _native.load(require_device=True)
    ctx = engine.DeviceGrid(engine.Grid(SHAPE, 1e-4), np.float32, 0, slab=SLAB)
    glo, ghi, flags = ctx.slab_ghosts()
    plane_bytes = SHAPE[1] * SHAPE[2] * 4
    h_lo, off_lo = ctx.ipc_export(glo[1])
    h_hi, off_hi = ctx.ipc_export(ghi[1])
    h_f, off_f = ctx.ipc_export(flags[1])
    assert len(h_hi) == 64 and h_lo == h_hi        # one level buffer, one allocation
    # two ghost planes per neighbour: the low ghost region starts the
    # allocation, the high one follows the slab's own planes
    assert off_lo == 0 and off_hi == (2 + SLAB[1] - SLAB[0]) * plane_bytes
    assert off_f == 4                              # in_flags[1] (parity-0 slot)
    with pytest.raises(Exception):
        ctx.ipc_export(0)

    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    p = mpc.Process(target=_mapper, args=(((h_hi, off_hi), (h_f, off_f)), q))
    p.start()
    status, detail = q.get(timeout=300)
    p.join(timeout=60)
    assert status == "ok", detail
    assert detail, "reopening a handle must reuse the mapping"
    torch.cuda.synchronize()
    got = _device_view(ghi[1], plane_bytes, np.float32, 0).cpu().numpy()
    assert np.all(got == 7.0)
    assert int(_device_view(flags[1], 4, np.int32, 0).cpu().item()) == 3
    lo = _device_view(glo[1], plane_bytes, np.float32, 0).cpu().numpy()
    assert not np.any(lo == 7.0)                   # only the mapped plane was written
    ctx.close()
