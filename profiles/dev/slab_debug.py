"""Dev: drive a peer-store slab decomposition on one GPU sweep by sweep,
polling the streams with a deadline; on a stall print every slab's flag
words and release the streams (wo_slab_abort).

    python profiles/dev/slab_debug.py [shape0 shape1 shape2 parts src_plane n_steps]
"""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
sys.path.insert(0, "tests/golden")
import paper_2509_15744_b200 as W  # noqa: E402
from paper_2509_15744_b200 import distributed as D  # noqa: E402
from paper_2509_15744_b200.distributed import SlabGradient, slab_ranges  # noqa: E402

import os  # noqa: E402

WHOLE = os.environ.get("WHOLE", "0") == "1"
args = [int(a) for a in sys.argv[1:]] or [40, 16, 128, 4, 21, 40]
shape, parts, src_plane, n_steps = tuple(args[:3]), args[3], args[4], args[5]
from test_slabs_gpu import _problem_planes  # noqa: E402

problem, mat = _problem_planes(W, shape, 7, src_plane, (2, 5, shape[0] - 3), n_steps)
cfg = W.SuperpositionConfig(k=1e13, precision="single")
ref = W.gradient_superposed(problem, mat, cfg)
sg = SlabGradient(problem, mat, cfg, slab_ranges(shape[0], parts), halo="peer").upload()
if os.environ.get("NO2") == "1":
    sg.two_step = False
    for c in sg.ctxs:
        c.set_two_step(0)
print("two_step", sg.two_step, "streams", [hex(c.stream_ptr) for c in sg.ctxs], flush=True)
flags = [c.slab_ghosts()[2] for c in sg.ctxs]


def poll(tag, deadline=8.0):
    t0 = time.time()
    streams = [torch.cuda.ExternalStream(c.stream_ptr) for c in sg.ctxs]
    while time.time() - t0 < deadline:
        done = [s.query() for s in streams]
        if all(done):
            print(f"{tag}: all streams done in {time.time() - t0:.3f}s", flush=True)
            return True
        time.sleep(0.01)
    print(f"{tag}: STALL, done = {[s.query() for s in streams]}", flush=True)
    for i, c in enumerate(sg.ctxs):
        print(f"  slab {i}: flags/sent/epoch/idle {c.slab_state()}", flush=True)
    return False


try:
    grid = problem.grid
    plane = grid.shape[1] * grid.shape[2]
    for ev in range(2):
        source, shot = sg._shots[0]
        n, dt = n_steps, problem.time.dt
        g_src = grid.flat_index(source.node)
        amp = D.source_amplitude_table([source], dt, n)
        for c in sg.ctxs:
            c.zero_accumulator()
            owned, local = D.localize(shot.support_idx, grid.shape, c.i_begin, c.i_end)
            c.set_support(local)
            c.reset_window()
        src_local = [D.local_source(g_src, plane, c.alloc_range, c.i_begin) for c in sg.ctxs]
        print("src_local", src_local, flush=True)
        if WHOLE:   # whole sweeps per slab (the multi-device order)
            for c, s in zip(sg.ctxs, src_local):
                c.sweep_forward_range(n, 1, n, [] if s is None else [s],
                                      np.zeros((0, n)) if s is None else amp, True, dt)
        else:
            sg._forward_all(n, src_local, amp, True, dt)
        if not poll(f"eval {ev} forward"):
            raise SystemExit(3)
        print("stats", [c.stats()["pair_launches"] for c in sg.ctxs], flush=True)
        sg.run()
        print(f"eval {ev} run ok; bits equal:",
              sg.download().tobytes() == ref.gradient.tobytes(), flush=True)
finally:
    for c in sg.ctxs:
        c.slab_abort()
    sg.close()
