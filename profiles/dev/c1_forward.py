import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2509_15744_b200 as W
from paper_2509_15744_b200 import engine
n, N = 256, 3200
dx = 0.02 / 255; dt = 7.5e-9
grid = W.build_grid((n, n), dx)
mat = W.MaterialModel.rho_scaled(np.ones((n, n)), grid, rho0=2700.0, c0=6000.0)
src = W.SourceSpec(node=(128, 3), amplitude=1e12, frequency=1e6, cycles=2)
ctx = engine.get_context(grid, np.float32)
ctx.set_material(mat, dt)
amp = engine.source_amplitude_table([src], dt, N)
sf = [grid.flat_index(src.node)]
for rep in range(4):
    ctx.reset_window(); ctx.zero_accumulator()
    ctx.synchronize(); ctx.timer_mark(0)
    ctx.sweep_forward(N, sf, amp, accumulate=True, dt=dt, scale=0.0)
    ctx.timer_mark(1)
    print(rep, round(ctx.timer_elapsed_ms(0, 1), 2), "ms forward sweep")
