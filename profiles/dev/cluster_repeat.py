import sys, numpy as np
sys.path[:0] = ['/root/repo', '/root/repo/tests', '/root/repo/tests/golden']
import paper_2509_15744_b200 as W
from paper_2509_15744_b200 import engine
import test_two_step_gpu as T
problem, mat, _, _, _ = T._problem(W, (64, 128), "rho_scaled", 40, 11)
problem = W.FwiProblem(grid=problem.grid, time=problem.time, material=mat,
                       sources=problem.sources[:1], sensors=problem.sensors, measured=problem.measured[:1])
ctx = engine.get_context(problem.grid, np.float32)
cfg = W.SuperpositionConfig(k=1e13, precision="single")
ctx.set_cluster(False); off = W.gradient_superposed(problem, mat, cfg)
ctx.set_cluster(None)
for gr in (False, True):
    ctx.set_graphs(gr)
    rs = [W.gradient_superposed(problem, mat, cfg) for _ in range(4)]
    print("graphs", gr, [r.gradient.tobytes() == off.gradient.tobytes() for r in rs], [r.cost == off.cost for r in rs])
    d = np.abs(rs[-1].gradient - off.gradient); print(" maxdiff", d.max(), "at", np.unravel_index(d.argmax(), d.shape), "n diff", (d > 0).sum())
