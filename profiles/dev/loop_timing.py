"""Dev: invert() iterations with the optimisation loop on the device vs the
host (256^3 FWI, fp32 gradients)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2509_15744_b200 as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 256
wl = bench.workload(n, steps)
problem, model = bench.build_problem(W, wl)
for dev in (True, False, True, False):
    t0 = time.perf_counter()
    res = W.invert(problem, k=wl["k"], iterations=4, precision="single", device_loop=dev,
                   snapshot_every=0)
    el = time.perf_counter() - t0
    its = [r["wall_time"] for r in res.log[:-1]]
    print(f"device_loop={dev!s:5s} total {el:6.2f} s  per-iteration {[round(t, 3) for t in its]}",
          flush=True)
