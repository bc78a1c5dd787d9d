"""Dev: wall time of calibrate_k, batched (one forward per precision) vs one
gradient_superposed per decade, on a 3D single-shot FWI problem."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2509_15744_b200 as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
wl = bench.workload(n, 256)
problem, model = bench.build_problem(W, wl)
for batch in (True, False, True):
    t0 = time.perf_counter()
    try:
        cal = W.calibrate_k(problem, model, k_start=1e16, min_decades=4, max_decades=6,
                            batch=batch)
        what = f"k={cal.k:.1e} decades={len(cal.rows)}"
    except W.ConfigError as e:   # no admissible k: same work either way
        what = "no admissible k (" + str(e).count("rel_diff") * "." + ")"
    el = time.perf_counter() - t0
    print(f"batch={batch!s:5s} {el:7.2f} s  {what}", flush=True)
