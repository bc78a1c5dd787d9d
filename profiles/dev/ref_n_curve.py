"""The reference's own gradient_superposed (baseline/_ref waveopt, Numba,
1 process = 1 core) on the bench grid (256^3 fp32, same source / sensors /
sphere-void truth) as a function of the step count N: the CPU rate falls
with N as the wavefront's subnormal tail grows.

    python profiles/dev/ref_n_curve.py N [N ...]    (one process per N, concurrently)
"""
import json
import multiprocessing as mp
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402


def one(n_steps, q):
    R = bench.load_reference_package()
    wl = bench.workload(256, n_steps)
    problem, model = bench.build_problem(R, wl)
    cfg = R.SuperpositionConfig(k=wl["k"], precision="single")
    small = bench.workload(16, 4)
    p2, m2 = bench.build_problem(R, small)
    R.gradient_superposed(p2, m2, cfg)
    t0 = time.perf_counter()
    R.gradient_superposed(problem, model, cfg)
    el = time.perf_counter() - t0
    q.put({"n_steps": n_steps, "seconds": el,
           "gcell_upd_s": 2 * (n_steps - 1) * 256**3 / el / 1e9, "cpu": bench.cpu_model()})


if __name__ == "__main__":
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=one, args=(int(n), q)) for n in sys.argv[1:]]
    for p in ps:
        p.start()
    for _ in ps:
        print(json.dumps(q.get()), flush=True)
    for p in ps:
        p.join()
