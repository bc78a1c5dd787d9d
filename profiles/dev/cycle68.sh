# run_forward history read-back through the pinned staging download
out=gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > $out/c69_tests.log 2>&1; echo "tests rc $?"; tail -4 $out/c69_tests.log
python - > $out/c69_hist_timing.txt 2>&1 <<'PY'
import time, numpy as np, paper_2509_15744_b200 as W
from paper_2509_15744_b200 import solver
for shape, n in (((256, 256), 800), ((96, 96, 96), 200)):
    grid = W.build_grid(shape, 2e-4); dt = 0.45 * 2e-4 / 6000 / np.sqrt(len(shape))
    mat = W.MaterialModel.rho_scaled(np.ones(shape), grid, rho0=2700.0, c0=6000.0)
    src = W.SourceSpec(node=tuple(s // 2 for s in shape), amplitude=1e12, frequency=3e6, cycles=2)
    for prec in (np.float32, np.float64):
        for fused in (True, False):
            solver.MAX_KERNEL_SOURCES = 8 if fused else 0
            cnt = [0]
            def cb(k, u): cnt[0] += 1
            W.run_forward(mat, W.TimeConfig(n, dt), [src], None, dtype=prec, on_step=cb)
            t = time.perf_counter()
            W.run_forward(mat, W.TimeConfig(n, dt), [src], None, dtype=prec, on_step=cb)
            ms = (time.perf_counter() - t) * 1e3
            print(shape, np.dtype(prec).name, "fused" if fused else "per-step", round(ms, 1), "ms", round(ms / (n - 1) * 1e3, 1), "us/step")
PY
cat $out/c69_hist_timing.txt
