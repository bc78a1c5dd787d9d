"""C1 (2D 256^2, N=3200) and C3-2D (512^2, N=2000) superposed-gradient
rates, fp32 and fp64 (dev; launch-latency-bound cases): python profiles/dev/c1_rate.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "profiles")]

import configs  # noqa: E402

for name, make in (("C1 2D 256^2 N=3200", lambda: configs.fwi((256, 256), 3200)),
                   ("C3 TATO 2D 512^2 N=2000", lambda: configs.tato((512, 512), 2000))):
    problem, mat = make()
    for prec in ("single", "double"):
        r = configs.rate(problem, mat, prec, reps=5)
        print(name, prec, round(r["gcell_upd_s"], 2), "Gcell/s", round(r["ms_per_gradient"], 3),
              "ms", flush=True)
