"""C1 (2D 256^2, N=3200) superposed gradients at one precision (dev: ncu target)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "profiles")]

import configs  # noqa: E402

problem, mat = configs.fwi((256, 256), 3200)
print(configs.rate(problem, mat, sys.argv[1] if len(sys.argv) > 1 else "single", reps=1))
