"""Dev: fp64 (single-step kernel) superposed gradient on an n^3 grid."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "profiles"))
import configs  # noqa: E402
import paper_2509_15744_b200 as W  # noqa: E402

n = int(sys.argv[1])
prec = sys.argv[2] if len(sys.argv) > 2 else "double"
problem, mat = configs.fwi((n, n, n), 24)
from paper_2509_15744_b200 import engine  # noqa: E402
ctx = engine.get_context(problem.grid, W.precision_dtype(prec))
ctx.set_two_step(0)
W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=1e13, precision=prec))
