"""Dev: one superposed gradient on an n^3 FWI grid (for ncu per-pass timing)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "profiles"))
import configs  # noqa: E402
import paper_2509_15744_b200 as W  # noqa: E402

n = int(sys.argv[1])
problem, mat = configs.fwi((n, n, n), 24)
W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=1e13, precision="single"))
