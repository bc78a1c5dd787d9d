"""Dev: one TATO 192^3 gradient (for ncu)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "profiles"))
import configs  # noqa: E402
import paper_2509_15744_b200 as W  # noqa: E402

problem, mat = configs.tato((192, 192, 192), 60)
W.gradient_superposed(problem, mat, W.SuperpositionConfig(k=1e13, precision="single"))
print("ok")
