"""Dev: superposed gradient with sweep graphs on / off (C1 2D 256^2 and C2 256^3)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "profiles"))
import configs  # noqa: E402
import paper_2509_15744_b200 as W  # noqa: E402
from paper_2509_15744_b200 import gradients as G  # noqa: E402

for name, make in (("C1", lambda: configs.fwi((256, 256), 3200)),
                   ("C2", lambda: configs.fwi((256, 256, 256), 1024))):
    problem, mat = make()
    for graphs in (False, True):
        plan = G.SuperposedPlan(problem, mat, W.SuperpositionConfig(k=1e13, precision="single")).upload()
        plan.ctx.set_graphs(graphs)
        ref = None
        for _ in range(3):
            plan.run()
        plan.ctx.synchronize()
        plan.ctx.timer_mark(0)
        for _ in range(5):
            plan.run()
        plan.ctx.timer_mark(1)
        g = plan.download()
        print(f"{name} graphs={graphs!s:5s} {plan.ctx.timer_elapsed_ms(0, 1) / 5:8.2f} ms/gradient "
              f"checksum {float(abs(g).sum()):.17g}", flush=True)
        plan.ctx.set_graphs(True)
