"""Per-CTA timeline of one two-step launch (dev; needs a -DWB_T2_TIMELINE=1
library):

    python -m paper_2509_15744_b200.build_native -DWB_T2_TIMELINE=1 \\
        --out=paper_2509_15744_b200/_lib/tl.so
    WAVEB200_LIB=paper_2509_15744_b200/_lib/tl.so \\
        python profiles/dev/cta_timeline.py --grid 256 [--call 300] [--out f.json]

Runs one superposed gradient without sweep graphs; the --call-th two-step
launch dumps (start, first TMA data, end, SM) per CTA.  Prints the launch
span, CTA duration statistics per wave (CTAs grouped by start order), the
start-to-first-data latency and the idle SM-time.
"""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "profiles"))


def analyse(path):
    raw = np.fromfile(path, dtype=np.uint64)
    gx, gy, gz, chunk = (int(v) for v in raw[:4])
    t = raw[4:].reshape(-1, 4).astype(np.int64)
    t0 = t[:, 0].min()
    start, data, end, sm = t[:, 0] - t0, t[:, 1] - t0, t[:, 2] - t0, t[:, 3]
    dur = end - start
    n = len(t)
    order = np.argsort(start, kind="stable")
    n_sm = int(sm.max()) + 1
    per_sm = np.bincount(sm, minlength=n_sm)
    slots = 3 * n_sm
    waves = []
    for w in range(0, n, slots):
        idx = order[w:w + slots]
        waves.append({"ctas": int(len(idx)),
                      "start_us": [round(float(start[idx].min()) / 1e3, 2),
                                   round(float(start[idx].max()) / 1e3, 2)],
                      "dur_us_p10_50_90": [round(float(np.percentile(dur[idx], q)) / 1e3, 2)
                                           for q in (10, 50, 90)],
                      "first_data_us_p50_90": [round(float(np.percentile(
                          (data - start)[idx], q)) / 1e3, 2) for q in (50, 90)]})
    span = float(end.max())
    busy = float(dur.sum())
    return {"grid": [gx, gy, gz], "chunk": chunk, "ctas": n, "sms": n_sm,
            "ctas_per_sm_min_max": [int(per_sm.min()), int(per_sm.max())],
            "span_us": round(span / 1e3, 2),
            "slot_utilisation": round(busy / (slots * span), 3),
            "last_start_us": round(float(start.max()) / 1e3, 2),
            "first_end_us": round(float(end.min()) / 1e3, 2),
            "waves": waves}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--n-steps", type=int, default=1024)
    ap.add_argument("--call", type=int, default=300)
    ap.add_argument("--file", default="/tmp/wb_t2_timeline.bin")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    os.environ["WB_T2_TL_CALL"] = str(args.call)
    os.environ["WB_T2_TL_FILE"] = args.file
    if os.path.exists(args.file):
        os.remove(args.file)
    import configs
    import paper_2509_15744_b200 as W
    from paper_2509_15744_b200 import gradients as G

    n = args.grid
    problem, mat = configs.fwi((n, n, n), args.n_steps)
    plan = G.SuperposedPlan(problem, mat, W.SuperpositionConfig(k=1e13, precision="single"))
    plan.upload()
    plan.ctx.set_graphs(False)
    plan.run()
    plan.ctx.synchronize()
    res = analyse(args.file)
    res["grid_cells"] = n
    print(json.dumps(res, indent=1))
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
