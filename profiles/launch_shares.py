"""Summarise an ncu launch list (``--metrics gpu__time_duration.sum --csv``)
into per-kernel totals and shares of the captured launches.

    python profiles/launch_shares.py launches.csv "<command line>" [share.json] > launches.txt

With a third argument the shares are also written as JSON (bench.py reads
profiles/launch_share.json: the dominant kernel's share of the step)."""

import collections
import csv
import json
import sys


def main():
    path = sys.argv[1]
    cmd = sys.argv[2] if len(sys.argv) > 2 else ""
    rows = []
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1000.0 if unit in ("ns", "nsecond") else (v * 1000.0 if unit in ("ms", "msecond") else v)
        rows.append((r["Kernel Name"].split("(")[0], us))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for name, us in rows:
        tot[name] += us
        cnt[name] += 1
    all_us = sum(tot.values()) or 1.0
    print(f"# ncu --metrics gpu__time_duration.sum --clock-control none {cmd}")
    print(f"# per-kernel totals over {len(rows)} launches (cold-cache, serialised; "
          "shares matter, not absolutes)")
    for name in sorted(tot, key=tot.get, reverse=True):
        print(f"{name[:90]:90s} n={cnt[name]:5d} total_us={tot[name]:9.1f} "
              f"share={100 * tot[name] / all_us:5.1f}% mean_us={tot[name] / cnt[name]:7.2f}")
    if len(sys.argv) > 3:
        # kernels of one family (template instantiations) summed by base name
        fam = collections.defaultdict(lambda: [0.0, 0])
        for name in tot:
            base = name.split("<")[0]
            fam[base][0] += tot[name]
            fam[base][1] += cnt[name]
        out = {"source": f"{path} ({cmd})", "launches": len(rows),
               "kernels": {k: {"share": v[0] / all_us, "launches": v[1], "total_us": v[0]}
                           for k, v in sorted(fam.items(), key=lambda kv: -kv[1][0])}}
        with open(sys.argv[3], "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
