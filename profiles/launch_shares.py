"""Summarise an ncu launch list (``--metrics gpu__time_duration.sum --csv``)
into per-kernel totals and shares of the captured launches.

    python profiles/launch_shares.py launches.csv "<command line>" > launches.txt
"""

import collections
import csv
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


if __name__ == "__main__":
    main()
