"""Aggregate an ncu launch list (`--metrics gpu__time_duration.sum --csv`) per kernel:
launches, total / average duration, share of the listed kernel time.

    python tools/launch_summary.py gpurun_out/launches.csv > profiles/r01_launches_cfg1.txt
"""
import csv
import re
import sys
from collections import defaultdict


def short(name):
    name = re.sub(r"\(.*$", "", name.replace("void ", ""))
    return name.strip()


def main(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
                 "nsecond": 1e-3}.get(r["Metric Unit"], 1.0)
        k = short(r["Kernel Name"])
        tot[k] += float(r["Metric Value"].replace(",", "")) * scale
        cnt[k] += 1
    grand = sum(tot.values())
    print(f"# {path}: {sum(cnt.values())} launches, {grand / 1e3:.3f} ms listed kernel time "
          "(cold-cache, serialised)")
    print(f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>7s}")
    for k in sorted(tot, key=tot.get, reverse=True):
        print(f"{k:60s} {cnt[k]:8d} {tot[k]:12.1f} {tot[k] / cnt[k]:10.2f} "
              f"{tot[k] / grand:7.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
