"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel:
count, total and mean device time, share.  Usage: python tools/launch_summary.py launches.csv [skip]"""
import csv
import sys
from collections import defaultdict


def main(path, skip=0):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"], float(r["Metric Value"]), r["Metric Unit"]))
    rows = rows[skip:]
    agg = defaultdict(lambda: [0, 0.0])
    for name, v, unit in rows:
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(unit, 1.0)
        short = name.split("(")[0][:110]
        agg[short][0] += 1
        agg[short][1] += v * scale
    tot = sum(v[1] for v in agg.values())
    print(f"{len(rows)} launches, {tot:.1f} us total (cold-cache, serialised)")
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{100 * t / tot:6.2f} %  {t:10.1f} us  {n:5d} x  {t / n:9.2f} us  {name}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
