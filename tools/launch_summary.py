"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: share of device
time per kernel.  Usage: python tools/launch_summary.py launches.csv [command-string]"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    rows = []
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"], float(r["Metric Value"]) / 1e3))  # ns -> us
    agg = defaultdict(lambda: [0, 0.0])
    for name, us in rows:
        short = name.split("(")[0] if not name.startswith("void cub") else name[:110]
        agg[short][0] += 1
        agg[short][1] += us
    tot = sum(v[1] for v in agg.values())
    if len(sys.argv) > 2:
        print("# command:", sys.argv[2])
    print(f"# {len(rows)} launches, {tot / 1e3:.3f} ms total device time")
    print("# share%  launches  avg_us  kernel")
    for name, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{100 * us / tot:7.2f} {c:7d} {us / c:11.2f}  {name}")


if __name__ == "__main__":
    main()
