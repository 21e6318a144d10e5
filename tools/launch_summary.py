"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv --log-file X.csv ...`)
into per-kernel shares of the summed device time.

    python tools/launch_summary.py X.csv "<header comment>" > X_summary.txt"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        us = float(r["Metric Value"].replace(",", "")) * scale.get(r.get("Metric Unit", "ns"), 1e-3)
        tot[name] += us
        cnt[name] += 1
    total = sum(tot.values())
    if len(sys.argv) > 2:
        print(sys.argv[2])
    print(f"# {sum(cnt.values())} launches, {total / 1e3:.1f} ms summed")
    print("share   launches  mean_us  kernel")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{100 * tot[k] / total:5.1f}%  {cnt[k]:7d}  {tot[k] / cnt[k]:8.1f}  {k}")


if __name__ == "__main__":
    main()
