"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per kernel name: launches, total / mean us, share.  python scripts/launch_summary.py file.csv"""
import csv
import collections
import sys


def load(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1000.0 if unit == "ns" else (v * 1000.0 if unit == "ms" else v)
        name = r["Kernel Name"].split("(")[0]
        rows.append((name, us))
    return rows


def main(path):
    rows = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, us in rows:
        agg[name][0] += 1
        agg[name][1] += us
    total = sum(v[1] for v in agg.values())
    print(f"{len(rows)} launches, {total:.1f} us kernel time")
    for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"  {us:10.1f} us  {100 * us / total:5.1f} %  {n:5d} x  {us / n:8.2f} us  {name[:90]}")


if __name__ == "__main__":
    main(sys.argv[1])
