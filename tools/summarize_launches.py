"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel count, total and mean device time, share of the profiled region."""

import csv
import sys
from collections import defaultdict


def main(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
        name = r["Kernel Name"]
        short = name.split("(")[0].split("<")[0].replace("void ", "")
        rows.append((short, v * scale))
    agg = defaultdict(lambda: [0, 0.0])
    for n, us in rows:
        agg[n][0] += 1
        agg[n][1] += us
    total = sum(v[1] for v in agg.values())
    print(f"{len(rows)} launches, {total / 1e3:.3f} ms device time (serialised)")
    print(f"{'kernel':48s} {'count':>6s} {'total us':>10s} {'mean us':>9s} {'share':>6s}")
    for n, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{n[:48]:48s} {c:6d} {us:10.1f} {us / c:9.2f} {100 * us / total:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
