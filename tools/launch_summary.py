"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel:
count, total time, share.  Usage: python tools/launch_summary.py file.csv"""
import csv
import re
import sys
from collections import defaultdict


def short(name):
    name = re.sub(r"\(.*", "", name)          # drop the parameter list
    name = re.sub(r"^void ", "", name)
    return name.replace("pf::", "")


def main(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        ns = v * {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3,
                  "ms": 1e6, "msecond": 1e6}.get(unit, 1)
        rows.append((short(r["Kernel Name"]), ns))
    agg = defaultdict(lambda: [0, 0.0])
    for k, ns in rows:
        agg[k][0] += 1
        agg[k][1] += ns
    tot = sum(v[1] for v in agg.values())
    print(f"| kernel | launches | total ms | share |\n|---|---:|---:|---:|")
    for k, (c, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {c} | {ns / 1e6:.3f} | {100 * ns / tot:.1f}% |")
    print(f"| **all** | {len(rows)} | {tot / 1e6:.3f} | 100% |")


if __name__ == "__main__":
    main(sys.argv[1])
