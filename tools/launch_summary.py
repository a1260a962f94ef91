#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

usage: python tools/launch_summary.py gpurun_out/launches.csv [--md out.md]
Prints per kernel: launches, total / mean device time and share of the total.
The times are ncu's (cold-cache, serialised): compare SHARES, not absolutes.
"""
import csv
import re
import sys
from collections import OrderedDict


def load(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r["Kernel Name"]).strip()
        rows.append((name, r["Grid Size"], r["Block Size"], float(r["Metric Value"].replace(",", ""))))
    return rows


def summarise(rows):
    agg = OrderedDict()
    for name, grid, block, ns in rows:
        a = agg.setdefault(name, {"n": 0, "ns": 0.0, "grid": grid, "block": block})
        a["n"] += 1
        a["ns"] += ns
    total = sum(a["ns"] for a in agg.values()) or 1.0
    out = ["| kernel | launches | grid | block | total ms | mean us | share |", "|---|---|---|---|---|---|---|"]
    for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
        out.append(f"| `{name}` | {a['n']} | {a['grid']} | {a['block']} | {a['ns'] / 1e6:.3f} | "
                   f"{a['ns'] / a['n'] / 1e3:.1f} | {a['ns'] / total:.1%} |")
    out.append(f"| **total** | {len(rows)} | | | {total / 1e6:.3f} | | 100% |")
    return "\n".join(out)


if __name__ == "__main__":
    table = summarise(load(sys.argv[1]))
    print(table)
    if "--md" in sys.argv:
        with open(sys.argv[sys.argv.index("--md") + 1], "w") as f:
            f.write(table + "\n")
