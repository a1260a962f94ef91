#!/usr/bin/env python
"""Opcode histogram (instructions executed, stall samples) of one kernel in an
ncu report; optional per-unit normalisation.
usage: python tools/ncu_sass_hist.py report.ncu-rep [units] [top]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
i = next(k for k, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[i:]))))


def f(r, k):
    try:
        return float(r.get(k) or 0)
    except ValueError:
        return 0.0


tot = sum(f(r, "Instructions Executed") for r in rows)
st = sum(f(r, "Warp Stall Sampling (All Samples)") for r in rows) or 1
print(f"warp instructions {tot:.0f} ({tot / units:.1f} per unit), stall samples {st:.0f}")
c, cs = Counter(), Counter()
for r in rows:
    op = r["Source"].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    o = o.split(".")[0]
    c[o] += f(r, "Instructions Executed")
    cs[o] += f(r, "Warp Stall Sampling (All Samples)")
for o, v in c.most_common(top):
    print(f"{o:12s} {v / tot:6.1%} {v / units:8.1f}/unit  stall {cs[o] / st:6.1%}")
