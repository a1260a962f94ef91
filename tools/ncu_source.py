#!/usr/bin/env python
"""Top SASS instructions by warp-stall samples from an ncu report.
usage: python tools/ncu_source.py report.ncu-rep [top_n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
key = "Warp Stall Sampling (All Samples)"
tot = sum(float(r.get(key) or 0) for r in rows) or 1
for i, r in enumerate(rows):
    r["_i"] = i
srt = sorted(rows, key=lambda r: -float(r.get(key) or 0))
for r in srt[:top]:
    s = float(r.get(key) or 0)
    print(f"{s / tot:6.1%}  #{r['_i']:4d}  {r.get('Source', '').strip()[:100]}")
