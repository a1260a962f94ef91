#!/usr/bin/env python
"""Per-SASS-instruction shared-memory wavefronts (actual vs ideal) from an ncu report.
usage: python tools/ncu_smem.py report.ncu-rep [top_n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
f = lambda r, k: float((r.get(k) or "0").replace(",", "") or 0)
tot = sum(f(r, "L1 Wavefronts Shared") for r in rows)
ideal = sum(f(r, "L1 Wavefronts Shared Ideal") for r in rows)
print(f"total shared wavefronts {tot:.3e}  ideal {ideal:.3e}")
for i, r in sorted(enumerate(rows), key=lambda x: -f(x[1], "L1 Wavefronts Shared"))[:top]:
    w = f(r, "L1 Wavefronts Shared")
    print(f"{w / tot:6.1%}  x{w / max(f(r, 'L1 Wavefronts Shared Ideal'), 1):4.2f}  exec {f(r, 'Instructions Executed'):10.0f}  #{i:4d} {r['Source'].strip()[:70]}")
