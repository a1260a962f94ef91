#!/usr/bin/env python
"""Write profiles/ncu_summary.json from an `ncu --set full` capture of one
k_sweep_gz launch (C4, original ordering).  The record carries the sha256 of
paper_1606_00803_b200/csrc/gz.cu at capture time: bench.py reports the
capture's DRAM bytes as roofline.traffic only while the kernel source is
unchanged.  usage: python tools/ncu_summary.py REP "how it was captured"
"""
import csv
import hashlib
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, how = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = csv.reader(io.StringIO(out))
hdr = next(r)
units = next(r)
vals = next(r)
d = dict(zip(hdr, zip(vals, units)))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "nsecond": 1e-3, "msecond": 1e3}


def f(k):
    v, u = d[k]
    return float(v.replace(",", "")) * scale.get(u, 1)


rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
with open(os.path.join(ROOT, "paper_1606_00803_b200", "csrc", "gz.cu"), "rb") as fh:
    sha = hashlib.sha256(fh.read()).hexdigest()
rec = {
    "config": "C4", "ordering": "original", "kernel": "k_sweep_gz", "sweeps": 1,
    "dram_bytes": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
    "ncu_duration_us": f("gpu__time_duration.sum"),
    "smem_wavefronts": f("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    "smem_bank_conflicts": f("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    "issue_active_pct": f("sm__inst_issued.avg.pct_of_peak_sustained_active"),
    "l2_hit_pct": f("lts__t_sector_hit_rate.pct"),
    "warp_instructions": f("smsp__inst_executed.sum"),
    "gz_cu_sha256": sha,
    "source": how,
}
path = os.path.join(ROOT, "profiles", "ncu_summary.json")
with open(path, "w") as fh:
    json.dump({"kernels": [rec]}, fh, indent=1)
print(json.dumps(rec, indent=1))
