#!/usr/bin/env python
"""Dev tool: the key metrics and top stall reasons of each kernel in an ncu
--set full capture.  usage: python tools/ncu_keys.py REP [REP...]"""
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sector_hit_rate.pct',
        'l1tex__t_sector_hit_rate.pct', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'launch__grid_size', 'launch__block_size', 'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum',
        'lts__t_sectors_srcunit_tex_op_read.sum', 'sm__inst_executed.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed']
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        print("==", rep, v[h.index("Kernel Name")][:60])
        for k in KEYS:
            if k in h:
                print("  %-60s %-12s %s" % (k, u[h.index(k)], v[h.index(k)]))
        st = []
        for i, k in enumerate(h):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    st.append((float(v[i].replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(x for x, _ in st) or 1
        print("  stalls:", ", ".join("%s %.0f%%" % (k, 100 * x / tot) for x, k in sorted(st, reverse=True)[:8]))
