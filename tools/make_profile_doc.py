#!/usr/bin/env python
"""Dev tool: write profiles/ncu_summary.json and profiles/round1_final_gz.md
from an ncu --set full capture of k_sweep_gz, a bench.py JSON line and launch
lists.  usage: python tools/make_profile_doc.py REP BENCH_JSON LAUNCHES_DEVICE_CSV LAUNCHES_E2E_CSV"""
import csv
import io
import json
import subprocess
import sys

sys.path.insert(0, "tools")
from launch_summary import load, summarise  # noqa: E402

rep, bench_path, l1, l2 = sys.argv[1:5]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = csv.reader(io.StringIO(out))
hdr = next(r); units = next(r); vals = next(r)
d = dict(zip(hdr, zip(vals, units)))


def f(k):
    v, u = d[k]
    v = float(v.replace(",", ""))
    return v * 1e6 if u == "Mbyte" else (v * 1e9 if u == "Gbyte" else (v * 1e3 if u == "Kbyte" else v))


keys = [k for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
tot = sum(float(d[k][0]) for k in keys if d[k][0])
stalls = sorted(((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(d[k][0]) / tot) for k in keys if d[k][0]),
                key=lambda kv: -kv[1])[:6]
rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
b = json.loads(open(bench_path).read().strip().splitlines()[-1])
bsw = b["roofline"]["b_sweep"]
summ = {"kernels": [{
    "config": "C4", "ordering": "original", "kernel": "k_sweep_gz", "sweeps": 1,
    "dram_bytes": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
    "ncu_duration_us": f("gpu__time_duration.sum"),
    "smem_wavefronts": f("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    "smem_pipe_pct": f("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    "smem_bank_conflicts": f("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    "issue_active_pct": f("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
    "l2_hit_pct": f("lts__t_sector_hit_rate.pct"),
    "source": "profiles/round1_final_gz.md: ncu --set full --clock-control none, one k_sweep_gz launch "
              f"(1 sweep; kd tiles T=4096, 64-update items, {int(f('launch__block_size'))} threads), tools/prof_one.py --schedule gz"}]}
json.dump(summ, open("profiles/ncu_summary.json", "w"), indent=1)
open("profiles/round1_final_bench.json", "w").write(json.dumps(b) + "\n")


def trunc(t, n=14):
    o = []
    for ln in t.splitlines()[:n]:
        c = ln.split("|")
        if len(c) > 2 and len(c[1]) > 90:
            c[1] = c[1][:88] + "…`"
        o.append("|".join(c))
    return "\n".join(o)


e2e = b["e2e"]
doc = f"""# Round 1 (final) — k_sweep_gz on C4, and the e2e path

Written by `tools/make_profile_doc.py` from B200 `gpurun` captures at the end of
round 1. The kernel: GZ ghost-zone sweep, kd tiles of T=4096 owned vertices,
two updates per lane (64-update items), {int(f('launch__block_size')) // 32 - 2} worker warps + region producer +
record loader ({int(f('launch__block_size'))} threads), predicated shared-memory gathers over
gap-placed rows, Markstein division from an RN(1/d) table, register-resident
loader state (DESIGN.md 6.1).

## Bench (`python bench.py`, C4 / original / 50 sweeps)

- value **{b['value'] / 1e9:.2f} G vertex-updates/s**, {b['ms_per_step']:.2f} ms per step
- roofline: achieved {b['roofline']['achieved']:.0f} GB/s of measured {b['roofline']['peak']} GB/s = **{b['roofline']['frac']:.3f}**
  ({b['roofline']['launch_ms'] * 1e3:.1f} us per sweep launch; algorithmic {bsw / 1e9:.3f} GB per sweep)
- e2e: **{e2e['value'] / 1e9:.2f} G vertex-updates/s**, {e2e['ms_per_step']:.1f} ms per step. This covers
  `{e2e["path"]}`.
  Phases (ms): {json.dumps({k: round(v, 1) for k, v in e2e['phases_ms'].items()})}
- cpu_baseline: {(f"{b['cpu_baseline']['value'] / 1e9:.3f} G vertex-updates/s on {b['cpu_baseline']['cores']} host cores ({b['cpu_baseline']['kind']}: {b['cpu_baseline']['sample']})") if b.get('cpu_baseline') else 'not run'}
- clocks {json.dumps(b['clocks'])}

Full JSON line: `profiles/round1_final_bench.json`.

## ncu --set full, one k_sweep_gz launch (1 sweep)

`ncu --set full --clock-control none --import-source on -k regex:k_sweep_gz -s 1 -c 1 python tools/prof_one.py --schedule gz --sweeps 1 --reps 2`

| metric | value |
|---|---|
| duration (cold, under ncu) | {f('gpu__time_duration.sum'):.1f} us |
| DRAM read / write | {rd / 1e6:.1f} MB / {wr / 1e6:.1f} MB ({(rd + wr) / 1e9:.3f} GB; algorithmic {bsw / 1e9:.3f} GB → {(rd + wr) / bsw:.2f}x) |
| L2 hit rate | {f('lts__t_sector_hit_rate.pct'):.1f} % |
| shared-memory data pipe | {f('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed'):.1f} % of peak ({f('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum') / 1e6:.1f} M wavefronts, {f('l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum') / 1e6:.1f} M bank conflicts) |
| issue active | {f('sm__issue_active.avg.pct_of_peak_sustained_elapsed'):.1f} % |
| warps active | {f('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} % of peak |
| registers / thread | {f('launch__registers_per_thread'):.0f} |
| top stall reasons (pc sampling) | {', '.join(f'{k} {v:.0%}' for k, v in stalls)} |

## Launch list, device-timed path (`bench.py --steps 2 --warmup 3 --no-e2e --no-cpu`)

The timed region is 50 `k_sweep_gz` launches per step (100 % of the step's
kernels); the other rows are the one-off setup.

{trunc(summarise(load(l1)))}

## Launch list, one e2e step (`tools/prof_e2e.py --steps 2 --prof`, `ncu --profile-from-start off`)

{trunc(summarise(load(l2)), 18)}
"""
open("profiles/round1_final_gz.md", "w").write(doc)
print("wrote profiles/round1_final_gz.md, profiles/ncu_summary.json, profiles/round1_final_bench.json")
