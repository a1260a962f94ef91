#!/usr/bin/env python
"""Dev tool: N back-to-back e2e steps (bench.py's path) with per-phase CUDA
events; prints every step slower than the median by > 5 ms, with its phases.
usage: python tools/dev/e2e_outliers.py [N]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import meshgen
import paper_1606_00803_b200 as lms

N = int(sys.argv[1]) if len(sys.argv) > 1 else 20
m = meshgen.make_config("C4")
hc = [torch.from_numpy(c).pin_memory() for c in m["coords"]]
he = torch.from_numpy(m["elems"]).pin_memory()
hout = [torch.empty_like(t).pin_memory() for t in hc]
dev = torch.device("cuda")
s = torch.cuda.current_stream()
names = ["h2d", "build_csr", "order+permute", "schedule+sweeps", "d2h", "close"]
rows = []
for k in range(N):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    wt = [time.perf_counter()]
    ev[0].record(s)
    dc = [x.to(dev, non_blocking=True) for x in hc]; de = he.to(dev, non_blocking=True); ev[1].record(s); wt.append(time.perf_counter())
    g = lms.Mesh.build_csr(dc, de); ev[2].record(s); wt.append(time.perf_counter())
    p = g.order("original", 0); g.permute(p); ev[3].record(s); wt.append(time.perf_counter())
    g.set_schedule("auto", 0, 0); g.smooth(50); ev[4].record(s); wt.append(time.perf_counter())
    for o, h in zip(g.coords(), hout):
        h.copy_(o, non_blocking=True)
    ev[5].record(s); wt.append(time.perf_counter())
    torch.cuda.synchronize()
    g.close(); ev[6].record(s); wt.append(time.perf_counter())
    torch.cuda.synchronize()
    ph = {n: round(ev[i].elapsed_time(ev[i + 1]), 2) for i, n in enumerate(names)}
    host = {n: round((wt[i + 1] - wt[i]) * 1e3, 2) for i, n in enumerate(names)}
    rows.append((round(ev[0].elapsed_time(ev[6]), 2), ph, host))
med = sorted(r[0] for r in rows)[len(rows) // 2]
print(json.dumps({"steps": N, "median_ms": med, "all": [r[0] for r in rows]}))
for i, (t, ph, host) in enumerate(rows):
    if t > med + 5:
        print(json.dumps({"step": i, "ms": t, "gpu": ph, "host": host}))
