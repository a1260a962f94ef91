#!/usr/bin/env python
"""Dev tool: one warm e2e step of bench.py's path (H2D, build_csr, order,
permute, set_schedule, smooth(N), D2H) with per-phase wall times
(synchronised); the last step runs between cudaProfilerStart/Stop, so
`ncu --profile-from-start off` lists exactly its kernels.
usage: python tools/prof_e2e.py [--config C4] [--sweeps 50] [--schedule auto]"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import meshgen
import paper_1606_00803_b200 as lms

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--sweeps", type=int, default=50)
ap.add_argument("--schedule", default="auto")
ap.add_argument("--ordering", default="original")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--prof", action="store_true", help="bracket the last step with cudaProfilerStart/Stop")
ap.add_argument("--loop", action="store_true", help="also time bench.py-style back-to-back steps")
ap.add_argument("--loop-n", type=int, default=3, help="steps of the longer back-to-back loop")
a = ap.parse_args()
m = meshgen.make_config(a.config)
hc = [torch.from_numpy(c).pin_memory() for c in m["coords"]]
he = torch.from_numpy(m["elems"]).pin_memory()
hout = [torch.empty_like(t).pin_memory() for t in hc]
dev = torch.device("cuda")


def step(prof):
    t = [time.perf_counter()]
    def mark():
        torch.cuda.synchronize(); t.append(time.perf_counter())
    if prof:
        torch.cuda.profiler.start()
    dc = [x.to(dev, non_blocking=True) for x in hc]; de = he.to(dev, non_blocking=True); mark()
    g = lms.Mesh.build_csr(dc, de); mark()
    p = g.order(a.ordering, 0); g.permute(p); mark()
    g.set_schedule(a.schedule, 0, 0); mark()
    g.smooth(a.sweeps); mark()
    for o, h in zip(g.coords(), hout):
        h.copy_(o, non_blocking=True)
    mark()
    if prof:
        torch.cuda.profiler.stop()
    g.close()
    mark()
    names = ["h2d", "build_csr", "order+permute", "schedule", "sweeps", "d2h", "close"]
    return {n: round((t[i + 1] - t[i]) * 1e3, 2) for i, n in enumerate(names)} | {"total": round((t[-1] - t[0]) * 1e3, 2)}


for i in range(a.steps):
    print(json.dumps(step(i == a.steps - 1 and a.prof)))
# back-to-back steps without intermediate syncs (bench.py's e2e loop)
if a.loop:
    def plain():
        dc = [x.to(dev, non_blocking=True) for x in hc]; de = he.to(dev, non_blocking=True)
        g = lms.Mesh.build_csr(dc, de)
        p = g.order(a.ordering, 0); g.permute(p)
        g.set_schedule(a.schedule, 0, 0); g.smooth(a.sweeps)
        for o, h in zip(g.coords(), hout):
            h.copy_(o, non_blocking=True)
        torch.cuda.synchronize()
        g.close()
    for n in (1, a.loop_n):
        t0 = time.perf_counter()
        for _ in range(n):
            plain()
        print(json.dumps({"loop_steps": n, "ms_per_step": round((time.perf_counter() - t0) * 1e3 / n, 2)}))
