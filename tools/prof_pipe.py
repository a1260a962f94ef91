#!/usr/bin/env python
"""Dev tool: bench.py's two-jobs-in-flight e2e loop with host timestamps at
every API call and CUDA events per phase on each job's stream, to see which
copies overlap which kernels.  usage: python tools/prof_pipe.py [--config C4]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen  # noqa: E402
import paper_1606_00803_b200 as lms  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--sweeps", type=int, default=50)
ap.add_argument("--jobs", type=int, default=5)
a = ap.parse_args()
m = meshgen.make_config(a.config)
hc = [torch.from_numpy(c).pin_memory() for c in m["coords"]]
he = torch.from_numpy(m["elems"]).pin_memory()
strs = [torch.cuda.Stream(), torch.cuda.Stream()]
houts = [[torch.empty(m.V, dtype=torch.float64).pin_memory() for _ in range(m["dim"])] for _ in range(2)]


def run(n, log):
    keep = []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(strs[0])
    strs[1].wait_event(e0)
    for k in range(n):
        st = strs[k % 2]
        evs, hts = [], []

        def mark(name):
            e = torch.cuda.Event(enable_timing=True)
            e.record(st)
            evs.append((name, e))
            hts.append((name, (time.perf_counter() - t0) * 1e3))
        with torch.cuda.stream(st):
            mark("start")
            g = lms.Mesh.build_csr_host(hc, he)
            g.set_async_errors(True)
            mark("build")
            p = g.order("original", 0)
            g.permute(p)
            mark("order")
            g.smooth(1)
            mark("sched+1")
            g.smooth(a.sweeps - 1)
            mark("sweeps")
            out = g.coords()
            for o, h in zip(out, houts[k % 2]):
                h.copy_(o, non_blocking=True)
            mark("d2h")
        keep.append((g, out, p))
        log.append((k, evs, hts))
    torch.cuda.synchronize()
    tot = (time.perf_counter() - t0) * 1e3
    for g, _, _ in keep:
        g.check()
        g.close()
    return tot, e0


run(a.jobs, [])
log = []
tot, e0 = run(a.jobs, log)
for k, evs, hts in log:
    dev = {nm: round(e0.elapsed_time(e), 2) for nm, e in evs}
    host = {nm: round(t, 2) for nm, t in hts}
    print(json.dumps({"job": k, "stream": k % 2, "device_ms_at": dev, "host_ms_at": host}))
print(json.dumps({"total_ms": tot, "per_job_ms": tot / a.jobs}))
