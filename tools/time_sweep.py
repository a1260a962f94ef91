#!/usr/bin/env python
"""Dev tool: marginal sweep time of a schedule on a config (CUDA events).
Times lms_smooth(n1) and lms_smooth(n2) per ordering and reports
(t2 - t1) / (n2 - n1) -- the per-sweep cost without the per-call setup
(graph instantiation, layout conversion) -- and its HBM roofline fraction
against B_sweep (bench.b_sweep).  One JSON line per ordering."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen  # noqa: E402
import paper_1606_00803_b200 as lms  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C3")
p.add_argument("--orderings", default="original,bfs,rdr")
p.add_argument("--schedule", default="auto")
p.add_argument("--tile", type=int, default=0)
p.add_argument("--lag", type=int, default=0, help="GZ: sweeps per pass")
p.add_argument("--n1", type=int, default=2)
p.add_argument("--n2", type=int, default=42)
p.add_argument("--reps", type=int, default=3)
a = p.parse_args()
HBM = 6543.4
m = meshgen.make_config(a.config)
coords = [torch.from_numpy(c).cuda() for c in m["coords"]]
el = torch.from_numpy(m["elems"]).cuda()


def timed(gm, n):
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s0.record()
    gm.smooth(n)
    s1.record()
    torch.cuda.synchronize()
    return s0.elapsed_time(s1)


for kind in a.orderings.split(","):
    with lms.Mesh.build_csr(coords, el) as gm:
        inf = gm.info()
        V, nnz, dim = inf["V"], inf["nnz"], inf["dim"]
        if kind != "original":
            gm.permute(gm.order(kind, 803 if kind == "random" else 0))
        gm.set_schedule(a.schedule, a.tile, a.lag)
        gm.smooth(1)
        vfree = gm.schedule_info()["n_free"]
        bsw = 4 * (V + 1) + 4 * nnz + 8 * dim * V + 8 * dim * vfree
        per = []
        for _ in range(a.reps):
            t1, t2 = timed(gm, a.n1), timed(gm, a.n2)
            per.append((t2 - t1) / (a.n2 - a.n1))
        t = sorted(per)[len(per) // 2]
        print(json.dumps({"config": a.config, "ordering": kind, "schedule": gm.schedule_info()["kind"],
                          "sweep_us": t * 1e3, "frac_hbm": bsw / (t / 1e3) / 1e9 / HBM,
                          "call_overhead_ms": timed(gm, 1) - t, "b_sweep": bsw}), flush=True)
