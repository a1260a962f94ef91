#!/usr/bin/env python
"""Ordering study on the B200 (the paper's Figs. 6,
11, 12 and Sec. 5.5 on one GPU).  For a configuration and each ordering: the
ordering's cost (lms_order + lms_permute, CUDA events), the GZ sweep time and
its HBM roofline fraction (B_sweep per sweep), and the paper's own figures:
  speedup(ord) = T_ori / T_ord                     (one GPU)
  gain(algo)   = (T_algo - T_rdr) / T_algo         (algo = ori, bfs)
  reordering cost in sweeps = t_order / T_ori
One JSON object (RESULT line)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen  # noqa: E402
import paper_1606_00803_b200 as lms  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C4")
p.add_argument("--orderings", default="original,random,bfs,rbfs,rcm,rdr,rdrw")
p.add_argument("--sweeps", type=int, default=20)
p.add_argument("--reps", type=int, default=3)
a = p.parse_args()
HBM = 6543.4
m = meshgen.make_config(a.config)
coords = [torch.from_numpy(c).cuda() for c in m["coords"]]
el = torch.from_numpy(m["elems"]).cuda()


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


res = {}
for kind in a.orderings.split(","):
    with lms.Mesh.build_csr(coords, el) as gm:
        inf = gm.info()
        V, nnz, dim = inf["V"], inf["nnz"], inf["dim"]
        torch.cuda.synchronize()
        e0 = ev()
        perm = gm.order(kind, 803 if kind == "random" else 0)
        e1 = ev()
        gm.permute(perm)
        e2 = ev()
        gm.smooth(1)  # schedule build
        torch.cuda.synchronize()
        vfree = gm.schedule_info()["n_free"]
        bsw = 4 * (V + 1) + 4 * nnz + 8 * dim * V + 8 * dim * vfree
        ts = []
        for _ in range(a.reps):
            s0 = ev()
            gm.smooth(a.sweeps)
            s1 = ev()
            torch.cuda.synchronize()
            ts.append(s0.elapsed_time(s1) / a.sweeps)
        t = sorted(ts)[len(ts) // 2]
        res[kind] = {"order_ms": e0.elapsed_time(e1), "permute_ms": e1.elapsed_time(e2), "sweep_us": t * 1e3,
                     "frac_hbm": bsw / (t / 1e3) / 1e9 / HBM, "schedule": gm.schedule_info()}
        print(json.dumps({kind: res[kind]}), flush=True)
ori = res.get("original", {}).get("sweep_us")
for kind, r in res.items():
    if ori:
        r["speedup_vs_ori"] = ori / r["sweep_us"]
        r["reorder_cost_sweeps"] = (r["order_ms"] + r["permute_ms"]) * 1e3 / ori
if "rdr" in res:
    for algo in ("original", "bfs"):
        if algo in res:
            res["rdr"]["gain_vs_" + algo] = (res[algo]["sweep_us"] - res["rdr"]["sweep_us"]) / res[algo]["sweep_us"]
print("RESULT " + json.dumps({"config": a.config, "V": m.V, "sweeps": a.sweeps, "orderings": res}))
