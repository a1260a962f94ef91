#!/usr/bin/env python
"""Convergence study on the B200.

For a configuration and each ordering: Alg. 1's loop (lms_smooth_until, stop
rule 5e-6) under the colour-GS schedule (GZ) and under the Jacobi
variant -- sweeps to convergence, final quality, time per iteration (sweep +
global quality + host decision) -- plus the bare sweep and quality kernels'
times and HBM fractions.  With --seq-mesh, also the oracle's storage-order
Gauss-Seidel (Alg. 1 literally, CPU) on a smaller mesh, for the iteration
count the paper's own in-place loop needs.  Prints one JSON object."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen  # noqa: E402
import paper_1606_00803_b200 as lms  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C4")
p.add_argument("--orderings", default="original,bfs,rdr,random")
p.add_argument("--eps", type=float, default=5e-6)
p.add_argument("--max", type=int, default=2000)
p.add_argument("--seq-mesh", type=int, default=0, help="n: also run the CPU oracle on an n x n grid")
a = p.parse_args()

HBM = 6543.4
m = meshgen.make_config(a.config)
coords = [torch.from_numpy(c).cuda() for c in m["coords"]]
el = torch.from_numpy(m["elems"]).cuda()
out = {"config": a.config, "eps": a.eps, "runs": []}


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


for kind in a.orderings.split(","):
    seed = 803 if kind == "random" else 0
    for sched in (("gz" if m["dim"] == 2 else "auto"), "jacobi"):
        with lms.Mesh.build_csr(coords, el) as gm:
            gm.permute(gm.order(kind, seed))
            gm.set_schedule(sched)
            inf = gm.info()
            V, nnz, dim = inf["V"], inf["nnz"], inf["dim"]
            vfree = gm.schedule_info()["n_free"]
            bsw = 4 * (V + 1) + 4 * nnz + 8 * dim * V + 8 * dim * vfree
            c0 = gm.coords()  # the relabelled initial coordinates
            gm.smooth(1)  # schedule build + warm-up (one sweep of the trajectory: re-imported below)
            gm.import_coords(c0)
            gm.global_quality()  # incidence build
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            k, hist, why = gm.smooth_until(goal=1.0, eps=a.eps, max_sweeps=a.max)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            # bare kernels
            e0 = ev()
            gm.smooth(10)
            e1 = ev()
            for _ in range(10):
                gm.global_quality()
            e2 = ev()
            torch.cuda.synchronize()
            sweep_ms = e0.elapsed_time(e1) / 10
            q_ms = e1.elapsed_time(e2) / 10
            n_el = m.n_el
            kk = m["elems"].shape[1]
            q_bytes = n_el * 4 * kk + 8 * dim * V + n_el * 8 + n_el * 4 * kk + 4 * (V + 1) + n_el * 8
            out["runs"].append({
                "ordering": kind, "schedule": sched, "sweeps": k, "stop": why, "Q0": hist[0], "Qk": hist[-1],
                "loop_s": dt, "ms_per_iteration": dt * 1e3 / max(k, 1),
                "updates_per_s_loop": vfree * k / dt if k else None,
                "sweep_us": sweep_ms * 1e3, "sweep_frac_hbm": bsw / (sweep_ms / 1e3) / 1e9 / HBM,
                "quality_us": q_ms * 1e3, "quality_alg_bytes": q_bytes,
                "quality_frac_hbm": q_bytes / (q_ms / 1e3) / 1e9 / HBM,
                "history_head": hist[:4], "history_tail": hist[-3:]})
            print(json.dumps(out["runs"][-1]), flush=True)

if a.seq_mesh:
    import oracle
    sm = meshgen.grid2d(a.seq_mesh, a.seq_mesh, 0.3)
    om = oracle.prepare(sm)
    res = {}
    for method in ("colour", "jacobi", "seq"):
        for kind in ("original", "bfs", "rdr", "random"):
            perm = oracle.order(om, kind, 803 if kind == "random" else 0)
            pm = oracle.permute_mesh(om, perm)
            t0 = time.perf_counter()
            _, qs, why = oracle.smooth_until(pm["coords"], pm, goal=1.0, eps=a.eps, max_sweeps=a.max, method=method)
            res[f"{method}/{kind}"] = {"sweeps": len(qs) - 1, "stop": why, "Qk": qs[-1],
                                       "cpu_s": time.perf_counter() - t0}
    out["oracle_grid"] = {"n": a.seq_mesh, "results": res}
    print(json.dumps(out["oracle_grid"]), flush=True)
print("RESULT " + json.dumps(out))
