#!/usr/bin/env python
"""Reuse-distance study on the GPU (the paper's Table III and
Eq. 2): for a mesh and each ordering, the trace of one sequential sweep, its
reuse distances (lms_reuse_distance), Table III quantiles, mean, and the Eq. 2
model with the paper's Westmere capacities (66-byte nodes) and
latencies (L2 10, L3 38, memory 175 cycles, the minimum of each
quoted range, SPEC defaults).  One JSON line per ordering."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen  # noqa: E402
import paper_1606_00803_b200 as lms  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "paper"
if name == "paper":  # Table II scale: 0.30-0.39 M vertices, ~2 triangles per vertex
    m = meshgen.grid2d(610, 610, 0.3, seed=meshgen.MESH_SEED)
else:
    m = meshgen.make_config(name)
caps = (32768 // 66, 262144 // 66, 25165824 // 66)
lat = (10, 38, 175)
coords = [torch.from_numpy(c).cuda() for c in m["coords"]]
el = torch.from_numpy(m["elems"]).cuda()
for kind in ("original", "bfs", "rdr", "random"):
    with lms.Mesh.build_csr(coords, el) as gm:
        gm.permute(gm.order(kind, 803 if kind == "random" else 0))
        tr = gm.trace()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d = lms.reuse_distance(tr, m.V)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        st = lms.reuse_stats(d, quantiles=(0.5, 0.75, 0.9, 1.0), capacities=caps)
    n = st["n"]
    n1, n2, n3 = st["n_ge"]
    m1 = n1 / n
    m2 = n2 / n1 if n1 else 0.0
    m3 = n3 / n2 if n2 else 0.0
    cost = (m1 * lat[0] + m1 * m2 * lat[1] + m1 * m2 * m3 * lat[2]) * n
    print(json.dumps({"mesh": name, "V": m.V, "ordering": kind, "accesses": n, "q50": st["quantiles"][0],
                      "q75": st["quantiles"][1], "q90": st["quantiles"][2], "max": st["quantiles"][3],
                      "mean": st["mean"], "cold": st["n_cold"], "reuse_misses_L1_L2_L3": st["n_ge"],
                      "eq2_extra_cycles": cost, "gpu_reuse_s": dt}), flush=True)
