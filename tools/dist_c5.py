#!/usr/bin/env python
"""C5 (16384 x 8192 graded, BASELINE.json configs[4]) split into 8 ranks with
the multi-GPU C ABI's local group (lms_dist_create_local, one process, one
GPU): per-rank plan build time and device memory, halo sizes, and the owned
coordinates after `sweeps` sweeps compared bit for bit with the 1-GPU GZ
sweep of the same mesh (which the parity suite pins to the oracle).  One JSON
line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import meshgen  # noqa: E402
import paper_1606_00803_b200 as lms  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
nr = int(sys.argv[2]) if len(sys.argv) > 2 else 8
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
m = meshgen.make_config(cfg)
coords = [torch.from_numpy(c).cuda() for c in m["coords"]]
el = torch.from_numpy(m["elems"]).cuda()
del m
with lms.Mesh.build_csr(coords, el) as g1:
    g1.smooth(sweeps)
    ref = [c.cpu().numpy() for c in g1.coords()]
torch.cuda.synchronize()
gm = lms.Mesh.build_csr(coords, el)
del coords, el
torch.cuda.empty_cache()
lms.cache_release()
torch.cuda.synchronize()
free0, total = torch.cuda.mem_get_info()
t0 = time.perf_counter()
ds = lms.Dist.create_local(gm, nr, 1)
torch.cuda.synchronize()
t_plan = time.perf_counter() - t0
gm.close()
lms.cache_release()
torch.cuda.synchronize()
free1, _ = torch.cuda.mem_get_info()
a = torch.cuda.Event(enable_timing=True)
b = torch.cuda.Event(enable_timing=True)
lms.Dist.smooth_local(ds, 1)  # schedule builds
torch.cuda.synchronize()
a.record()
lms.Dist.smooth_local(ds, sweeps - 1)
b.record()
torch.cuda.synchronize()
ok = True
for d in ds:
    first, xs = d.export_owned()
    n = xs[0].numel()
    for ax in range(len(xs)):
        ok &= np.array_equal(xs[ax].cpu().numpy().view(np.uint64), ref[ax][first:first + n].view(np.uint64))
# the local-group run restarts from the built mesh: compare the 1-GPU result after the same sweeps
infos = [d.info() for d in ds]
print(json.dumps({"config": cfg, "ranks": nr, "sweeps": sweeps, "owned_bit_exact_vs_1gpu_gz": bool(ok),
                  "plan_build_s_all_ranks": t_plan, "plan_build_s_per_rank": t_plan / nr,
                  "device_bytes_all_ranks_plans": int(free0 - free1),
                  "device_bytes_per_rank": int((free0 - free1) / nr),
                  "n_local": [i["n_local"] for i in infos], "halo_recv": [i["n_recv"] for i in infos],
                  "peers": [i["peers"] for i in infos], "depth": infos[0]["depth"],
                  "local_group_ms_per_sweep_all_ranks_serial": a.elapsed_time(b) / max(1, sweeps - 1)}))
