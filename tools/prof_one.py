#!/usr/bin/env python
"""Dev tool: a short, deterministic run for ncu -- build a config, order,
permute, set the schedule, then lms_smooth(sweeps) `reps` times."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen  # noqa: E402
import paper_1606_00803_b200 as lms  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C4")
p.add_argument("--ordering", default="original")
p.add_argument("--schedule", default="s3")
p.add_argument("--tile", type=int, default=0)
p.add_argument("--lag", type=int, default=0)
p.add_argument("--sweeps", type=int, default=1)
p.add_argument("--reps", type=int, default=2)
p.add_argument("--tiling", default="auto")
a = p.parse_args()
m = meshgen.make_config(a.config)
gm = lms.Mesh.build_csr([torch.from_numpy(c).cuda() for c in m["coords"]], torch.from_numpy(m["elems"]).cuda())
gm.permute(gm.order(a.ordering, 803))
gm.set_schedule(a.schedule, a.tile, a.lag, tiling=a.tiling)
for _ in range(a.reps):
    gm.smooth(a.sweeps)
torch.cuda.synchronize()
print("done", gm.schedule_info())
