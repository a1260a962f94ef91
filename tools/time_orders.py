#!/usr/bin/env python
"""Times lms_order for each ordering on a config (CUDA events), one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen  # noqa: E402
import paper_1606_00803_b200 as lms  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
kinds = sys.argv[2].split(",") if len(sys.argv) > 2 else ["original", "random", "bfs", "rdr"]
m = meshgen.make_config(cfg)
gm = lms.Mesh.build_csr([torch.from_numpy(c).cuda() for c in m["coords"]], torch.from_numpy(m["elems"]).cuda())
out = {"config": cfg}
for k in kinds:
    for rep in range(2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        gm.order(k, 803 if k == "random" else 0)
        b.record()
        torch.cuda.synchronize()
        out[k + "_ms"] = a.elapsed_time(b)
print(json.dumps(out))
