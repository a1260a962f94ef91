#!/usr/bin/env python
"""Dev tool: time lms_build_csr (CSR + boundary + colouring) on a config (CUDA events)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import meshgen
import paper_1606_00803_b200 as lms
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
m = meshgen.make_config(cfg)
coords = [torch.from_numpy(c).cuda() for c in m["coords"]]
elems = torch.from_numpy(m["elems"]).cuda()
ts = []
for r in range(int(os.environ.get("REPS", "8"))):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); g = lms.Mesh.build_csr(coords, elems); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b)); C = g.info()["C"]; g.close()
print(json.dumps({"config": cfg, "blocks": os.environ.get("LMS_JP_BLOCKS"), "threads": os.environ.get("LMS_JP_THREADS"), "build_ms": ts, "C": C}))
