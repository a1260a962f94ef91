#!/usr/bin/env python
"""Dev tool: repeated lms_build_csr_host builds (pinned and pageable, with a
bad-index error build in between) and 4-sweep smooths on a mid-size mesh; checks
every result against the first.  usage: python tools/dev/stress_host.py [N]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import meshgen
import paper_1606_00803_b200 as lms

N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
m = meshgen.grid2d(700, 600, 0.3, seed=9)
hc = [torch.from_numpy(np.ascontiguousarray(c)).pin_memory() for c in m["coords"]]
he = torch.from_numpy(np.ascontiguousarray(m["elems"])).pin_memory()
bad = he.clone(); bad[7, 2] = m.V + 3
ref = None
for k in range(N):
    src = hc if k % 2 == 0 else [t.clone() for t in hc]  # pinned / pageable
    g = lms.Mesh.build_csr_host(src, he if k % 2 == 0 else he.clone())
    g.smooth(4)
    out = torch.stack([c.cpu() for c in g.coords()])
    g.close()
    if ref is None:
        ref = out
    elif not torch.equal(out, ref):
        print("FAILED at", k); sys.exit(1)
    if k % 10 == 5:
        try:
            lms.Mesh.build_csr_host(hc, bad)
            print("FAILED: bad index accepted"); sys.exit(1)
        except lms.LMSError:
            pass
print("ok", N, "host builds")
