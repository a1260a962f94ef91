#!/usr/bin/env python
"""Dev tool: C4 under one ordering, GZ sweeps vs the oracle -- mismatch stats."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import meshgen  # noqa: E402
import oracle  # noqa: E402
import paper_1606_00803_b200 as lms  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "random"
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = sys.argv[3] if len(sys.argv) > 3 else "C4"
m = meshgen.make_config(cfg)
om = oracle.prepare(m)
seed = 803 if kind == "random" else 0
perm = oracle.order(om, kind, seed)
pm = oracle.permute_mesh(om, perm)
want = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], sweeps)
gm = lms.Mesh.build_csr([torch.from_numpy(c).cuda() for c in m["coords"]], torch.from_numpy(m["elems"]).cuda())
gm.permute(torch.from_numpy(perm).cuda())
gm.smooth(sweeps)
got = [c.cpu().numpy() for c in gm.coords()]
bad = np.zeros(m.V, dtype=bool)
for a in range(2):
    bad |= got[a].view(np.uint64) != want[a].view(np.uint64)
print(kind, sweeps, gm.schedule_info(), "mismatched", int(bad.sum()), "max abs",
      max(float(np.abs(got[a] - want[a]).max()) for a in range(2)))
if bad.any():
    idx = np.nonzero(bad)[0][:10]
    print("first bad", idx, [(got[0][i], want[0][i]) for i in idx[:3]])
    deg = np.diff(pm["row_ptr"])
    print("deg of bad", np.bincount(deg[bad]))
