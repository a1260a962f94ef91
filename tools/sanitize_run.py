#!/usr/bin/env python
"""Driver for compute-sanitizer (tools/sanitize.sh): a small mesh through every
hot kernel family -- CSR build, the in-order colouring kernels (batched and
per-thread), BFS, the RDR walk, relabelling, the GZ / S1 / S3 sweeps -- each
result checked bit-exactly against the oracle, so a sanitizer run is also a
parity run."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import meshgen  # noqa: E402
import oracle  # noqa: E402
import paper_1606_00803_b200 as lms  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
m = meshgen.grid2d(100, 100, 0.3, seed=1606) if what != "3d" else meshgen.kuhn3d(10, 0.25, seed=4)
om = oracle.prepare(m)
coords = [torch.from_numpy(c).cuda() for c in m["coords"]]
el = torch.from_numpy(np.asarray(m["elems"], dtype=np.int32)).cuda()
scheds = [("gz", 0, 1), ("gz", 300, 2), ("s1", 0, 0), ("s3", 256, 0)] if what in ("all", "3d") else [("gz", 0, 1)]
for kind in ("rdr", "bfs"):
    perm = oracle.order(om, kind, 0)
    pm = oracle.permute_mesh(om, perm)
    want = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], 3)
    for sched in scheds:
        with lms.Mesh.build_csr(coords, el) as gm:
            assert np.array_equal(gm.colour().cpu().numpy(), om["colour"])
            p = gm.order(kind)
            assert np.array_equal(p.cpu().numpy(), perm), kind
            gm.permute(p)
            gm.set_schedule(*sched)
            gm.smooth(3)
            got = [c.cpu().numpy() for c in gm.coords()]
            assert all(np.array_equal(a.view(np.uint64), b.view(np.uint64)) for a, b in zip(got, want)), (kind, sched)
torch.cuda.synchronize()
print("sanitize_run OK", what)
