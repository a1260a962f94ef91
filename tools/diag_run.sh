#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2/t32_s2.log
: > $O
python - >> $O 2>&1 <<'PY'
import sys, json; sys.path.insert(0, '.')
import numpy as np, torch, meshgen, oracle, paper_1606_00803_b200 as lms
m = meshgen.make_config("C3"); om = oracle.prepare(m)
coords = [torch.from_numpy(c).cuda() for c in m["coords"]]; el = torch.from_numpy(m["elems"]).cuda()
for kind in ("bfs", "rdr", "original"):
    perm = oracle.order(om, kind, 0); pm = oracle.permute_mesh(om, perm)
    want = oracle.smooth(pm["coords"], pm["row_ptr"], pm["col"], pm["colour"], pm["C"], 3)
    for sched in ("s1", "s2"):
        with lms.Mesh.build_csr(coords, el) as gm:
            gm.permute(torch.from_numpy(perm).cuda()); gm.set_schedule(sched); gm.smooth(3)
            got = [c.cpu().numpy() for c in gm.coords()]
            ok = all(np.array_equal(a.view(np.uint64), b.view(np.uint64)) for a, b in zip(got, want))
            gm.smooth(2); torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); gm.smooth(20); b.record(); torch.cuda.synchronize()
            us = a.elapsed_time(b) / 20 * 1e3
            print(kind, sched, "bitexact", ok, "us/sweep %.1f frac %.3f" % (us, 222603068 / (us * 1e-6) / 1e9 / 6543.4), flush=True)
PY
