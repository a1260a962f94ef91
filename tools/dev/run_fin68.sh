#!/bin/bash
timeout 600 python -m pytest tests -m gpu -x -q -k "colour or build or csr or smoke or unaligned" 2>&1 | tail -1
export LMS_COLOUR_VERBOSE=1
for c in C4 C3 C5 C2; do REPS=2 timeout 120 python tools/time_colour.py $c 2>&1 | grep "\[colour\]" | tail -1 | sed "s/^/$c /"; done
python - <<'PY'
import sys, time, torch
sys.path.insert(0, '.')
import meshgen, paper_1606_00803_b200 as lms
m = meshgen.grid2d(1000, 1200, 0.3, seed=5)
c = [torch.from_numpy(a).cuda() for a in m["coords"]]; e = torch.from_numpy(m["elems"]).cuda()
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); g = lms.Mesh.build_csr(c, e); torch.cuda.synchronize()
    print("grid 1000x1200 build_csr ms", round((time.perf_counter() - t) * 1e3, 1)); g.close()
PY
