#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fin39_tests.log 2>&1; tail -1 gpurun_out/fin39_tests.log
export LMS_COLOUR_VERBOSE=1
for cfg in C4 C3 C5 C2 C1; do REPS=2 timeout 120 python tools/time_colour.py $cfg 2>&1 | grep "\[colour\]" | sed "s/^/$cfg /"; done > gpurun_out/fin39.log 2>&1
python - >> gpurun_out/fin39.log 2>&1 <<'PY'
import sys, time, torch
sys.path.insert(0, '.')
import meshgen, paper_1606_00803_b200 as lms
for nx, ny in ((1000, 1200), (3000, 1000)):
    m = meshgen.grid2d(nx, ny, 0.3, seed=5)
    c = [torch.from_numpy(a).cuda() for a in m["coords"]]; e = torch.from_numpy(m["elems"]).cuda()
    for _ in range(2):
        torch.cuda.synchronize(); t = time.perf_counter(); g = lms.Mesh.build_csr(c, e); torch.cuda.synchronize()
        print("grid", nx, ny, "build_csr ms", round((time.perf_counter() - t) * 1e3, 1)); g.close()
PY
echo done
