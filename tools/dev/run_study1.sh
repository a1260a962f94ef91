#!/bin/bash
# ordering study + 3D schedules (dev tool)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/st_smoke.log 2>&1; echo rc=$? >> gpurun_out/st_smoke.log
timeout 1200 python tools/explore.py --config C4 --sweeps 10 --reps 2 --orderings original,bfs,random,rdr \
   --variants gz:3600:1,s1:0:0,s3:4096:0 > gpurun_out/st_c4.log 2>&1
timeout 600 python tools/explore.py --config C2 --sweeps 20 --reps 2 --orderings original,bfs,random,rdr \
   --variants gz:3600:1,gz:1600:1,s1:0:0,s3:4096:0 > gpurun_out/st_c2.log 2>&1
timeout 900 python tools/explore.py --config C3 --sweeps 10 --reps 2 --orderings original,bfs,rdr,random \
   --variants s1:0:0,s3:4096:0,gz:512:1,gz:256:1 > gpurun_out/st_c3.log 2>&1
echo done
