#!/bin/bash
export LMS_GZ_VERBOSE=1
LMS_GZ_STATS=1 timeout 300 python tools/explore.py --config C4 --sweeps 2 --reps 1 --variants gz:4096:1,gz:3600:1 > gpurun_out/gz17_stats.log 2>&1
for w in 22 20 18; do LMS_GZ_WORKERS=$w timeout 300 python tools/explore.py --config C4 --sweeps 12 --reps 3 --variants gz:4096:1 >> gpurun_out/gz17_w.log 2>&1; done
echo done
