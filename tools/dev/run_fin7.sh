#!/bin/bash
export LMS_GZ_VERBOSE=1
for rm in 4 16 64 100000; do
  echo "RUN_MIN=$rm"
  LMS_GZ_STATS=1 LMS_GZ_RUN_MIN=$rm timeout 300 python tools/prof_one.py --schedule gz --sweeps 1 --reps 2 2>&1 | grep "gz stats" | tail -2
  LMS_GZ_RUN_MIN=$rm timeout 300 python tools/explore.py --config C4 --sweeps 24 --reps 2 --variants gz:4096:1 2>&1 | tail -2
done > gpurun_out/fin7.log 2>&1
echo done
