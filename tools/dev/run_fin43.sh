#!/bin/bash
for lp in 1 0; do
  echo "LANE_PLACE=$lp"
  LMS_GZ_LANE_PLACE=$lp timeout 600 python tools/explore.py --config C4 --sweeps 24 --reps 3 --variants gz:4096:1 2>&1 | grep -o '"us_per_sweep": [0-9.]*'
  LMS_GZ_LANE_PLACE=$lp LMS_GZ_VERBOSE=2 timeout 300 python tools/prof_one.py --schedule gz --sweeps 1 --reps 1 2>&1 | grep records
done > gpurun_out/fin43.log 2>&1
LMS_GZ_LANE_PLACE=0 timeout 600 python -m pytest tests -m gpu -x -q -k "gz" > gpurun_out/fin43_tests.log 2>&1; tail -1 gpurun_out/fin43_tests.log
