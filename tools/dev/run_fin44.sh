#!/bin/bash
for upl in 1 2; do for w in 22 14; do
  echo "UPL=$upl W=$w"
  LMS_GZ_UPL=$upl LMS_GZ_WORKERS=$w LMS_GZ_VERBOSE=1 timeout 600 python tools/explore.py --config C4 --sweeps 24 --reps 2 --variants gz:4096:1,gz:3000:1 2>&1 | grep -oE '^\[gz\] [a-z]+ T=[0-9]+|"us_per_sweep": [0-9.]*'
done; done > gpurun_out/fin44.log 2>&1
LMS_GZ_UPL=2 timeout 600 python -m pytest tests -m gpu -x -q -k "gz" > gpurun_out/fin44_tests.log 2>&1; tail -1 gpurun_out/fin44_tests.log
