#!/bin/bash
for w in 16 18 20 22; do
  echo "W=$w"
  LMS_GZ_WORKERS=$w LMS_GZ_VERBOSE=1 timeout 600 python tools/explore.py --config C4 --sweeps 24 --reps 3 --variants gz:4096:1 2>&1 | grep -oE '^\[gz\] [a-z]+ T=[0-9]+ P=1 tiles=[0-9]+ items=[0-9]+ NB=[0-9] RR=[0-9]+|"us_per_sweep": [0-9.]*'
done > gpurun_out/fin45.log 2>&1
