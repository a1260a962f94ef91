#!/bin/bash
for rr in 8 16; do for t in 4096 3600; do
  echo "RR=$rr T=$t"
  LMS_GZ_RR=$rr LMS_GZ_VERBOSE=1 timeout 600 python tools/explore.py --config C4 --sweeps 24 --reps 3 --variants gz:$t:1 2>&1 | grep -oE '^\[gz\] [a-z]+ T=[0-9]+ P=1 tiles=[0-9]+ items=[0-9]+ NB=[0-9] RR=[0-9]+|"us_per_sweep": [0-9.]*'
done; done > gpurun_out/fin60.log 2>&1
