#!/bin/bash
export LMS_GZ_VERBOSE=1
for w in 22 26 30; do for br in "3 8" "2 16" "1 32"; do set -- $br
  echo "W=$w BS_LOG2=$1 RR=$2"
  LMS_GZ_WORKERS=$w LMS_GZ_BS_LOG2=$1 LMS_GZ_RR=$2 timeout 300 python tools/explore.py --config C4 --sweeps 24 --reps 2 --variants gz:4096:1 2>&1 | tail -2
done; done > gpurun_out/fin3.log 2>&1
echo done
