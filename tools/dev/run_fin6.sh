#!/bin/bash
export LMS_GZ_VERBOSE=1
timeout 600 python -m pytest tests -m gpu -x -q -k "gz or smoke or C4" > gpurun_out/fin6_tests.log 2>&1
tail -2 gpurun_out/fin6_tests.log
for br in "3 8" "2 16"; do set -- $br
  echo "BS_LOG2=$1 RR=$2"
  LMS_GZ_STATS=1 LMS_GZ_BS_LOG2=$1 LMS_GZ_RR=$2 timeout 300 python tools/prof_one.py --schedule gz --sweeps 1 --reps 2 2>&1 | grep "gz stats" | tail -2
  LMS_GZ_BS_LOG2=$1 LMS_GZ_RR=$2 timeout 300 python tools/explore.py --config C4 --sweeps 24 --reps 2 --variants gz:4096:1,gz:3000:1 2>&1 | grep -v "^\[gz\]" | tail -2
done > gpurun_out/fin6.log 2>&1
echo done
