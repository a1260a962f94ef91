#!/bin/bash
export LMS_GZ_VERBOSE=1 LMS_GZ_STATS=1
for br in "3 8" "2 16"; do set -- $br
  echo "BS_LOG2=$1 RR=$2"
  LMS_GZ_BS_LOG2=$1 LMS_GZ_RR=$2 timeout 300 python tools/prof_one.py --schedule gz --sweeps 1 --reps 3 2>&1 | grep "gz" | tail -4
done > gpurun_out/fin5.log 2>&1
echo done
