#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gz or C4" > gpurun_out/gz5_tests.log 2>&1
echo rc=$? >> gpurun_out/gz5_tests.log
export LMS_GZ_VERBOSE=1
for cfg in "2 8" "2 6" "3 6" "3 5"; do
  set -- $cfg
  LMS_GZ_GROUPS=$1 LMS_GZ_WARPS=$2 timeout 300 python tools/explore.py --config C4 --sweeps 12 --reps 2 \
    --variants gz:900:1,gz:1300:1,gz:600:1 > gpurun_out/gz5_explore_$1_$2.log 2>&1
done
LMS_GZ_STATS=1 LMS_GZ_GROUPS=2 LMS_GZ_WARPS=8 timeout 300 python tools/explore.py --config C4 --sweeps 2 --reps 1 --variants gz:900:1 > gpurun_out/gz5_stats.log 2>&1

cmd="python tools/prof_one.py --schedule gz --tile 900 --lag 1 --sweeps 1 --reps 2"
$cmd > gpurun_out/prof_plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep_gz -s 1 -c 1 -o gpurun_out/gz5_prof $cmd > gpurun_out/gz5_ncu.log 2>&1
echo done
