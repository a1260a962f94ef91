#!/bin/bash
# GZ persistent kernel: parity, then a tuning sweep (dev tool)
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gz or C4" > gpurun_out/gz2_tests.log 2>&1
echo rc=$? >> gpurun_out/gz2_tests.log
export LMS_GZ_VERBOSE=1
for cfg in "2 2 6" "2 3 4" "2 2 4" "1 2 6" "3 3 4" "2 4 3"; do
  set -- $cfg
  LMS_GZ_PRODUCERS=$1 LMS_GZ_GROUPS=$2 LMS_GZ_WARPS=$3 timeout 300 python tools/explore.py --config C4 --sweeps 12 \
    --variants gz:900:1,gz:600:1,gz:1300:1,gz:600:2 > gpurun_out/gz2_explore_$1_$2_$3.log 2>&1
done
echo done
