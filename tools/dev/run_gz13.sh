#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gz or C4" > gpurun_out/gz14_tests.log 2>&1
echo rc=$? >> gpurun_out/gz14_tests.log
export LMS_GZ_VERBOSE=1
for w in 18 22; do
  LMS_GZ_WORKERS=$w timeout 300 python tools/explore.py --config C4 --sweeps 12 --reps 2 \
    --variants gz:2500:1,gz:3000:1,gz:3600:1 > gpurun_out/gz14_explore_$w.log 2>&1
done
LMS_GZ_STATS=1 timeout 300 python tools/explore.py --config C4 --sweeps 2 --reps 1 --variants gz:3600:1 > gpurun_out/gz14_stats.log 2>&1
echo done
