#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gz or C4" > gpurun_out/gz16_tests.log 2>&1
echo rc=$? >> gpurun_out/gz16_tests.log
export LMS_GZ_VERBOSE=1
for u in 2 1; do for w in 22 16; do
  LMS_GZ_UPL=$u LMS_GZ_WORKERS=$w timeout 300 python tools/explore.py --config C4 --sweeps 12 --reps 2 \
    --variants gz:2500:1,gz:3600:1,gz:4096:1 > gpurun_out/gz16_explore_${u}_$w.log 2>&1
done; done
LMS_GZ_STATS=1 timeout 300 python tools/explore.py --config C4 --sweeps 2 --reps 1 --variants gz:3600:1 > gpurun_out/gz16_stats.log 2>&1
echo done
