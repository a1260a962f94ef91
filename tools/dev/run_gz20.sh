#!/bin/bash
export LMS_GZ_VERBOSE=1
timeout 120 python tools/explore.py --config C1 --sweeps 4 --reps 1 --variants gz:900:1 > gpurun_out/gz20_c1.log 2>&1; echo rc=$? >> gpurun_out/gz20_c1.log
timeout 200 python tools/explore.py --config C4 --sweeps 4 --reps 1 --variants gz:4096:1 > gpurun_out/gz20_c4.log 2>&1; echo rc=$? >> gpurun_out/gz20_c4.log
echo done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -x -q -k "gz or C4 or deep" > gpurun_out/gz20_tests.log 2>&1; echo rc=$? >> gpurun_out/gz20_tests.log
for sk in 1 0; do LMS_GZ_SKEW=$sk timeout 300 python tools/explore.py --config C4 --sweeps 12 --reps 3 --variants gz:4096:1,gz:3600:1 >> gpurun_out/gz20_w.log 2>&1; done
LMS_GZ_STATS=1 timeout 300 python tools/explore.py --config C4 --sweeps 2 --reps 1 --variants gz:4096:1 > gpurun_out/gz20_stats.log 2>&1
