#!/bin/bash
export LMS_GZ_VERBOSE=1
for sk in 0 1 2 3 4 6; do LMS_GZ_SKEW=$sk timeout 300 python tools/explore.py --config C4 --sweeps 12 --reps 3 --variants gz:4096:1 >> gpurun_out/gz21_w.log 2>&1; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -x -q -k "gz or C4 or deep" > gpurun_out/gz21_tests.log 2>&1; echo rc=$? >> gpurun_out/gz21_tests.log
