#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gz" > gpurun_out/c5_tests.log 2>&1
echo rc=$? >> gpurun_out/c5_tests.log
free -g > gpurun_out/c5_free.txt
LMS_GZ_VERBOSE=1 timeout 1500 python tools/explore.py --config C5 --sweeps 6 --reps 2 --variants gz:0:1,gz:3000:1 > gpurun_out/c5_explore.log 2>&1
echo rc=$? >> gpurun_out/c5_explore.log
echo done
