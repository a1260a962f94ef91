#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gz or C4 or C2" > gpurun_out/s2_tests.log 2>&1
echo rc=$? >> gpurun_out/s2_tests.log
LMS_GZ_VERBOSE=2 timeout 300 python tools/explore.py --config C4 --sweeps 12 --reps 2 --variants gz:3600:1 > gpurun_out/s2_explore.log 2>&1
timeout 600 python bench.py --steps 5 --no-cpu > gpurun_out/s2_bench.log 2>&1
echo done
