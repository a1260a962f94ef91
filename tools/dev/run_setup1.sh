#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s1_tests.log 2>&1
echo rc=$? >> gpurun_out/s1_tests.log
LMS_GZ_VERBOSE=2 timeout 300 python tools/explore.py --config C4 --sweeps 12 --reps 2 --variants gz:3600:1 > gpurun_out/s1_explore.log 2>&1
timeout 600 python bench.py --steps 5 --no-cpu > gpurun_out/s1_bench.log 2>&1
echo done
