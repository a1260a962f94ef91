#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fin10_tests.log 2>&1
tail -2 gpurun_out/fin10_tests.log
LMS_GZ_VERBOSE=2 timeout 300 python tools/prof_one.py --schedule gz --sweeps 1 --reps 2 > gpurun_out/fin10_gzbuild.log 2>&1
timeout 300 python tools/prof_e2e.py > gpurun_out/fin10_e2e.log 2>&1
timeout 300 python tools/explore.py --config C4 --sweeps 24 --reps 2 --variants gz:4096:1 2>&1 | tail -2 >> gpurun_out/fin10_e2e.log
echo done
