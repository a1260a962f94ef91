#!/bin/bash
LMS_GZ_VERBOSE=2 timeout 300 python tools/prof_one.py --schedule gz --sweeps 1 --reps 2 > gpurun_out/fin8_gzbuild.log 2>&1
REPS=3 timeout 300 python tools/time_colour.py > gpurun_out/fin8_colour.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/fin8_bench.log 2>&1
echo done
