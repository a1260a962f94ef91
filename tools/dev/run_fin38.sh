#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fin38_tests.log 2>&1; tail -1 gpurun_out/fin38_tests.log
export LMS_COLOUR_VERBOSE=1
for cfg in C4 C3 C5 C2 C1; do REPS=1 timeout 120 python tools/time_colour.py $cfg 2>&1 | grep "\[colour\]" | sed "s/^/$cfg /"; done > gpurun_out/fin38.log 2>&1
LMS_GC_WCHUNK=8192 REPS=1 timeout 120 python tools/time_colour.py C5 2>&1 | grep "\[colour\]" | sed "s/^/C5-8192 /" >> gpurun_out/fin38.log
echo done
