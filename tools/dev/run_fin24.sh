#!/bin/bash
export LMS_COLOUR_VERBOSE=1
for cfg in C4 C3 C5; do LMS_GC_CHUNK=128 REPS=1 timeout 120 python tools/time_colour.py $cfg 2>&1 | grep "\[colour\]" | sed "s/^/$cfg /"; REPS=1 timeout 120 python tools/time_colour.py $cfg 2>&1 | grep "\[colour\]" | sed "s/^/$cfg /"; done > gpurun_out/fin24.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "colour or build or smoke" > gpurun_out/fin24_tests.log 2>&1; tail -1 gpurun_out/fin24_tests.log
echo done
