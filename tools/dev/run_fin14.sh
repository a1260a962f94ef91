#!/bin/bash
export LMS_COLOUR_VERBOSE=1
for cfg in C4 C3 C5 C2; do for S in 128 256; do echo "$cfg S=$S"; LMS_GC_CHUNK=$S REPS=1 timeout 120 python tools/time_colour.py $cfg 2>&1 | grep "\[colour" ; done; done > gpurun_out/fin14.log 2>&1
unset LMS_COLOUR_VERBOSE
timeout 600 python -m pytest tests -m gpu -x -q -k "colour or build or smoke" > gpurun_out/fin14_tests.log 2>&1; tail -1 gpurun_out/fin14_tests.log
echo done
