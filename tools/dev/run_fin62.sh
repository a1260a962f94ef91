#!/bin/bash
export LMS_COLOUR_VERBOSE=1
for c in C4 C5 C2; do for w in 8 16; do LMS_GC_WARPS=$w REPS=2 timeout 120 python tools/time_colour.py $c 2>&1 | grep "\[colour\]" | tail -1 | sed "s/^/$c warps=$w /"; done; done > gpurun_out/fin62.log 2>&1
LMS_GC_WARPS=16 timeout 600 python -m pytest tests -m gpu -x -q -k "colour" 2>&1 | tail -1 >> gpurun_out/fin62.log
