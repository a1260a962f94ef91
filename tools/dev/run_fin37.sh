#!/bin/bash
export LMS_COLOUR_VERBOSE=1 LMS_COLOUR_STATS=1
for cfg in C4 C3 C5 C2; do for cps in 1 2; do for sw in 1024 2048 4096; do LMS_GC_CTAS_PER_SM=$cps LMS_GC_WCHUNK=$sw REPS=1 timeout 120 python tools/time_colour.py $cfg 2>&1 | grep "\[colour\]" | sed "s/^/$cfg cps=$cps /"; done; done; done > gpurun_out/fin37.log 2>&1
echo done
