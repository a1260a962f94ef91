#!/bin/bash
timeout 600 python -m pytest tests -m gpu -x -q -k "colour or build or smoke or csr" > gpurun_out/fin36_tests.log 2>&1; tail -1 gpurun_out/fin36_tests.log
export LMS_COLOUR_VERBOSE=1 LMS_COLOUR_STATS=1
for cfg in C4 C3 C5 C2; do for sw in 512 1024 2048; do LMS_GC_WCHUNK=$sw REPS=1 timeout 120 python tools/time_colour.py $cfg 2>&1 | grep "\[colour" | sed "s/^/$cfg /"; done; done > gpurun_out/fin36.log 2>&1
echo done
