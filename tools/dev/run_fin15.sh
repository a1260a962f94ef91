#!/bin/bash
LMS_GC_CHUNK=128 REPS=1 timeout 300 python tools/time_colour.py C4 > gpurun_out/fin15_plain.log 2>&1 && \
LMS_GC_CHUNK=128 REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gc_seq -c 1 -o gpurun_out/gc_seq python tools/time_colour.py C4 > gpurun_out/fin15_ncu.log 2>&1
echo done
