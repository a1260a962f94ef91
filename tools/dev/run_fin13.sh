#!/bin/bash
export LMS_COLOUR_VERBOSE=1
timeout 600 python -m pytest tests -m gpu -x -q -k "colour or build or smoke" > gpurun_out/fin13_tests.log 2>&1; tail -1 gpurun_out/fin13_tests.log
for cfg in C4 C3 C5; do
  for S in 64 128 256; do LMS_GC_CHUNK=$S REPS=2 timeout 300 python tools/time_colour.py $cfg 2>&1 | grep "\[colour\]" | tail -1 | sed "s/^/$cfg /"; done
done > gpurun_out/fin13_colour.log 2>&1
echo done
