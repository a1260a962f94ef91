#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fin11_tests.log 2>&1
tail -2 gpurun_out/fin11_tests.log
for cfg in C4 C3 C5; do
  for S in 64 128 256; do echo "cfg=$cfg S=$S"; LMS_GC_CHUNK=$S REPS=3 timeout 300 python tools/time_colour.py $cfg 2>&1 | tail -1; done
  echo "cfg=$cfg jp"; LMS_COLOUR=jp REPS=2 timeout 300 python tools/time_colour.py $cfg 2>&1 | tail -1
done > gpurun_out/fin11_colour.log 2>&1
echo done
