#!/bin/bash
# batched colouring: mirror-loop variant timing and knobs
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "colour" 2>&1 | tail -1
for env in "X=1" "LMS_GC_MIRROR=0" "LMS_GC_MIRROR=4096" "LMS_GC_MIRROR=65536"; do
  echo "== $env"
  env $env LMS_COLOUR_VERBOSE=1 LMS_COLOUR_STATS=1 timeout 300 python tools/prof_e2e.py --steps 3 2>&1 | grep -E "\[colour|total" | tail -3
done
