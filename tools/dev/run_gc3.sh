#!/bin/bash
# batched colouring: eight mirror loads per lane; mirror on/off with the batch shift
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "colour" 2>&1 | tail -1
for env in "X=1" "LMS_GC_MIRROR=0"; do for cfg in C4 C2; do
  echo "== $cfg $env"
  env $env LMS_COLOUR_VERBOSE=1 LMS_COLOUR_STATS=1 timeout 300 python tools/prof_e2e.py --config $cfg --steps 3 2>&1 | grep -E "\[colour|total" | tail -3
done; done
