#!/bin/bash
# batched colouring knobs with the batch shift
for env in "X=1" "LMS_GC_CTAS_PER_SM=2" "LMS_GC_WCHUNK=2048" "LMS_GC_WCHUNK=8192"; do
  echo "== $env"
  env $env LMS_COLOUR_VERBOSE=1 timeout 300 python tools/prof_e2e.py --steps 3 2>&1 | grep -E "\[colour" | tail -1
done
