#!/bin/bash
# batched colouring: per-chunk batch shift (LMS_GC_SHIFT) on/off
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "colour or orderings or sweeps" 2>&1 | tail -1
for cfg in C4 C2 C5; do for sh in 1 0; do
  echo "== $cfg shift=$sh"
  LMS_GC_SHIFT=$sh LMS_COLOUR_VERBOSE=1 LMS_COLOUR_STATS=1 timeout 300 python tools/prof_e2e.py --config $cfg --steps 3 2>&1 | grep -E "\[colour|total" | tail -3
done; done
