#!/bin/bash
# batched colouring: re-scan from the first missing input
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "colour or sweeps_bit_exact or build_csr_host" 2>&1 | tail -1
for cfg in C4 C2; do
  LMS_COLOUR_VERBOSE=1 LMS_COLOUR_STATS=1 timeout 300 python tools/prof_e2e.py --config $cfg --steps 3 2>&1 | grep -E "\[colour" | tail -2
done
