#!/bin/bash
for bt in "148 256" "148 128" "296 256"; do
  set -- $bt
  LMS_JP_BLOCKS=$1 LMS_JP_THREADS=$2 timeout 300 python tools/time_colour.py C4 >> gpurun_out/colour_t.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "csr_fixed_colour or C2 or C3 or C4" > gpurun_out/colour_tests.log 2>&1; echo rc=$? >> gpurun_out/colour_tests.log
