#!/bin/bash
for b in 148 296; do LMS_JP_BLOCKS=$b timeout 300 python tools/time_colour.py C4 >> gpurun_out/colour_t3.log 2>&1; done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "csr_fixed_colour or C2 or C3 or C4 or w1" > gpurun_out/colour_tests.log 2>&1; echo rc=$? >> gpurun_out/colour_tests.log
