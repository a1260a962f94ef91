#!/bin/bash
# records-build kernel: parity subset, timing, one full ncu capture
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gz or sweeps" 2>&1 | tail -1
timeout 300 python tools/prof_e2e.py --steps 3 2>&1 | tail -2
LMS_GZ_VERBOSE=1 timeout 300 python tools/explore.py --config C4 --orderings original --sweeps 24 --reps 3 --variants gz:4096:1 2>&1 | grep -oE '"us_per_sweep": [0-9.]*'
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gzd_records -c 1 -f -o gpurun_out/rec3 python tools/prof_e2e.py --steps 1 > gpurun_out/rec3.log 2>&1; echo ncu=$?
