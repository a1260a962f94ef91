#!/bin/bash
# records occ update + warp-aggregated first-free: parity subset, timing, e2e launch list
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gz or sweeps or colour" 2>&1 | tail -1
timeout 300 python tools/prof_e2e.py --steps 3 2>&1 | tail -2
LMS_GZ_VERBOSE=1 timeout 300 python tools/explore.py --config C4 --orderings original --sweeps 24 --reps 3 --variants gz:4096:1 2>&1 | grep -oE '"us_per_sweep": [0-9.]*'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/e2e4_launches.csv python tools/prof_e2e.py --steps 2 --prof > gpurun_out/e2e4.log 2>&1; echo ncu=$?
