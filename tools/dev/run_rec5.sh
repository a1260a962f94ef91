#!/bin/bash
# records: bucket index for the region-slot lookups
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gz or sweeps or build_csr_host" 2>&1 | tail -1
LMS_GZ_VERBOSE=2 timeout 300 python tools/prof_e2e.py --steps 3 2>&1 | grep -E "records|total" | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_gzd_records -c 2 --csv python tools/prof_e2e.py --steps 2 2>/dev/null | grep -E "gzd_records" | tail -2 | awk -F'","' '{print $NF}'
LMS_GZ_VERBOSE=1 timeout 300 python tools/explore.py --config C4 --orderings original --sweeps 24 --reps 3 --variants gz:4096:1 2>&1 | grep -oE '"us_per_sweep": [0-9.]*'
