#!/bin/bash
for k in 1 2; do LMS_GZ_VERBOSE=2 timeout 300 python tools/prof_one.py --schedule gz --sweeps 1 --reps 2 2>&1 | grep records | tail -1; done
timeout 600 python tools/explore.py --config C4 --sweeps 24 --reps 3 --variants gz:4096:1 2>&1 | grep -o '"us_per_sweep": [0-9.]*'
timeout 600 python -m pytest tests -m gpu -x -q -k "gz or smoke" 2>&1 | tail -1
