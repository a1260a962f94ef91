#!/bin/bash
for w in 18 20; do for k in 1 2; do LMS_GZ_WORKERS=$w timeout 600 python tools/explore.py --config C4 --sweeps 24 --reps 3 --variants gz:4096:1 2>&1 | grep -o '"us_per_sweep": [0-9.]*' | sed "s/^/W=$w /"; done; done
