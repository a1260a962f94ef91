#!/bin/bash
for k in 1 2 3 4 5 6; do LMS_GZ_UPL=2 LMS_GZ_WORKERS=18 timeout 300 python tools/prof_e2e.py --steps 0 --loop --loop-n 40 2>&1 | grep -E "loop_steps\": 40|LMSError|Error:" | head -2; done
timeout 600 python tools/explore.py --config C4 --sweeps 24 --reps 3 --variants gz:4096:1 2>&1 | grep -o '"us_per_sweep": [0-9.]*'
LMS_GZ_UPL=2 LMS_GZ_WORKERS=18 timeout 600 python tools/explore.py --config C4 --sweeps 24 --reps 3 --variants gz:4096:1 2>&1 | grep -o '"us_per_sweep": [0-9.]*'
timeout 600 python -m pytest tests -m gpu -x -q -k "gz or smoke" 2>&1 | tail -1
