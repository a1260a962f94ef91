#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for o in original bfs rdr random; do
  LMS_GZ_VERBOSE=1 timeout 600 python tools/explore.py --config C4 --orderings $o --sweeps 24 --reps 3 --variants gz:4096:1 2>&1 | grep -oE 'NPW=[0-9]|NW=[0-9]+|"us_per_sweep": [0-9.]*' | paste -sd' ' | sed "s/^/$o /"
done
for k in 1 2; do timeout 300 python tools/prof_e2e.py --steps 0 --loop --loop-n 40 2>&1 | grep -E "loop_steps\": 40|LMSError|Error:" | head -2; done
