#!/bin/bash
for cfg in "2 17" "1 18"; do set -- $cfg; for o in original bfs; do
  LMS_GZ_PRODUCERS=$1 LMS_GZ_WORKERS=$2 LMS_GZ_VERBOSE=1 timeout 600 python tools/explore.py --config C4 --orderings $o --sweeps 24 --reps 3 --variants gz:4096:1 2>&1 | grep -oE '"us_per_sweep": [0-9.]*|Error[^"]*' | head -2 | sed "s/^/prod=$1 W=$2 $o /"
done; done
LMS_GZ_WORKERS=17 timeout 600 python -m pytest tests -m gpu -x -q -k "gz or smoke" 2>&1 | tail -1
