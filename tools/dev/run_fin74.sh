#!/bin/bash
timeout 600 python -m pytest tests -m gpu -x -q -k "gz or smoke" 2>&1 | tail -1
for pr in 2 1; do for o in original bfs; do
  LMS_GZ_PRODUCERS=$pr LMS_GZ_VERBOSE=1 timeout 600 python tools/explore.py --config C4 --orderings $o --sweeps 24 --reps 3 --variants gz:4096:1 2>&1 | grep -oE '^\[gz\] [a-z]+ T=[0-9]+ P=1 tiles=[0-9]+ items=[0-9]+ NB=[0-9]|"us_per_sweep": [0-9.]*' | paste - - | sed "s/^/prod=$pr $o /"
done; done
