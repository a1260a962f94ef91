#!/bin/bash
for c in C2 C4 C5; do for nb in 0 1; do
  if [ $nb = 1 ]; then export LMS_GZ_NO_BALANCE=1; else unset LMS_GZ_NO_BALANCE; fi
  echo "$c nobalance=$nb"
  LMS_GZ_VERBOSE=1 timeout 600 python tools/explore.py --config $c --sweeps 12 --reps 3 --variants gz:4096:1 2>&1 | grep -oE '^\[gz\] [a-z]+ T=[0-9]+ P=1 tiles=[0-9]+|"us_per_sweep": [0-9.]*|"frac": [0-9.]*'
done; done > gpurun_out/fin61.log 2>&1
unset LMS_GZ_NO_BALANCE
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fin61_tests.log 2>&1; tail -1 gpurun_out/fin61_tests.log
