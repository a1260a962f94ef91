#!/bin/bash
export LMS_GZ_VERBOSE=1
for rr in 8 4; do
  echo "RR=$rr"
  LMS_GZ_RR=$rr timeout 600 python tools/explore.py --config C4 --sweeps 24 --reps 2 --variants gz:4096:1,gz:4600:1,gz:5200:1,gz:6000:1 2>&1 | grep -v "^\[gz build" | cut -c1-220
done > gpurun_out/fin34.log 2>&1
echo done
