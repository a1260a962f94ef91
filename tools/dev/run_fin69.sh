#!/bin/bash
for pf in 0 1; do for upl in 2 1; do
  echo "PF=$pf UPL=$upl"
  LMS_GZ_PREFETCH=$pf LMS_GZ_UPL=$upl timeout 600 python tools/explore.py --config C4 --sweeps 24 --reps 3 --variants gz:4096:1 2>&1 | grep -o '"us_per_sweep": [0-9.]*'
done; done > gpurun_out/fin69.log 2>&1
LMS_GZ_PREFETCH=1 timeout 600 python -m pytest tests -m gpu -x -q -k "gz or smoke" > gpurun_out/fin69_tests.log 2>&1; tail -1 gpurun_out/fin69_tests.log
