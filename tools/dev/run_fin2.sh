#!/bin/bash
export LMS_GZ_VERBOSE=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fin2_tests.log 2>&1
tail -3 gpurun_out/fin2_tests.log
timeout 600 python tools/explore.py --config C4 --sweeps 24 --reps 3 --variants gz:4096:1,gz:3600:1 > gpurun_out/fin2_c4.log 2>&1
timeout 300 python tools/explore.py --config C2 --sweeps 24 --reps 3 --variants gz:4096:1 > gpurun_out/fin2_c2.log 2>&1
timeout 600 python tools/explore.py --config C5 --sweeps 12 --reps 2 --variants gz:3000:1 > gpurun_out/fin2_c5.log 2>&1
echo done
