#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gz or C4" > gpurun_out/gz18_tests.log 2>&1
echo rc=$? >> gpurun_out/gz18_tests.log
export LMS_GZ_VERBOSE=1
for w in 22 20; do LMS_GZ_WORKERS=$w timeout 300 python tools/explore.py --config C4 --sweeps 12 --reps 3 --variants gz:4096:1,gz:3600:1 >> gpurun_out/gz18_w.log 2>&1; done
echo done
