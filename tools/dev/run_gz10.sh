#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gz10_tests.log 2>&1
echo rc=$? >> gpurun_out/gz10_tests.log
cmd="python tools/prof_one.py --schedule gz --tile 2500 --lag 1 --sweeps 1 --reps 2"
$cmd > gpurun_out/prof_plain10.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep_gz -s 1 -c 1 -o gpurun_out/gz10_prof $cmd > gpurun_out/gz10_ncu.log 2>&1
echo done
