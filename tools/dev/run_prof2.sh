#!/bin/bash
cmd="python tools/prof_one.py --schedule gz --sweeps 1 --reps 2"
$cmd > gpurun_out/p2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep_gz -s 1 -c 1 -o gpurun_out/gz_p2 $cmd > gpurun_out/p2_ncu.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p2_tests.log 2>&1; echo rc=$? >> gpurun_out/p2_tests.log
echo done
