#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fin28_tests.log 2>&1; tail -1 gpurun_out/fin28_tests.log
timeout 600 python bench.py > gpurun_out/fin28_bench.log 2>&1
cmd="python tools/prof_one.py --schedule gz --sweeps 1 --reps 2"
$cmd > gpurun_out/fin28_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep_gz -s 1 -c 1 -o gpurun_out/gz_fin28 $cmd > gpurun_out/fin28_ncu.log 2>&1
timeout 600 python tools/explore.py --config C5 --sweeps 8 --reps 2 --variants gz:3000:1,gz:4096:1 > gpurun_out/fin28_c5.log 2>&1
timeout 300 python tools/explore.py --config C2 --sweeps 24 --reps 3 --variants gz:4096:1 > gpurun_out/fin28_c2.log 2>&1
echo done
