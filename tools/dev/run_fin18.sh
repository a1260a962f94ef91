#!/bin/bash
timeout 600 python bench.py > gpurun_out/fin18_bench.log 2>&1
cmd="python tools/prof_one.py --schedule gz --sweeps 1 --reps 2"
$cmd > gpurun_out/fin18_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep_gz -s 1 -c 1 -o gpurun_out/gz_fin18 $cmd > gpurun_out/fin18_ncu.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/fin18_b2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin18_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/fin18_ncu2.log 2>&1
echo done
