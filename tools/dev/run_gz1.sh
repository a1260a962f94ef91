#!/bin/bash
# GZ tuning sweep + one ncu capture (dev tool)
for th in 256 512; do
  LMS_GZ_THREADS=$th timeout 300 python tools/explore.py --config C4 --sweeps 12 \
    --variants gz:1600:1,gz:900:1,gz:2500:1,gz:1600:2,gz:900:2,gz:900:3,gz:600:3 > gpurun_out/gz_explore_$th.log 2>&1
done
cmd="python tools/prof_one.py --schedule gz --tile 1600 --lag 1 --sweeps 1 --reps 2"
$cmd > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep_gz -s 1 -c 1 -o gpurun_out/gz_prof $cmd > gpurun_out/gz_ncu.log 2>&1
echo done
