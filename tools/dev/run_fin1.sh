#!/bin/bash
export LMS_GZ_VERBOSE=1
timeout 600 python tools/explore.py --config C2 --sweeps 24 --reps 3 --variants gz:4096:1,gz:1600:1,gz:1600:2,gz:900:2,gz:900:4,gz:600:4 > gpurun_out/fin1_c2.log 2>&1
timeout 600 python tools/explore.py --config C4 --sweeps 24 --reps 2 --variants gz:4096:2,gz:2500:2 > gpurun_out/fin1_c4p2.log 2>&1
cmd="python tools/prof_one.py --schedule gz --sweeps 1 --reps 2"
$cmd > gpurun_out/fin1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep_gz -s 1 -c 1 -o gpurun_out/gz_fin1 $cmd > gpurun_out/fin1_ncu.log 2>&1
echo done
