#!/bin/bash
cmd="python tools/prof_one.py --config C4 --schedule gz --sweeps 1 --reps 1"
$cmd > gpurun_out/s3_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/s3_launches.csv $cmd > gpurun_out/s3_ncu.log 2>&1
echo done
