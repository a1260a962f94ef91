#!/bin/bash
cmd="python tools/time_colour.py C4"
$cmd > gpurun_out/c2_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/c2_launches.csv $cmd > gpurun_out/c2_ncu.log 2>&1
echo done
