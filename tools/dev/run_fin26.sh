#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fin26_tests.log 2>&1; tail -1 gpurun_out/fin26_tests.log
timeout 600 python tools/explore.py --config C4 --sweeps 24 --reps 3 --variants gz:4096:1 > gpurun_out/fin26_c4.log 2>&1
LMS_GZ_VERBOSE=2 timeout 300 python tools/prof_one.py --schedule gz --sweeps 1 --reps 2 2>&1 | grep "records" >> gpurun_out/fin26_c4.log
cmd="python tools/prof_one.py --schedule gz --sweeps 1 --reps 2"
$cmd > /dev/null 2>&1 && ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_sweep_gz -s 1 -c 1 $cmd > gpurun_out/fin26_ncu.log 2>&1
echo done
