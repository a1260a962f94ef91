#!/bin/bash
for go in 0 1; do
  echo "GAP_OPEN=$go"
  LMS_GZ_GAP_OPEN=$go timeout 600 python tools/explore.py --config C4 --sweeps 24 --reps 3 --variants gz:4096:1 2>&1 | tail -1
  cmd="python tools/prof_one.py --schedule gz --sweeps 1 --reps 2"
  LMS_GZ_GAP_OPEN=$go $cmd > /dev/null 2>&1 && LMS_GZ_GAP_OPEN=$go ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,gpu__time_duration.sum --clock-control none -k regex:k_sweep_gz -s 1 -c 1 $cmd 2>&1 | grep -E "wavefronts|conflicts|duration"
done > gpurun_out/fin32.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "gz or smoke" > gpurun_out/fin32_tests.log 2>&1; tail -1 gpurun_out/fin32_tests.log
echo done
