#!/bin/bash
for o in original bfs rdr random; do
  timeout 900 python bench.py --ordering $o --steps 3 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 > gpurun_out/ord_$o.json
  cmd="python tools/prof_one.py --schedule auto --ordering $o --sweeps 1 --reps 2"
  $cmd > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none -k regex:k_sweep -s 1 -c 1 --csv $cmd > gpurun_out/ord_ncu_$o.csv 2>/dev/null
done
echo done
