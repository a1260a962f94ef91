#!/bin/bash
# round-1 evidence: bench (default), launch list, one full ncu capture of the GZ kernel
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/clocks_bench.csv &
SMI=$!
timeout 600 python bench.py > gpurun_out/bench_gz.log 2>&1; echo rc=$? >> gpurun_out/bench_gz.log
kill $SMI
cmd="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
$cmd > gpurun_out/bench_gz_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_gz.csv $cmd > gpurun_out/ncu_launch.log 2>&1
cmd2="python tools/prof_one.py --schedule gz --sweeps 1 --reps 2"
$cmd2 > gpurun_out/prof_plain_b1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep_gz -s 1 -c 1 -o gpurun_out/gz_bench_prof $cmd2 > gpurun_out/gz_bench_ncu.log 2>&1
echo done
