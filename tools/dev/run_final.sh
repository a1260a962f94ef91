#!/bin/bash
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/final_ref.log 2>&1; echo "ref rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29541 bench.py --force-dist --steps 2 --warmup 3 > gpurun_out/final_dist.log 2>&1; echo "dist rc=$?"
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 300 python tools/prof_e2e.py --steps 2 > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/final_e2e_launches.csv python tools/prof_e2e.py --steps 2 --prof > /dev/null 2>&1
cmd="python tools/prof_one.py --schedule gz --sweeps 1 --reps 2"
$cmd > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_sweep_gz -s 1 -c 1 -o gpurun_out/gz_final $cmd > /dev/null 2>&1
echo done
