#!/bin/bash
timeout 600 python bench.py > gpurun_out/fin41_bench.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin41_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 300 python tools/prof_e2e.py --steps 2 > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/fin41_e2e_launches.csv python tools/prof_e2e.py --steps 2 --prof > /dev/null 2>&1
echo done
