#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fin16_tests.log 2>&1; tail -1 gpurun_out/fin16_tests.log
timeout 600 python bench.py > gpurun_out/fin16_bench.log 2>&1
timeout 300 python tools/prof_e2e.py > gpurun_out/fin16_e2e.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/fin16_launches.csv python tools/prof_e2e.py --steps 2 --prof > gpurun_out/fin16_ncu.log 2>&1
echo done
