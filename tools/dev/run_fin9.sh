#!/bin/bash
timeout 300 python tools/prof_e2e.py > gpurun_out/fin9_e2e.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/fin9_launches.csv python tools/prof_e2e.py --steps 2 --prof > gpurun_out/fin9_ncu.log 2>&1
echo done
