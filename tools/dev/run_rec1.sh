#!/bin/bash
# records-build kernel: timing + one full ncu capture
timeout 300 python tools/prof_e2e.py --steps 3 2>&1 | tail -2
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gzd_records -c 1 -f -o gpurun_out/rec1 python tools/prof_e2e.py --steps 1 > gpurun_out/rec1.log 2>&1; echo ncu=$?
