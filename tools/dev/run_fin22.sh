#!/bin/bash
timeout 300 python tools/prof_e2e.py --steps 16 --loop > gpurun_out/fin22_e2e.log 2>&1
LMS_CACHE_GB=0 timeout 300 python tools/prof_e2e.py --steps 8 > gpurun_out/fin22_nocache.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fin22_tests.log 2>&1; tail -1 gpurun_out/fin22_tests.log
echo done
