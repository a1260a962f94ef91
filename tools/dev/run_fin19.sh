#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fin19_tests.log 2>&1; tail -1 gpurun_out/fin19_tests.log
timeout 300 python tools/prof_e2e.py --loop > gpurun_out/fin19_e2e.log 2>&1
LMS_CSR=sort timeout 300 python tools/prof_e2e.py --steps 2 >> gpurun_out/fin19_e2e.log 2>&1
echo done
