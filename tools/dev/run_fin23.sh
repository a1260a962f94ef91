#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fin23_tests.log 2>&1; tail -1 gpurun_out/fin23_tests.log
LMS_GZ_VERBOSE=2 timeout 300 python tools/prof_e2e.py --steps 4 > gpurun_out/fin23_e2e.log 2>&1
echo done
