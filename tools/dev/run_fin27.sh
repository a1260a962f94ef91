#!/bin/bash
LMS_GZ_VERBOSE=2 timeout 300 python tools/prof_one.py --schedule gz --sweeps 1 --reps 2 2>&1 | grep "records"
timeout 600 python -m pytest tests -m gpu -x -q -k "gz or smoke" > gpurun_out/fin27_tests.log 2>&1; tail -1 gpurun_out/fin27_tests.log
