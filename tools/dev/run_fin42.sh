#!/bin/bash
timeout 600 python -m pytest tests -m gpu -x -q -k "csr or build or smoke or colour" > gpurun_out/fin42_tests.log 2>&1; tail -1 gpurun_out/fin42_tests.log
LMS_BUILD_VERBOSE=1 timeout 300 python tools/prof_e2e.py --steps 3 2>&1 | grep -E "unique|total" | tail -4
