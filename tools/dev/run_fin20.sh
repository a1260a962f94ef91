#!/bin/bash
LMS_GZ_VERBOSE=2 timeout 300 python tools/prof_e2e.py --steps 5 > gpurun_out/fin20_e2e.log 2>&1
echo done
