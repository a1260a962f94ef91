#!/bin/bash
run() { echo "--- $1"; shift; for k in 1 2 3; do env "$@" timeout 300 python tools/prof_e2e.py --steps 0 --loop --loop-n 40 2>&1 | grep -E "loop_steps\": 40|LMSError|Error:" | head -2; done; }
run default X=1
run upl1 LMS_GZ_UPL=1
run lanes LMS_GC=lanes
run nocache LMS_CACHE_GB=0
