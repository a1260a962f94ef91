#!/bin/bash
run() { echo "--- $1"; shift; for k in 1 2 3; do env "$@" timeout 200 python tools/dev/stress_e2e.py 100 5 2>&1 | grep -E "^ok|FAILED"; done; }
run upl2 LMS_GZ_UPL=2 LMS_GZ_WORKERS=18
run upl2_nocache LMS_GZ_UPL=2 LMS_GZ_WORKERS=18 LMS_CACHE_GB=0
run upl2_lanes LMS_GZ_UPL=2 LMS_GZ_WORKERS=18 LMS_GC=lanes
run upl1 X=1
