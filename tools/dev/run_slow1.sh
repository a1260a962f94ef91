#!/bin/bash
for env in "X=1" "LMS_GC_MIRROR=0" "X=2"; do
echo "== $env"
env $env LMS_COLOUR_VERBOSE=1 LMS_COLOUR_STATS=1 LMS_BUILD_VERBOSE=1 timeout 300 python tools/prof_e2e.py --steps 2 2>&1 | grep -vE "^\s*$" | head -40
done
