#!/bin/bash
# schedule-build phase timings (synchronising)
LMS_GZ_VERBOSE=2 timeout 300 python tools/prof_e2e.py --steps 2 2>&1 | tail -16
