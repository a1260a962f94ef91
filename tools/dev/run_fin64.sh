#!/bin/bash
for sl in 0 100 500 2000; do LMS_GC_MIRROR_SLEEP=$sl LMS_COLOUR_VERBOSE=1 REPS=2 timeout 120 python tools/time_colour.py C4 2>&1 | grep "\[colour\]" | tail -1 | sed "s/^/sleep=$sl /"; done
