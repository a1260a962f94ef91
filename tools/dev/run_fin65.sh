#!/bin/bash
export LMS_COLOUR_VERBOSE=1
for c in C4 C5 C2; do REPS=2 timeout 120 python tools/time_colour.py $c 2>&1 | grep "\[colour\]" | tail -1 | sed "s/^/$c /"; done
timeout 600 python -m pytest tests -m gpu -x -q -k "colour or build or csr or smoke" 2>&1 | tail -1
