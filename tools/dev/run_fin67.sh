#!/bin/bash
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
LMS_GZ_VERBOSE=2 timeout 300 python tools/prof_one.py --schedule gz --sweeps 1 --reps 1 2>&1 | grep "gz build"
timeout 300 python tools/prof_e2e.py --steps 0 --loop --loop-n 20 2>&1 | grep -E "loop_steps|Error"
