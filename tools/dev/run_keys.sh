#!/bin/bash
# packed (tile, id) sort keys + batch-shift colouring test
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gz or sweeps or colour" 2>&1 | tail -1
LMS_GZ_VERBOSE=2 timeout 300 python tools/prof_e2e.py --steps 3 2>&1 | tail -13
for k in 1 2; do timeout 300 python tools/prof_e2e.py --steps 0 --loop --loop-n 20 2>&1 | grep -E "loop_steps|Error" | head -2; done
