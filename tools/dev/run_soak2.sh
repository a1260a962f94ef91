#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
for k in 1 2 3 4 5 6; do timeout 300 python tools/prof_e2e.py --steps 0 --loop --loop-n 40 2>&1 | grep -E "loop_steps\": 40|LMSError|Error:" | head -2; done
for k in 1 2; do timeout 200 python tools/dev/stress_e2e.py 100 50 2>&1 | grep -E "^ok|FAILED"; done
