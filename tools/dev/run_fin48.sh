#!/bin/bash
echo "--- UPL=1 loop"; LMS_GZ_UPL=1 timeout 300 python tools/prof_e2e.py --steps 1 --loop 2>&1 | grep -E "loop_steps|Error" | head -3
echo "--- UPL=2 loop, blocking"; CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/prof_e2e.py --steps 1 --loop 2>&1 | grep -E "loop_steps|Error" | head -3
echo "--- UPL=2 loop again"; timeout 300 python tools/prof_e2e.py --steps 1 --loop 2>&1 | grep -E "loop_steps|Error" | head -3
echo "--- memcheck C2 loop"; timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python tools/prof_e2e.py --config C2 --sweeps 3 --steps 1 --loop 2>&1 | grep -E "loop_steps|Error|Invalid|=========" | head -20
