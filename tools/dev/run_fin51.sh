#!/bin/bash
for k in 1 2 3 4 5; do timeout 300 python tools/prof_e2e.py --steps 0 --loop --loop-n 40 2>&1 | grep -E "loop_steps\": 40|LMSError|Error:" | head -2; done
timeout 600 python bench.py > gpurun_out/fin51_bench.log 2>&1
