#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fin56_tests.log 2>&1; tail -1 gpurun_out/fin56_tests.log
for k in 1 2 3 4 5 6; do timeout 300 python tools/prof_e2e.py --steps 0 --loop --loop-n 40 2>&1 | grep -E "loop_steps\": 40|LMSError|Error:" | head -2; done
for k in 1 2; do timeout 200 python tools/dev/stress_e2e.py 100 50 2>&1 | grep -E "^ok|FAILED"; done
timeout 600 python bench.py > gpurun_out/fin56_bench.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
