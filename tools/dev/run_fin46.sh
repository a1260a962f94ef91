#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fin46_tests.log 2>&1; tail -1 gpurun_out/fin46_tests.log
timeout 600 python bench.py > gpurun_out/fin46_bench.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin46_smoke.log 2>&1; tail -1 gpurun_out/fin46_smoke.log
echo done
