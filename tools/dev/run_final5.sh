#!/bin/bash
timeout 900 python bench.py > gpurun_out/final5_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/final5_bench.log | python -c "import json,sys; b=json.loads(sys.stdin.read()); print(round(b['value']/1e9,2), b['e2e']['ms_per_step'], b['e2e']['step_ms'], b['cpu_baseline']['value'])"
