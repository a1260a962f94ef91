#!/bin/bash
# bench e2e per-step times, twice
for k in 1 2; do timeout 900 python bench.py --no-cpu 2>&1 | tail -1 | python -c "import json,sys; b=json.loads(sys.stdin.read()); print(round(b['value']/1e9,2), b['e2e']['ms_per_step'], b['e2e']['step_ms'])"; done
