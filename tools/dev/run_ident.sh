#!/bin/bash
# identity permutation fast path
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for k in 1 2; do timeout 900 python bench.py --no-cpu 2>&1 | tail -1 | python -c "import json,sys; b=json.loads(sys.stdin.read()); print(round(b['value']/1e9,2), round(b['e2e']['value']/1e9,2), b['e2e']['ms_per_step'], b['e2e']['step_ms'], b['e2e']['phases_ms'])"; done
