#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py --no-cpu 2>&1 | tail -1 | python -c "import json,sys; b=json.loads(sys.stdin.read()); print(round(b['value']/1e9,2), b['roofline']['frac'], round(b['e2e']['value']/1e9,2), b['e2e']['ms_per_step'])"
