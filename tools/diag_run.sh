#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2/t25_hint.log
: > $O
b() { r=$(env "$@" python bench.py --no-e2e --no-cpu --steps 5 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['roofline']['launch_ms'])" 2>&1 | tail -1); echo "$* $r" >> $O; }
b LMS_GZ_HINT=0
b LMS_GZ_HINT=1
b LMS_GZ_HINT=0
b LMS_GZ_HINT=1
