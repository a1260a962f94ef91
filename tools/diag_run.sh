#!/bin/bash
# dev A/B harness: bench sweep-launch time under environment variants
mkdir -p gpurun_out/r2
O=${OUT:-gpurun_out/r2/ab.log}
: > $O
b() { r=$(env "$@" python bench.py --no-e2e --no-cpu --steps 5 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['roofline']['launch_ms'])" 2>&1 | tail -1); echo "$* $r" >> $O; }
for v in "$@"; do b $v; done
