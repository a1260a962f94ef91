#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2/t38.log
: > $O
b() { r=$(env "$@" python bench.py --no-e2e --no-cpu --steps 5 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['roofline']['launch_ms'])" 2>&1 | tail -1); echo "$* $r" >> $O; }
b LMS_GZ_X=0
b LMS_GZ_X=0
LMS_GZ_STATS=1 python tools/prof_one.py --schedule gz --sweeps 1 --reps 2 >> $O 2>&1
python tools/diag_c4.py random 1 2>&1 | grep -v "deg\|first" | cut -c100-300 >> $O
python -m pytest tests/test_gpu_parity.py -x -q -k "gz or C4 or C2" 2>&1 | tail -1 >> $O
