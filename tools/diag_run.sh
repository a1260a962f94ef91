#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2/t16_diag.log
: > $O
run() { echo -n "$1 :: " >> $O; shift; env "$@" python tools/diag_c4.py random 1 2>&1 | grep -v "deg\|first" | tail -1 | cut -c120-300 >> $O; }
run NEW
run NEW
run NEW_W10 LMS_GZ_WORKERS=10
run NEW_W4 LMS_GZ_WORKERS=4
run NEW_UPL1 LMS_GZ_UPL=1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2 >> $O
python bench.py --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('bench', d['roofline']['launch_ms'], d['roofline']['frac'])" >> $O
