#!/bin/bash
# One GPU call for a round's evidence (run from the repo root under gpurun):
# the GPU suite, the suite again on the bounds-checked build, the bench line,
# the reference arm, the bench's ncu launch list, one ncu --set full capture
# of the sweep kernel, and the ordering study on C4 / CP.  Logs -> $OUT.
set -u
OUT=${OUT:-gpurun_out/final}
mkdir -p "$OUT"
timeout 2400 python -m pytest tests -m gpu -q > "$OUT/gpu_tests.log" 2>&1
LMS_LIB_PATH=$PWD/paper_1606_00803_b200/liblms_bounds.so timeout 2400 python -m pytest tests -m gpu -q > "$OUT/gpu_tests_bounds.log" 2>&1
python bench.py > "$OUT/bench.log" 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > "$OUT/bench_reference.log" 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file "$OUT/launches_bench.csv" \
  python bench.py --steps 2 --warmup 1 > "$OUT/ncu_launch.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_gz -s 1 -c 1 -o "$OUT/gz_final" \
  python tools/prof_one.py --schedule gz --sweeps 1 --reps 2 > "$OUT/ncu_full.log" 2>&1
timeout 1200 python tools/ordering_study.py --config C4 > "$OUT/ostudy_C4.log" 2>&1
timeout 900 python tools/ordering_study.py --config CP --orderings original,random,bfs,rbfs,rcm,dfs,rdr > "$OUT/ostudy_CP.log" 2>&1
