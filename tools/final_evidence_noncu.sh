#!/bin/bash
# final_evidence.sh without the ncu steps (captured separately: tools/dev/run_ncu_final.sh)
# One GPU call for a round's evidence (run from the repo root under gpurun):
# the GPU suite, the suite again on the bounds-checked build, the bench line,
# the reference arm, the multi-GPU path at one rank, the ordering study on
# C4 / CP and the 3D (S2) sweep times on C3.  Logs -> $OUT.
set -u
OUT=${OUT:-gpurun_out/final}
mkdir -p "$OUT"
nvidia-smi > "$OUT/smi.txt" 2>&1
timeout 2400 python -m pytest tests -m gpu -q > "$OUT/gpu_tests.log" 2>&1
LMS_LIB_PATH=$PWD/paper_1606_00803_b200/liblms_bounds.so timeout 2400 python -m pytest tests -m gpu -q > "$OUT/gpu_tests_bounds.log" 2>&1
python bench.py > "$OUT/bench.log" 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > "$OUT/bench_reference.log" 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 1 --force-dist --steps 5 --warmup 3 --no-cpu > "$OUT/bench_dist1.log" 2>&1
timeout 1200 python tools/ordering_study.py --config C4 > "$OUT/ostudy_C4.log" 2>&1
timeout 900 python tools/ordering_study.py --config CP --orderings original,random,bfs,rbfs,rcm,dfs,rdr,rdrw > "$OUT/ostudy_CP.log" 2>&1
timeout 600 python tools/time_sweep.py --config C3 --orderings original,bfs,rdr,random > "$OUT/s2_C3.log" 2>&1
timeout 600 python tools/time_orders.py C4 original,random,bfs,rdr,rdrw > "$OUT/orders_C4.log" 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
