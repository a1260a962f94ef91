#!/bin/bash
# end-of-session evidence after the identity fast path
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 200 python tools/dev/stress_e2e.py 100 50 2>&1 | grep -E "^ok|FAILED"
timeout 900 python bench.py > gpurun_out/final7_bench.log 2>&1; echo "bench rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29541 bench.py --force-dist --steps 2 --warmup 3 > gpurun_out/final7_dist.log 2>&1; echo "dist rc=$?"
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final7_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 300 python tools/prof_e2e.py --steps 2 > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/final7_e2e_launches.csv python tools/prof_e2e.py --steps 2 --prof > /dev/null 2>&1
echo done
