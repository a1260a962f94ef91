#!/bin/bash
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --force-dist --steps 2 --warmup 1 2>&1 | tail -1 | cut -c1-300
timeout 900 python bench.py --config C5 --steps 2 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('C5', round(d['value']/1e9,2), round(d['roofline']['frac'],3))"
timeout 900 python bench.py --config C3 --ordering bfs --steps 2 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('C3 bfs', round(d['value']/1e9,2), round(d['roofline']['frac'],3))"
timeout 900 python bench.py --config C2 --steps 2 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('C2', round(d['value']/1e9,2), round(d['roofline']['frac'],3))"
