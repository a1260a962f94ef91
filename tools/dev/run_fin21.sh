#!/bin/bash
for r in 1 2; do timeout 600 python bench.py --no-cpu > gpurun_out/fin21_bench$r.log 2>&1; done
echo done
