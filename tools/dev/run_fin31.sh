#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fin31_tests.log 2>&1; tail -1 gpurun_out/fin31_tests.log
timeout 900 python tools/explore.py --config C3 --orderings original,bfs,rdr --sweeps 10 --reps 2 --variants s1:0:0 > gpurun_out/fin31_c3.log 2>&1
LMS_S1_XYZ4=0 timeout 900 python tools/explore.py --config C3 --orderings original,bfs --sweeps 10 --reps 2 --variants s1:0:0 > gpurun_out/fin31_c3_soa.log 2>&1
echo done
