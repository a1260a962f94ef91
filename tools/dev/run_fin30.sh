#!/bin/bash
export LMS_GZ_VERBOSE=1
timeout 900 python tools/explore.py --config C3 --orderings original,bfs,rdr --sweeps 10 --reps 2 --variants s1:0:0,gz:512:1,gz:1024:1,gz:2048:1 > gpurun_out/fin30_c3.log 2>&1
echo done
