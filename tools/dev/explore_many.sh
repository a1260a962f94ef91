#!/bin/bash
# usage: tools/explore_many.sh OUT CONFIG ORDERING "v1 v2 ..." [per-variant timeout]
out=$1; cfg=$2; ord=$3; vars=$4; to=${5:-120}
for v in $vars; do
  timeout $to python tools/explore.py --config $cfg --orderings $ord --variants $v >> $out 2>&1 || echo "{\"failed\": \"$v rc=$?\"}" >> $out
done
