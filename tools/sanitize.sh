#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over the hot
# kernels on small meshes (tools/sanitize_run.py checks every result against
# the oracle).  Logs -> gpurun_out/sanitize/, one-line summaries -> stdout.
set -u
OUT=${1:-gpurun_out/sanitize}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for what in all 3d; do
    log="$OUT/${tool}_${what}.log"
    extra=""
    [ "$tool" = memcheck ] && extra="--leak-check no"
    [ "$tool" = racecheck ] && extra="--racecheck-report hazard"
    timeout 1500 $CS --tool $tool $extra --print-limit 50 python tools/sanitize_run.py $what > "$log" 2>&1
    rc=$?
    echo "$tool $what rc=$rc :: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run OK' "$log" | tr '\n' ' ')"
  done
done
