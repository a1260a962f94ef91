#!/bin/bash
for k in 1 2; do timeout 300 python tools/dev/stress_gz.py sweeps 2>&1 | grep -E "ok|FAILED"; done
for k in 1 2; do timeout 300 python tools/dev/stress_gz.py rebuilds 2>&1 | grep -E "ok|FAILED"; done
