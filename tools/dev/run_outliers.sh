#!/bin/bash
timeout 300 python tools/dev/e2e_outliers.py 25 2>&1 | tail -8
LMS_GC_SHIFT=0 timeout 300 python tools/dev/e2e_outliers.py 25 2>&1 | tail -8
