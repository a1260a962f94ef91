#!/bin/bash
timeout 300 python tools/dev/stress_host.py 100 2>&1 | tail -2
