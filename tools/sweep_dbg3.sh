#!/bin/bash
cd "$(dirname "$0")/.."
export PYTHONUNBUFFERED=1
timeout 300 python tools/debug_randperm.py 2>&1 | tail -8
SHIFTADD_CLUSTER_HALF=0 timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python tools/time_gemv.py --pdl --reps 4 4096:4096:2 16384:4096:3 11008:4096:3 2>&1 | grep -v "^$" | tail -30
