#!/bin/bash
cd "$(dirname "$0")/.."
export PYTHONUNBUFFERED=1
timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python tools/debug_oob.py 11008 4096 3 2>&1 | grep -v "^$" | tail -25
SHIFTADD_CLUSTER_HALF=0 timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python tools/debug_oob.py 11008 4096 3 2>&1 | grep -v "^$" | tail -25
timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python tools/debug_oob.py 4096 11008 2 2>&1 | grep -v "^$" | tail -12
