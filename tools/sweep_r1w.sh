#!/bin/bash
cd "$(dirname "$0")/.."
timeout 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 11008:4096:3 2048:8192:3 768:768:3 4096:1024:2"
echo "== half --pdl"; timeout 300 python tools/time_gemv.py --pdl $SH
echo "== full2 --pdl"; SHIFTADD_CLUSTER_HALF=0 timeout 300 python tools/time_gemv.py --pdl $SH
SHIFTADD_CLUSTER_TRACE=1 timeout 120 python tools/trace_cluster.py 4096 4096 2 --pdl
SHIFTADD_CLUSTER_TRACE=1 timeout 120 python tools/trace_cluster.py 16384 4096 2 --pdl
timeout 900 python tools/bench_extra.py 2>&1 | grep -v Warn | tail -20
