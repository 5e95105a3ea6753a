#!/bin/bash
# cluster split-K M=1 kernel: parity, timing vs grid split-K, phase traces
cd "$(dirname "$0")/.."
timeout 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -12
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 11008:4096:3 768:768:3 4096:1024:2"
echo "== cluster --pdl"; timeout 300 python tools/time_gemv.py --pdl $SH
echo "== splitk --pdl"; timeout 300 python tools/time_gemv.py --pdl --splitk $SH 8192:8192:2
echo "== cluster C<=8 (K=8192) --pdl"; SHIFTADD_CLUSTER_MAXC=8 timeout 300 python tools/time_gemv.py --pdl 28672:8192:3 2048:8192:3 8192:8192:2 28672:8192:3
for s in "4096 4096 2" "16384 4096 3"; do SHIFTADD_CLUSTER_TRACE=1 timeout 120 python tools/trace_cluster.py $s; done
SHIFTADD_CLUSTER_MAXC=8 SHIFTADD_CLUSTER_TRACE=1 timeout 120 python tools/trace_cluster.py 28672 8192 3
