#!/bin/bash
cd "$(dirname "$0")/.."
SH="4096:11008:2 4096:11008:3 2048:11008:3 8192:8192:2 4096:8192:3 5120:13824:2"
echo "== default"; timeout 300 python tools/time_gemv.py --pdl $SH
echo "== C16"; SHIFTADD_CLUSTER_C16=1 timeout 300 python tools/time_gemv.py --pdl $SH
echo "== C16 no size cap"; SHIFTADD_CLUSTER_C16=1 SHIFTADD_CLUSTER_BIGC=1000 timeout 300 python tools/time_gemv.py --pdl $SH
