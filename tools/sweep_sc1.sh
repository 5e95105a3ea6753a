#!/bin/bash
cd "$(dirname "$0")/.."
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 11008:4096:3 768:768:3"
M="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3"
echo "== default"; timeout 300 python tools/time_gemv.py --pdl $SH; timeout 300 python tools/time_mix.py $M
echo "== SC=1 (C=16)"; SHIFTADD_CLUSTER_SC=1 timeout 300 python tools/time_gemv.py --pdl $SH; SHIFTADD_CLUSTER_SC=1 timeout 300 python tools/time_mix.py $M
