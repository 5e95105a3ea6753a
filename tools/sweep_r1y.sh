#!/bin/bash
cd "$(dirname "$0")/.."
timeout 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
SHIFTADD_CLUSTER_BTAIL=1 timeout 400 python -m pytest tests -m gpu -x -q -k "gemv or config or determin or basis" 2>&1 | tail -2
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 11008:4096:3 768:768:3"
M="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3"
echo "== full2 async tail"; timeout 300 python tools/time_gemv.py --pdl $SH; timeout 300 python tools/time_mix.py $M
echo "== full2 barrier tail"; SHIFTADD_CLUSTER_BTAIL=1 timeout 300 python tools/time_gemv.py --pdl $SH; SHIFTADD_CLUSTER_BTAIL=1 timeout 300 python tools/time_mix.py $M
echo "== half async"; SHIFTADD_CLUSTER_HALF=1 timeout 300 python tools/time_mix.py $M
echo "== full4"; SHIFTADD_CLUSTER_SC=4 timeout 300 python tools/time_mix.py $M
echo "== splitk"; SHIFTADD_CLUSTER=0 timeout 300 python tools/time_mix.py $M
timeout 600 python bench.py 2>/dev/null | tail -1
