#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
M="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3"
for rep in 1 2; do
  echo "== base"; (cd _base && timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1)
  echo "== new"; timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1
done
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 11008:4096:3 4096:11008:2 768:768:3"
timeout 300 python tools/time_gemv.py --pdl $SH 2>&1 | grep -v Warn
SHIFTADD_CLUSTER_TRACE=1 timeout 120 python tools/trace_cluster.py 16384 4096 3 --pdl 2>&1 | grep -v Warn | head -10
