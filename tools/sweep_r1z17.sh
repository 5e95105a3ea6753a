#!/bin/bash
# two items per consumer warp per stage (IPW2) vs one.
cd "$(dirname "$0")/.."
SHIFTADD_RING_IPW2=1 timeout 600 python -m pytest tests -m gpu -x -q -k "gemv or config or determin or basis or fused or misaligned" 2>&1 | tail -2
M="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3"
for rep in 1 2; do
  echo "== IPW1"; timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1
  echo "== IPW2"; SHIFTADD_RING_IPW2=1 timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1
done
SHIFTADD_RING_IPW2=1 SHIFTADD_CLUSTER_TRACE=1 timeout 120 python tools/trace_cluster.py 16384 4096 3 --pdl 2>&1 | grep -v Warn | head -9
