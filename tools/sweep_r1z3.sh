#!/bin/bash
# A/B on one box: round-start kernel (_base worktree) vs in-loop push; clusters of 16 (one
# slice per CTA) for K = 4096.
cd "$(dirname "$0")/.."
M="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3"
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 11008:4096:3 4096:11008:2 768:768:3"
SHIFTADD_CLUSTER_SC=1 timeout 300 python -m pytest tests -m gpu -x -q -k "gemv or config or determin or basis" 2>&1 | tail -2
for rep in 1 2; do
  echo "== base"; (cd _base && timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1)
  echo "== new"; timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1
  echo "== new SC=1"; SHIFTADD_CLUSTER_SC=1 timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1
done
echo "== base per-layer"; (cd _base && timeout 300 python tools/time_gemv.py --pdl $SH 2>&1 | grep -v Warn)
echo "== new per-layer"; timeout 300 python tools/time_gemv.py --pdl $SH 2>&1 | grep -v Warn
echo "== new SC=1 per-layer"; SHIFTADD_CLUSTER_SC=1 timeout 300 python tools/time_gemv.py --pdl $SH 2>&1 | grep -v Warn
for s in "4096 4096 2" "16384 4096 3"; do
  SHIFTADD_CLUSTER_SC=1 SHIFTADD_CLUSTER_TRACE=1 timeout 120 python tools/trace_cluster.py $s --pdl 2>&1 | grep -v Warn | head -14
done
